// coarsen.cu -- contraction of a graph by a compact partition
// (coarsen, H/louvain.hpp:154-220).  Members are grouped by community with a
// counting scatter, then the row engine (rows.cuh) reduces each coarse row's
// (z[v], w) entries by hash and sorts the distinct coarse neighbours.
// Inter-community entries keep both directions; intra-community entries
// count once (v >= u), so loops carry the internal weight and w(E') = w(E).
#include "rows.cuh"

namespace cdk {

__global__ void k_member_count(int64_t n, const int32_t *z, int32_t *csz) {
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < n;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u = base + threadIdx.x;
        const bool valid = u < n;
        const int32_t c = valid ? z[u] : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        if (valid && (__ffs(peers) - 1) == lane_id())
            atomicAdd(&csz[c], __popc(peers));
    }
}

__global__ void k_member_scatter(int64_t n, const int32_t *z, int64_t *cursor, int32_t *mem) {
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < n;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u = base + threadIdx.x;
        const bool valid = u < n;
        const int32_t c = valid ? z[u] : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        const int leader = __ffs(peers) - 1;
        int64_t b = 0;
        if (valid && leader == lane_id())
            b = static_cast<int64_t>(
                atomicAdd(reinterpret_cast<unsigned long long *>(&cursor[c]), static_cast<unsigned long long>(__popc(peers))));
        b = __shfl_sync(0xffffffffu, b, leader);
        if (valid)
            mem[b + __popc(peers & lanemask_lt())] = static_cast<int32_t>(u);
    }
}

struct CszGen {
    const int32_t *csz;
    __device__ int64_t operator()(int64_t c) const { return csz[c]; }
};
struct MemDegGen {
    const int32_t *mem;
    const int64_t *off;
    __device__ int64_t operator()(int64_t p) const { return off[mem[p] + 1] - off[mem[p]]; }
};

__global__ void k_row_fpre(int64_t nc, const int64_t *moff, const int64_t *mpre, int64_t *fpre) {
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c <= nc;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
        fpre[c] = mpre[moff[c]];
}

__global__ void k_check_used(int64_t nc, const int32_t *csz, int *flag) {
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < nc;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (csz[c] == 0)
            *flag = 1;
}

// ---------------------------------------------------------------------------
// Dense contraction (nc <= COARSEN_DENSE_MAX): a coarse row's tally is a dense
// fp64 array of nc slots in shared memory, indexed by the coarse id -- no
// hashing and no sort: the nonzero slots, read in index order, ARE the sorted
// coarse row.  Members of the row are walked warp by warp.
// ---------------------------------------------------------------------------
constexpr int64_t COARSEN_DENSE_MAX = 8192;  // 64 KB of fp64 slots
constexpr int DENSE_THREADS = 512;
// fine entries per contraction batch (row engine scratch ~24-40 B each)
constexpr int64_t COARSEN_CHUNK_ENTRIES = int64_t(1) << 29;
// batched contraction: coarse rows kept from pass A up to this many bytes
constexpr int64_t COARSEN_KEEP_BYTES = int64_t(16) << 30;

// A: the slot type -- uint32 when every weight is integral and every volume
// below 2^31 (graph int_weights: exact, native shared-memory atomics, half the
// shared memory), else fp64 (shared-memory fp64 adds are CAS loops).
template <class A>
__global__ void __launch_bounds__(DENSE_THREADS, 4) k_dense_rows(int64_t nc, const int64_t *moff, const int32_t *mem,
                                                              const int64_t *mpre, const int64_t *off,
                                                              const int32_t *col, const float *w, const int32_t *z,
                                                              const int64_t *fpre, int32_t *tkey, double *tval,
                                                              int64_t *deg2) {
    extern __shared__ __align__(8) unsigned char dense_smem[];
    A *acc = reinterpret_cast<A *>(dense_smem);
    __shared__ int wsum[DENSE_THREADS / 32 + 1];
    __shared__ double scr[DENSE_THREADS / 32][32];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    constexpr int NW = DENSE_THREADS / 32;
    const int per = static_cast<int>((nc + DENSE_THREADS - 1) / DENSE_THREADS);  // slots per thread
    for (int64_t c = blockIdx.x; c < nc; c += gridDim.x) {
        for (int64_t k = threadIdx.x; k < nc; k += DENSE_THREADS)
            acc[k] = A(0);
        __syncthreads();
        // tally: entry (u -> v) of a member u adds w to slot z[v]; intra-community
        // entries once (v >= u), H/louvain.hpp:180-186.  The row's own slot
        // (most entries: the community's internal weight) is summed in
        // registers; other labels combine per warp (match_any) before the
        // shared-memory atomic.
        // The members' rows are enumerated flat (SrcCoarsen): a warp takes 32
        // consecutive entries of the concatenated rows per step, so short
        // member rows do not leave most lanes idle behind a chain of
        // dependent loads per member.
        double self = 0.0;
        const SrcCoarsen src{moff, mem, mpre, off, col, w, z};
        const int64_t fb = fpre[c], fe = fpre[c + 1];
        if (fb + wid * 32 < fe) {
            auto cur = src.init(c, fb + wid * 32);
            for (int64_t f0 = fb + wid * 32; f0 < fe; f0 += NW * 32) {
                int32_t k;
                double wt;
                bool valid;
                src.load(c, f0, fe, cur, k, wt, valid);
                if (valid && k == static_cast<int32_t>(c)) {
                    self += wt;
                    valid = false;
                }
                double sum;
                if (warp_aggregate_sum(k, wt, valid, scr[wid], sum))
                    atomicAdd(&acc[k], static_cast<A>(sum));
            }
        }
        self = warp_sum(self);
        if (lane == 0 && self != 0.0)
            atomicAdd(&acc[c], static_cast<A>(self));
        __syncthreads();
        // emit the nonzero slots in index order at the row's scratch offset
        const int64_t k0 = static_cast<int64_t>(threadIdx.x) * per;
        int mine = 0;
        for (int i = 0; i < per; ++i)
            mine += (k0 + i < nc && acc[k0 + i] != A(0)) ? 1 : 0;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o)
                incl += t;
        }
        if (lane == 31)
            wsum[wid] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int i = 0; i < NW; ++i) {
                const int t = wsum[i];
                wsum[i] = s;
                s += t;
            }
            wsum[NW] = s;
        }
        __syncthreads();
        int64_t pos = fpre[c] + wsum[wid] + incl - mine;
        for (int i = 0; i < per; ++i) {
            const int64_t k = k0 + i;
            if (k < nc && acc[k] != A(0)) {
                tkey[pos] = static_cast<int32_t>(k);
                tval[pos] = static_cast<double>(acc[k]);
                ++pos;
            }
        }
        if (threadIdx.x == 0)
            deg2[c] = wsum[NW];
        __syncthreads();
    }
}

__global__ void k_dense_copy(int64_t nc, const int64_t *fpre, const int64_t *off2, const int32_t *tkey,
                             const double *tval, int32_t *col, float *w) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t c = gw; c < nc; c += nw) {
        const int64_t s = fpre[c], d = off2[c], len = off2[c + 1] - off2[c];
        for (int64_t i = lane; i < len; i += 32) {
            col[d + i] = tkey[s + i];
            w[d + i] = static_cast<float>(tval[s + i]);
        }
    }
}

static cd_graph *coarsen_dev_impl(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc, bool sorted) {
    const int64_t n = g->n;
    const int grid = grid_for(n, 256, ctx->num_sms * 8);
    DBuf<int32_t> csz(ctx, std::max<int64_t>(nc, 1));
    csz.zero();
    if (n > 0)
        CD_LAUNCH(ctx, "coarsen.prep", k_member_count, grid, 256, 0, n, z, csz.p);
    DBuf<int64_t> moff(ctx, nc + 1);
    exclusive_scan<int64_t>(ctx, nc, CszGen{csz.p}, moff.p, moff.p + nc);
    DBuf<int32_t> mem(ctx, std::max<int64_t>(n, 1));
    {
        DBuf<int64_t> cursor(ctx, nc + 1);
        CD_CUDA(cudaMemcpyAsync(cursor.p, moff.p, (nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (n > 0)
            CD_LAUNCH(ctx, "coarsen.prep", k_member_scatter, grid, 256, 0, n, z, cursor.p, mem.p);
    }
    DBuf<int64_t> mpre(ctx, n + 1);
    exclusive_scan<int64_t>(ctx, n, MemDegGen{mem.p, g->off.p}, mpre.p, mpre.p + n);
    DBuf<int64_t> fpre(ctx, nc + 1);
    CD_LAUNCH(ctx, "coarsen.prep", k_row_fpre, grid_for(nc + 1, 256, ctx->num_sms * 8), 256, 0, nc,
              static_cast<const int64_t *>(moff.p), static_cast<const int64_t *>(mpre.p), fpre.p);
    auto *cg = new cd_graph();
    cg->ctx = ctx;
    cg->n = nc;
    cg->weighted = true;
    if (nc > 0 && nc <= COARSEN_DENSE_MAX) {
        try {
            DBuf<int32_t> tkey(ctx, std::max<int64_t>(g->D, 1));
            DBuf<double> tval(ctx, std::max<int64_t>(g->D, 1));
            DBuf<int64_t> deg2(ctx, nc);
            auto launch = [&](auto kfn, size_t slot) {
                const size_t smem = size_t(nc) * slot;
                CD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(std::max<size_t>(smem, 1))));
                int per_sm = 0;
                CD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, DENSE_THREADS, smem));
                CD_LAUNCH(ctx, "coarsen.dense", kfn, grid_for(nc, 1, std::max(1, per_sm) * ctx->num_sms),
                          DENSE_THREADS, smem, nc, static_cast<const int64_t *>(moff.p),
                          static_cast<const int32_t *>(mem.p), static_cast<const int64_t *>(mpre.p),
                          static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p),
                          static_cast<const float *>(g->weighted ? g->w.p : nullptr), z,
                          static_cast<const int64_t *>(fpre.p), tkey.p, tval.p, deg2.p);
            };
            // integral weights whose total volume fits uint32: every slot sum does
            if (g->int_weights && 2.0 * g->total < 4294967296.0)
                launch(k_dense_rows<uint32_t>, sizeof(uint32_t));
            else
                launch(k_dense_rows<double>, sizeof(double));
            cg->off.alloc(ctx, nc + 1);
            exclusive_scan<int64_t>(ctx, nc, ArrayGen<int64_t>{deg2.p}, cg->off.p, cg->off.p + nc);
            CD_CUDA(cudaMemcpyAsync(&cg->D, cg->off.p + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
            CD_CUDA(cudaStreamSynchronize(ctx->stream));
            cg->col.alloc(ctx, std::max<int64_t>(cg->D, 1));
            cg->w.alloc(ctx, std::max<int64_t>(cg->D, 1));
            CD_LAUNCH(ctx, "coarsen.dense", k_dense_copy, grid_for(nc, 8, ctx->num_sms * 8), 256, 0, nc,
                      static_cast<const int64_t *>(fpre.p), static_cast<const int64_t *>(cg->off.p),
                      static_cast<const int32_t *>(tkey.p), static_cast<const double *>(tval.p), cg->col.p,
                      cg->w.p);
            graph_finalize(ctx, cg, g->int_weights);
        } catch (...) {
            delete cg;
            throw;
        }
        return cg;
    }
    try {
        SrcCoarsen src{moff.p, mem.p, mpre.p, g->off.p, g->col.p, g->weighted ? g->w.p : nullptr, z};
        bool want_w = true;
        const int64_t chunk = env_i64("CD_COARSEN_CHUNK_ENTRIES", COARSEN_CHUNK_ENTRIES);
        if (g->D <= chunk) {
            cg->D = run_row_engine(ctx, src, nc, fpre.p, g->D, std::max<int64_t>(nc, 1), DUP_SUM, want_w, cg->off,
                                   cg->col, cg->w, nullptr, "coarsen", sorted);
        } else {
            // the engine's scratch is ~24-40 B per fine entry: contract in
            // batches of coarse rows holding ~chunk fine entries each.  Pass
            // A runs every batch, writes its row offsets and keeps its rows
            // while they fit COARSEN_KEEP_BYTES; once the exact size is known
            // the coarse CSR is allocated and pass B copies the kept batches
            // and recomputes the others (a coarse graph about as large as the
            // fine one -- R-MAT level 0 -- never exists twice)
            const std::vector<int64_t> cut = split_rows(ctx, fpre.p, 0, nc, chunk);
            const size_t nb = cut.size() - 1;
            cg->off.alloc(ctx, nc + 1);
            std::vector<DBuf<int32_t>> kcol(nb);
            std::vector<DBuf<float>> kw(nb);
            std::vector<int64_t> bD(nb, 0), bbase(nb, 0);
            std::vector<char> kept(nb, 0);
            int64_t kept_bytes = 0;
            // keep what the device can hold next to the final CSR (bounded by
            // the fine entry count): free memory plus the pool's idle reserve
            int64_t keep_default = COARSEN_KEEP_BYTES;
            {
                size_t fr = 0, tot = 0;
                uint64_t reserved = 0, used = 0;
                if (cudaMemGetInfo(&fr, &tot) == cudaSuccess &&
                    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
                    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess) {
                    const int64_t avail = static_cast<int64_t>(fr) + static_cast<int64_t>(reserved - used);
                    const int64_t room = avail - g->D * int64_t(sizeof(int32_t) + sizeof(float)) -
                                         2 * chunk * int64_t(24) - (int64_t(8) << 30);
                    keep_default = std::max(keep_default, room);
                }
                cudaGetLastError();
            }
            const int64_t keep_budget = env_i64("CD_COARSEN_KEEP_BYTES", keep_default);
            auto run_batch = [&](size_t b, DBuf<int64_t> &boff, DBuf<int32_t> &bcol, DBuf<float> &bw) {
                const int64_t c0 = cut[b], rows = cut[b + 1] - c0;
                int64_t pr[2];
                CD_CUDA(cudaMemcpyAsync(&pr[0], fpre.p + c0, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
                CD_CUDA(cudaMemcpyAsync(&pr[1], fpre.p + c0 + rows, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                        ctx->stream));
                CD_CUDA(cudaStreamSynchronize(ctx->stream));
                DBuf<int64_t> bpre(ctx, rows + 1);
                CD_LAUNCH(ctx, "coarsen.prep", k_rebase, grid_for(rows + 1, 256, ctx->num_sms * 8), 256, 0, rows + 1,
                          static_cast<const int64_t *>(fpre.p + c0), pr[0], int64_t(0), bpre.p);
                SrcWindow<SrcCoarsen> win{src, c0, pr[0]};
                bool bw_want = true;
                return run_row_engine(ctx, win, rows, bpre.p, pr[1] - pr[0], std::max<int64_t>(nc, 1), DUP_SUM,
                                      bw_want, boff, bcol, bw, nullptr, "coarsen", sorted);
            };
            int64_t D = 0;
            for (size_t b = 0; b < nb; ++b) {
                const int64_t c0 = cut[b], rows = cut[b + 1] - c0;
                bbase[b] = D;
                if (rows == 0)
                    continue;
                DBuf<int64_t> boff;
                bD[b] = run_batch(b, boff, kcol[b], kw[b]);
                CD_LAUNCH(ctx, "coarsen.prep", k_rebase, grid_for(rows, 256, ctx->num_sms * 8), 256, 0, rows,
                          static_cast<const int64_t *>(boff.p), int64_t(0), D, cg->off.p + c0);
                const int64_t bytes = bD[b] * int64_t(sizeof(int32_t) + sizeof(float));
                if (kept_bytes + bytes <= keep_budget) {
                    kept[b] = 1;
                    kept_bytes += bytes;
                } else {
                    kcol[b].release();
                    kw[b].release();
                }
                D += bD[b];
            }
            cg->D = D;
            cg->col.alloc(ctx, std::max<int64_t>(D, 1));
            cg->w.alloc(ctx, std::max<int64_t>(D, 1));
            for (size_t b = 0; b < nb; ++b) {
                if (cut[b + 1] == cut[b] || bD[b] == 0)
                    continue;
                if (!kept[b]) {
                    DBuf<int64_t> boff;
                    run_batch(b, boff, kcol[b], kw[b]);
                }
                CD_CUDA(cudaMemcpyAsync(cg->col.p + bbase[b], kcol[b].p, bD[b] * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, ctx->stream));
                CD_CUDA(cudaMemcpyAsync(cg->w.p + bbase[b], kw[b].p, bD[b] * sizeof(float), cudaMemcpyDeviceToDevice,
                                        ctx->stream));
                kcol[b].release();
                kw[b].release();
            }
            CD_LAUNCH(ctx, "coarsen.prep", k_fill_i64, 1, 32, 0, int64_t(1), D, cg->off.p + nc);
        }
        graph_finalize(ctx, cg, g->int_weights);
    } catch (...) {
        delete cg;
        throw;
    }
    return cg;
}

// API-level check that z is a compact labelling of [0, nc)
bool is_compact_dev(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t nc) {
    DBuf<int32_t> csz(ctx, std::max<int64_t>(nc, 1));
    csz.zero();
    DBuf<int> flag(ctx, 1);
    flag.zero();
    if (n > 0)
        CD_LAUNCH(ctx, "coarsen.prep", k_member_count, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n, z, csz.p);
    CD_LAUNCH(ctx, "coarsen.prep", k_check_used, grid_for(nc, 256, ctx->num_sms * 8), 256, 0, nc,
              static_cast<const int32_t *>(csz.p), flag.p);
    int h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return h == 0;
}

}  // namespace cdk

namespace cdk {
// Contraction with its algorithmic bytes: 12 B per fine node
// (offsets + label), 8 (+4 weighted) B per fine entry (column + label gather
// [+ weight]), 8 B per coarse entry (column + weight) and per coarse node
// (offset), recorded as "coarsen.model" for the contraction roofline.
cd_graph *coarsen_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc, bool sorted) {
    cd_graph *cg = coarsen_dev_impl(ctx, g, z, nc, sorted);
    if (ctx->profiling)
        add_stat_work(ctx, "coarsen.model",
                      12.0 * g->n + (g->weighted ? 12.0 : 8.0) * g->D + 8.0 * cg->D + 8.0 * cg->n,
                      static_cast<double>(g->D));
    return cg;
}
}  // namespace cdk
