// graph.cu -- device CSR construction (Graph::from_edges, H/graph.hpp:48-81),
// finalize (H/graph.hpp:229-255), validation and the degree-tier work
// decomposition used by the sweep / move kernels.
#include "rows.cuh"

namespace cdk {

// ---------------------------------------------------------------------------
// finalize: vol(u) = sum w + loop (loop twice), loop(u), m, w(E), max degree
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_finalize(int64_t n, const int64_t *off, const int32_t *col,
                                                  const float *w, double *vol, double *loop, int64_t *acc_i,
                                                  double *acc_d) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int64_t m_loc = 0, maxdeg = 0, iso = 0;
    double tot_loc = 0.0, maxvol = 0.0;
    bool frac = false;
    for (int64_t u = gw; u < n; u += nw) {
        const int64_t s = off[u], e = off[u + 1];
        double vs = 0.0, lp = 0.0, up = 0.0;
        int64_t cnt = 0;
        for (int64_t i = s + lane; i < e; i += 32) {
            const int32_t v = col[i];
            const double wt = w ? static_cast<double>(w[i]) : 1.0;
            frac |= wt != floor(wt);
            vs += wt;
            if (v == u) {
                lp += wt;
                up += wt;
                ++cnt;
            } else if (v > u) {
                up += wt;
                ++cnt;
            }
        }
        vs = warp_sum(vs);
        lp = warp_sum(lp);
        up = warp_sum(up);
        cnt = warp_sum(cnt);
        if (lane == 0) {
            vol[u] = vs + lp;
            loop[u] = lp;
        }
        m_loc += cnt;
        tot_loc += up;
        maxdeg = max(maxdeg, e - s);
        maxvol = fmax(maxvol, vs + lp);
        iso += (e == s);
    }
    const bool any_frac = __any_sync(0xffffffffu, frac);
    if (lane == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i[0]), static_cast<unsigned long long>(m_loc));
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[1]), static_cast<unsigned long long>(maxdeg));
        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i[2]), static_cast<unsigned long long>(iso));
        if (any_frac)
            atomicOr(reinterpret_cast<unsigned long long *>(&acc_i[3]), 1ULL);
        // vol >= 0: the bit pattern of a non-negative double orders like its value
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[4]), static_cast<unsigned long long>(__double_as_longlong(maxvol)));
        atomicAdd(acc_d, tot_loc);
    }
}

// ---------------------------------------------------------------------------
// entry-parallel passes over a CSR: a thread per CSR_CHUNK consecutive
// entries finds its first row by binary search and walks the row boundaries,
// so hubs and the many tiny / empty rows of R-MAT cost the same per entry
// (a warp per row spent most of its time on 16.7M mostly short or empty rows:
// C3 finalize 8.8 ms -> one read of the columns)
// ---------------------------------------------------------------------------
constexpr int CSR_CHUNK = 16;

__device__ __forceinline__ int64_t row_of_entry(int64_t n, const int64_t *off, int64_t i) {
    int64_t lo = 0, hi = n - 1;  // last r with off[r] <= i (clamped: offsets may be invalid here)
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= i)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// offsets: off[0] = 0, nondecreasing, off[n] = D
__global__ void k_check_offsets(int64_t n, int64_t D, const int64_t *off, int64_t *flag) {
    bool bad = false;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = off[u], e = off[u + 1];
        bad |= s > e || s < 0 || e > D || (u == 0 && s != 0) || (u == n - 1 && e != D);
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0)
        flag[0] = 1;
}

// ranges, strictly ascending rows, weights > 0; FIN (unweighted graphs): also
// the self-loop count per row and the number of entries with v >= u (= m = w(E))
// (entries [ib, ie) of D; one launch covers [0, D))
template <bool FIN>
__global__ void __launch_bounds__(256) k_csr_entries(int64_t n, int64_t D, const int64_t *off, const int32_t *col,
                                                    const float *w, int64_t *flag, int32_t *loops,
                                                    unsigned long long *m_acc, int64_t ib = 0, int64_t ie = -1) {
    bool bad = false;
    unsigned long long m_loc = 0;
    if (ie < 0)
        ie = D;
    for (int64_t i0 = ib + (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * CSR_CHUNK; i0 < ie;
         i0 += static_cast<int64_t>(gridDim.x) * blockDim.x * CSR_CHUNK) {
        int64_t r = row_of_entry(n, off, i0);
        int64_t rs = off[r], re = off[r + 1];
        const int64_t i1 = min(i0 + CSR_CHUNK, ie);
        int32_t prev = i0 > 0 ? col[i0 - 1] : 0;
        for (int64_t i = i0; i < i1; ++i) {
            for (int guard = 0; i >= re && r + 1 < n && guard < 64; ++guard) {  // next nonempty row
                ++r;
                rs = re;
                re = off[r + 1];
            }
            if (i >= re) {  // more advance than the guard allows: finish by search
                r = row_of_entry(n, off, i);
                rs = off[r];
                re = off[r + 1];
            }
            const int32_t c = col[i];
            bad |= c < 0 || c >= n || (i > rs && prev >= c);
            if (w)
                bad |= !(w[i] > 0.0f);
            if (FIN && c >= r) {
                ++m_loc;
                if (c == r)
                    atomicAdd(&loops[r], 1);
            }
            prev = c;
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0)
        flag[0] = 1;
    if (FIN) {
        m_loc = warp_sum(m_loc);
        if (lane_id() == 0 && m_loc)
            atomicAdd(m_acc, m_loc);
    }
}

// integral weights (contractions of integer-weight graphs): per-row sums are
// exact in fp64 in any order, so the same entry-parallel walk sums each run
// of a row's entries in a register and adds it to the row once (rows split
// across threads add one partial per thread)
__global__ void __launch_bounds__(256) k_csr_entries_intw(int64_t n, int64_t D, const int64_t *off,
                                                         const int32_t *col, const float *w, double *vsum,
                                                         double *loop, unsigned long long *acc,
                                                         double *tot_acc) {
    unsigned long long m_loc = 0, frac = 0;
    double tot = 0.0;
    for (int64_t i0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * CSR_CHUNK; i0 < D;
         i0 += static_cast<int64_t>(gridDim.x) * blockDim.x * CSR_CHUNK) {
        int64_t r = row_of_entry(n, off, i0);
        int64_t re = off[r + 1];
        const int64_t i1 = min(i0 + CSR_CHUNK, D);
        // the chunk's entries first, as 16-byte loads all in flight: loaded one by one
        // inside the walk, every load waited behind the previous entry's atomics
        // (the pass ran at 0.9 TB/s)
        static_assert(CSR_CHUNK % 4 == 0, "vector loads");
        int32_t cbuf[CSR_CHUNK];
        float wbuf[CSR_CHUNK];
        if (i1 - i0 == CSR_CHUNK) {
#pragma unroll
            for (int k = 0; k < CSR_CHUNK / 4; ++k) {
                const int4 a = __ldcs(reinterpret_cast<const int4 *>(col + i0) + k);
                const float4 b = __ldcs(reinterpret_cast<const float4 *>(w + i0) + k);
                cbuf[4 * k] = a.x, cbuf[4 * k + 1] = a.y, cbuf[4 * k + 2] = a.z, cbuf[4 * k + 3] = a.w;
                wbuf[4 * k] = b.x, wbuf[4 * k + 1] = b.y, wbuf[4 * k + 2] = b.z, wbuf[4 * k + 3] = b.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < CSR_CHUNK; ++k) {
                cbuf[k] = i0 + k < i1 ? col[i0 + k] : 0;
                wbuf[k] = i0 + k < i1 ? w[i0 + k] : 0.0f;
            }
        }
        double run = 0.0;
#pragma unroll
        for (int k = 0; k < CSR_CHUNK; ++k) {
            const int64_t i = i0 + k;
            if (i >= i1)
                break;
            if (i >= re) {
                if (run != 0.0)
                    atomicAdd(&vsum[r], run);
                run = 0.0;
                for (int guard = 0; i >= re && r + 1 < n && guard < 64; ++guard)
                    re = off[++r + 1];
                if (i >= re) {
                    r = row_of_entry(n, off, i);
                    re = off[r + 1];
                }
            }
            const int32_t c = cbuf[k];
            const double wt = static_cast<double>(wbuf[k]);
            frac |= wt != floor(wt);
            run += wt;
            if (c >= r) {
                ++m_loc;
                tot += wt;
                if (c == r)
                    atomicAdd(&loop[r], wt);
            }
        }
        if (run != 0.0)
            atomicAdd(&vsum[r], run);
    }
    m_loc = warp_sum(m_loc);
    tot = warp_sum(tot);
    frac = __any_sync(0xffffffffu, frac != 0);
    if (lane_id() == 0) {
        if (m_loc)
            atomicAdd(&acc[0], m_loc);
        if (frac)
            atomicOr(&acc[3], 1ULL);
        if (tot != 0.0)
            atomicAdd(tot_acc, tot);
    }
}

__global__ void __launch_bounds__(256) k_finalize_nodes_w(int64_t n, const int64_t *off, double *vol,
                                                          const double *loop, int64_t *acc_i) {
    int64_t maxdeg = 0, iso = 0;
    double maxvol = 0.0;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t d = off[u + 1] - off[u];
        const double v = vol[u] + loop[u];  // the loop twice
        vol[u] = v;
        maxdeg = max(maxdeg, d);
        maxvol = fmax(maxvol, v);
        iso += d == 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        maxdeg = max(maxdeg, __shfl_xor_sync(0xffffffffu, maxdeg, o));
        maxvol = fmax(maxvol, __shfl_xor_sync(0xffffffffu, maxvol, o));
        iso += __shfl_xor_sync(0xffffffffu, iso, o);
    }
    if (lane_id() == 0) {
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[1]), static_cast<unsigned long long>(maxdeg));
        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i[2]), static_cast<unsigned long long>(iso));
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[4]),
                  static_cast<unsigned long long>(__double_as_longlong(maxvol)));
    }
}

// unweighted finalize, per node: vol = degree + loop (the loop twice)
__global__ void __launch_bounds__(256) k_finalize_unweighted(int64_t n, const int64_t *off, const int32_t *loops,
                                                             double *vol, double *loop, int64_t *acc_i) {
    int64_t maxdeg = 0, iso = 0;
    double maxvol = 0.0;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t d = off[u + 1] - off[u];
        const double lp = static_cast<double>(loops[u]);
        vol[u] = static_cast<double>(d) + lp;
        loop[u] = lp;
        maxdeg = max(maxdeg, d);
        maxvol = fmax(maxvol, static_cast<double>(d) + lp);
        iso += d == 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        maxdeg = max(maxdeg, __shfl_xor_sync(0xffffffffu, maxdeg, o));
        maxvol = fmax(maxvol, __shfl_xor_sync(0xffffffffu, maxvol, o));
        iso += __shfl_xor_sync(0xffffffffu, iso, o);
    }
    if (lane_id() == 0) {
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[1]), static_cast<unsigned long long>(maxdeg));
        atomicAdd(reinterpret_cast<unsigned long long *>(&acc_i[2]), static_cast<unsigned long long>(iso));
        atomicMax(reinterpret_cast<unsigned long long *>(&acc_i[4]),
                  static_cast<unsigned long long>(__double_as_longlong(maxvol)));
    }
}

void graph_finalize(cd_ctx *ctx, cd_graph *g, bool integral_weights) {
    g->vol.alloc(ctx, std::max<int64_t>(g->n, 1));
    g->loop.alloc(ctx, std::max<int64_t>(g->n, 1));
    DBuf<int64_t> acc_i(ctx, 5);
    DBuf<double> acc_d(ctx, 1);
    acc_i.zero();
    acc_d.zero();
    if (g->n > 0 && !g->weighted) {
        // integer counts: order-free, so entry-parallel (m = w(E) = entries with v >= u)
        DBuf<int32_t> loops(ctx, g->n);
        loops.zero();
        DBuf<int64_t> flag(ctx, 1);
        const int eg = grid_for((g->D + CSR_CHUNK - 1) / CSR_CHUNK, 256, ctx->num_sms * 32);
        if (g->D)
            CD_LAUNCH(ctx, "finalize", k_csr_entries<true>, eg, 256, 0, g->n, g->D,
                      static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p),
                      static_cast<const float *>(nullptr), flag.p, loops.p,
                      reinterpret_cast<unsigned long long *>(acc_i.p));
        CD_LAUNCH(ctx, "finalize", k_finalize_unweighted, grid_for(g->n, 256, ctx->num_sms * 16), 256, 0, g->n,
                  static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(loops.p), g->vol.p,
                  g->loop.p, acc_i.p);
        int64_t hi[5];
        CD_CUDA(cudaMemcpyAsync(hi, acc_i.p, sizeof(hi), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        g->m = hi[0];
        g->max_degree = hi[1];
        g->isolated = hi[2];
        std::memcpy(&g->max_vol, &hi[4], sizeof(double));
        g->int_weights = g->max_vol < 2147483648.0;
        g->total = static_cast<double>(hi[0]);
        g->binned = false;
        return;
    }
    if (g->n > 0 && g->weighted && integral_weights) {
        g->vol.zero();
        g->loop.zero();
        if (g->D)
            CD_LAUNCH(ctx, "finalize", k_csr_entries_intw,
                      grid_for((g->D + CSR_CHUNK - 1) / CSR_CHUNK, 256, ctx->num_sms * 32), 256, 0, g->n, g->D,
                      static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p),
                      static_cast<const float *>(g->w.p), g->vol.p, g->loop.p,
                      reinterpret_cast<unsigned long long *>(acc_i.p), acc_d.p);
        CD_LAUNCH(ctx, "finalize", k_finalize_nodes_w, grid_for(g->n, 256, ctx->num_sms * 16), 256, 0, g->n,
                  static_cast<const int64_t *>(g->off.p), g->vol.p, static_cast<const double *>(g->loop.p), acc_i.p);
        int64_t hi[5];
        double hd;
        CD_CUDA(cudaMemcpyAsync(hi, acc_i.p, sizeof(hi), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaMemcpyAsync(&hd, acc_d.p, sizeof(hd), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        if (hi[3] == 0) {
            g->m = hi[0];
            g->max_degree = hi[1];
            g->isolated = hi[2];
            std::memcpy(&g->max_vol, &hi[4], sizeof(double));
            g->int_weights = g->max_vol < 2147483648.0;
            g->total = hd;
            g->binned = false;
            return;
        }
        // a fractional weight after all: the fixed-order path below
        acc_i.zero();
        acc_d.zero();
    }
    if (g->n > 0)
        CD_LAUNCH(ctx, "finalize", k_finalize, grid_for(g->n, 8, ctx->num_sms * 16), 256, 0, g->n,
                  static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p),
                  static_cast<const float *>(g->weighted ? g->w.p : nullptr), g->vol.p, g->loop.p, acc_i.p, acc_d.p);
    int64_t hi[5];
    double hd;
    CD_CUDA(cudaMemcpyAsync(hi, acc_i.p, sizeof(hi), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&hd, acc_d.p, sizeof(hd), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    g->m = hi[0];
    g->max_degree = hi[1];
    g->isolated = hi[2];
    std::memcpy(&g->max_vol, &hi[4], sizeof(double));
    // exact integer tallies when every weight is integral and sums fit
    g->int_weights = hi[3] == 0 && g->max_vol < 2147483648.0;
    g->total = hd;
    g->binned = false;
}

// ---------------------------------------------------------------------------
// builder from canonical or arbitrary pairs (device arrays)
// ---------------------------------------------------------------------------
__global__ void k_pair_degree(int64_t m, const int32_t *u, const int32_t *v, int32_t *deg) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t a = u[i], b = v[i];
        atomicAdd(&deg[a], 1);
        if (a != b)
            atomicAdd(&deg[b], 1);
    }
}

__global__ void k_pair_scatter(int64_t m, const int32_t *u, const int32_t *v, const float *w, int64_t *cursor,
                               int32_t *rk, float *rw) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t a = u[i], b = v[i];
        const float wt = w ? w[i] : 1.0f;
        int64_t p = static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long *>(&cursor[a]), 1ULL));
        rk[p] = b;
        if (rw)
            rw[p] = wt;
        if (a != b) {
            p = static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long *>(&cursor[b]), 1ULL));
            rk[p] = a;
            if (rw)
                rw[p] = wt;
        }
    }
}

struct DegGen {
    const int32_t *deg;
    __device__ int64_t operator()(int64_t i) const { return deg[i]; }
};

cd_graph *graph_from_pairs(cd_ctx *ctx, int64_t n, int64_t m, const int32_t *u, const int32_t *v, const float *w,
                           DupMode mode) {
    DBuf<int32_t> deg(ctx, std::max<int64_t>(n, 1));
    deg.zero();
    const int blocks = ctx->num_sms * 8;
    if (m > 0)
        CD_LAUNCH(ctx, "build.prep", k_pair_degree, grid_for(m, 256, blocks), 256, 0, m, u, v, deg.p);
    DBuf<int64_t> fpre(ctx, n + 1);
    exclusive_scan<int64_t>(ctx, n, DegGen{deg.p}, fpre.p, fpre.p + n);
    int64_t F = 0;
    CD_CUDA(cudaMemcpyAsync(&F, fpre.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    deg.release();
    DBuf<int32_t> rk(ctx, std::max<int64_t>(F, 1));
    DBuf<float> rw;
    const bool weighted = (w != nullptr) && mode != DUP_ONE;
    if (weighted)
        rw.alloc(ctx, std::max<int64_t>(F, 1));
    {
        DBuf<int64_t> cursor(ctx, n + 1);
        CD_CUDA(cudaMemcpyAsync(cursor.p, fpre.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (m > 0)
            CD_LAUNCH(ctx, "build.prep", k_pair_scatter, grid_for(m, 256, blocks), 256, 0, m, u, v,
                      weighted ? w : static_cast<const float *>(nullptr), cursor.p, rk.p, weighted ? rw.p : nullptr);
    }
    auto *g = new cd_graph();
    g->ctx = ctx;
    g->n = n;
    g->weighted = weighted;
    bool dup = false;
    try {
        SrcFlat src{fpre.p, rk.p, weighted ? rw.p : nullptr};
        bool want_w = weighted;
        g->D = run_row_engine(ctx, src, n, fpre.p, F, std::max<int64_t>(n, 1), mode, want_w, g->off, g->col, g->w,
                              &dup, "build");
        if (dup && mode == DUP_ERROR)
            fail(CD_EINPUT, "duplicate edge");  // H/graph.hpp:178-181
        g->weighted = want_w;
        graph_finalize(ctx, g);
    } catch (...) {
        delete g;
        throw;
    }
    return g;
}

// ---------------------------------------------------------------------------
// row batching helpers (chunked builders and contraction)
// ---------------------------------------------------------------------------
// chunk boundaries: first row whose raw prefix reaches an even split of
// [pre[lo], pre[hi]) into k parts
__global__ void k_split_rows(const int64_t *pre, int64_t lo, int64_t hi, int k, int64_t *cut) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > k)
        return;
    if (i == 0 || i == k) {
        cut[i] = i == 0 ? lo : hi;
        return;
    }
    const int64_t p0 = pre[lo];
    const int64_t target = p0 + static_cast<int64_t>((static_cast<__int128>(pre[hi] - p0) * i) / k);
    int64_t a = lo, b = hi;
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (pre[mid] < target)
            a = mid + 1;
        else
            b = mid;
    }
    cut[i] = a;
}

__global__ void k_rebase(int64_t cnt, const int64_t *src, int64_t sub, int64_t add, int64_t *dst) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i] - sub + add;
}

__global__ void k_fill_i64(int64_t cnt, int64_t value, int64_t *dst) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = value;
}

std::vector<int64_t> split_rows(cd_ctx *ctx, const int64_t *pre_dev, int64_t lo, int64_t hi, int64_t chunk) {
    int64_t pr[2];
    CD_CUDA(cudaMemcpyAsync(&pr[0], pre_dev + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&pr[1], pre_dev + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    chunk = std::max<int64_t>(chunk, 1);
    const int k = static_cast<int>(std::max<int64_t>(1, (pr[1] - pr[0] + chunk - 1) / chunk));
    std::vector<int64_t> cut(k + 1);
    DBuf<int64_t> dcut(ctx, k + 1);
    CD_LAUNCH(ctx, "build.prep", k_split_rows, (k + 256) / 256, 256, 0, pre_dev, lo, hi, k, dcut.p);
    CD_CUDA(cudaMemcpyAsync(cut.data(), dcut.p, (k + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    // drop empty batches
    std::vector<int64_t> out{cut[0]};
    for (int i = 1; i <= k; ++i)
        if (cut[i] > out.back())
            out.push_back(cut[i]);
    if (out.size() == 1)
        out.push_back(hi);
    return out;
}

// ---------------------------------------------------------------------------
// validation of an input CSR (ranges, strictly ascending rows, weights > 0)
// ---------------------------------------------------------------------------
void graph_upload_validate(cd_ctx *ctx, int64_t n, int64_t D, const int64_t *off_dev, int32_t *col_dev,
                           const int32_t *col_host, float *w_dev, const float *w_host, cd_graph *g) {
    if (!ctx->copy_stream)
        CD_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    // one copy stream: chunks alternating over two streams do not interleave (the copy
    // engine drains one stream's chunks first, CD_UPLOAD_TRACE), so chunk 0 would land
    // half-way through and the validation overlap would be lost
    const cudaStream_t cs[2] = {ctx->copy_stream, ctx->copy_stream};
    const bool fin = g != nullptr && w_dev == nullptr && n > 0;
    DBuf<int64_t> flag(ctx, 1);
    flag.zero();
    DBuf<int32_t> loops;
    DBuf<int64_t> acc_i;
    if (fin) {
        loops.alloc(ctx, n);
        loops.zero();
        acc_i.alloc(ctx, 5);
        acc_i.zero();
    }
    if (n)
        CD_LAUNCH(ctx, "validate", k_check_offsets, grid_for(n, 256, ctx->num_sms * 16), 256, 0, n, D, off_dev,
                  flag.p);
    // the copies must not start before the destination buffers exist on the
    // library stream (stream-ordered pool allocations)
    cudaEvent_t ready = ctx_event(ctx);
    CD_CUDA(cudaEventRecord(ready, ctx->stream));
    CD_CUDA(cudaStreamWaitEvent(cs[0], ready, 0));
    const int64_t CH = upload_chunk(D);
    const int64_t nchunks = (D + CH - 1) / CH;
    std::vector<cudaEvent_t> done(static_cast<size_t>(nchunks));
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t ib = c * CH, ie = std::min(D, ib + CH);
        CD_CUDA(cudaMemcpyAsync(col_dev + ib, col_host + ib, (ie - ib) * sizeof(int32_t), cudaMemcpyDefault,
                                cs[c & 1]));
        if (w_dev)  // (the weights may live anywhere: cudaMemcpyDefault)
            CD_CUDA(cudaMemcpyAsync(w_dev + ib, w_host + ib, (ie - ib) * sizeof(float), cudaMemcpyDefault,
                                    cs[c & 1]));
        done[c] = ctx_event(ctx);
        CD_CUDA(cudaEventRecord(done[c], cs[c & 1]));
    }
    auto release = [&] {
        ctx->free_events.push_back(ready);
        for (cudaEvent_t e : done)
            ctx->free_events.push_back(e);
    };
    if (fin) {
        // the degree tiers need only the offsets: checked first, then built on
        // the library stream while the copy stream moves the columns
        int64_t h = 0;
        CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        if (h) {
            CD_CUDA(cudaStreamSynchronize(cs[0]));
            release();
            fail(CD_EINPUT, "malformed CSR (offsets, out-of-range or unsorted neighbours, or nonpositive weight)");
        }
        g->weighted = false;
        graph_ensure_bins(ctx, g);
    }
    // one entry of slack on each side: a chunk's first entry compares with the previous one;
    // an unweighted graph's chunks also count their self-loops and upper entries (finalize)
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t ib = c * CH, ie = std::min(D, ib + CH);
        CD_CUDA(cudaStreamWaitEvent(ctx->stream, done[c], 0));
        const int grid = grid_for((ie - ib + CSR_CHUNK - 1) / CSR_CHUNK, 256, ctx->num_sms * 32);
        if (fin)
            CD_LAUNCH(ctx, "validate", k_csr_entries<true>, grid, 256, 0, n, D, off_dev,
                      static_cast<const int32_t *>(col_dev), static_cast<const float *>(nullptr), flag.p, loops.p,
                      reinterpret_cast<unsigned long long *>(acc_i.p), ib, ie);
        else
            CD_LAUNCH(ctx, "validate", k_csr_entries<false>, grid, 256, 0, n, D, off_dev,
                      static_cast<const int32_t *>(col_dev), static_cast<const float *>(w_dev), flag.p,
                      static_cast<int32_t *>(nullptr), static_cast<unsigned long long *>(nullptr), ib, ie);
    }
    if (fin) {
        g->vol.alloc(ctx, n);
        g->loop.alloc(ctx, n);
        CD_LAUNCH(ctx, "finalize", k_finalize_unweighted, grid_for(n, 256, ctx->num_sms * 16), 256, 0, n, off_dev,
                  static_cast<const int32_t *>(loops.p), g->vol.p, g->loop.p, acc_i.p);
    }
    int64_t h = 0, hi[5] = {};
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    if (fin)
        CD_CUDA(cudaMemcpyAsync(hi, acc_i.p, sizeof(hi), cudaMemcpyDeviceToHost, ctx->stream));
    cudaEvent_t fin_ev = nullptr;
    static const bool trace = std::getenv("CD_UPLOAD_TRACE") != nullptr;
    if (trace) {
        fin_ev = ctx_event(ctx);
        CD_CUDA(cudaEventRecord(fin_ev, ctx->stream));
    }
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (trace) {  // diagnostic: when each chunk landed and when the graph was ready, ms after `ready`
        std::fprintf(stderr, "[cd upload] chunks landed (ms after the offsets check):");
        for (cudaEvent_t e : done) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ready, e);
            std::fprintf(stderr, " %.2f", ms);
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ready, fin_ev);
        std::fprintf(stderr, "; ready %.2f\n", ms);
        ctx->free_events.push_back(fin_ev);
    }
    release();
    if (h)
        fail(CD_EINPUT, "malformed CSR (offsets, out-of-range or unsorted neighbours, or nonpositive weight)");
    if (fin) {  // graph_finalize's unweighted path, from the chunks' counts
        g->m = hi[0];
        g->max_degree = hi[1];
        g->isolated = hi[2];
        std::memcpy(&g->max_vol, &hi[4], sizeof(double));
        g->int_weights = g->max_vol < 2147483648.0;
        g->total = static_cast<double>(hi[0]);
    }
}

void graph_validate_csr(cd_ctx *ctx, int64_t n, const int64_t *off, const int32_t *col, const float *w, int64_t D) {
    if (n == 0)
        return;
    DBuf<int64_t> flag(ctx, 1);
    flag.zero();
    CD_LAUNCH(ctx, "validate", k_check_offsets, grid_for(n, 256, ctx->num_sms * 16), 256, 0, n, D, off, flag.p);
    if (D)
        CD_LAUNCH(ctx, "validate", k_csr_entries<false>, grid_for((D + CSR_CHUNK - 1) / CSR_CHUNK, 256,
                                                                  ctx->num_sms * 32),
                  256, 0, n, D, off, col, w, flag.p, static_cast<int32_t *>(nullptr),
                  static_cast<unsigned long long *>(nullptr));
    int64_t h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h)
        fail(CD_EINPUT, "malformed CSR (offsets, out-of-range or unsorted neighbours, or nonpositive weight)");
}

// ---------------------------------------------------------------------------
// degree tiers and hub tables
// ---------------------------------------------------------------------------
__global__ void k_tiers(int64_t n, const int64_t *off, int64_t cluster_max, uint8_t *tier,
                        unsigned long long *counts) {
    __shared__ unsigned int sc[NUM_TIERS];
    if (threadIdx.x < NUM_TIERS)
        sc[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int t = tier_of_degree(off[u + 1] - off[u], cluster_max);
        tier[u] = static_cast<uint8_t>(t);
        if (t != TIER_NONE)
            atomicAdd(&sc[t], 1u);
    }
    __syncthreads();
    if (threadIdx.x < NUM_TIERS && sc[threadIdx.x])
        atomicAdd(&counts[threadIdx.x], static_cast<unsigned long long>(sc[threadIdx.x]));
}

// Stable partition of the nodes by tier in one pass for all tiers (was one
// scan + scatter per tier: 18 passes over n per graph, 6 graphs per C3 PLM
// run): blocks of TP_NODES consecutive nodes count their tiers, one scan over
// the tier-major (tier, block) counts gives every block's base per tier, and
// the blocks place their nodes in ascending order.
constexpr int TP_THREADS = 256, TP_ROUNDS = 8, TP_NODES = TP_THREADS * TP_ROUNDS;

__global__ void __launch_bounds__(TP_THREADS) k_tier_blockcount(int64_t n, const uint8_t *tier, int64_t nblk,
                                                                int32_t *bc) {
    __shared__ int c[NUM_TIERS];
    if (threadIdx.x < NUM_TIERS)
        c[threadIdx.x] = 0;
    __syncthreads();
    const int lane = lane_id();
    for (int r = 0; r < TP_ROUNDS; ++r) {
        const int64_t u = static_cast<int64_t>(blockIdx.x) * TP_NODES + r * TP_THREADS + threadIdx.x;
        const int t = u < n ? tier[u] : TIER_NONE;
#pragma unroll
        for (int tt = 0; tt < NUM_TIERS; ++tt) {
            const uint32_t m = __ballot_sync(0xffffffffu, t == tt);
            if (lane == 0 && m)
                atomicAdd(&c[tt], __popc(m));
        }
    }
    __syncthreads();
    if (threadIdx.x < NUM_TIERS)
        bc[threadIdx.x * nblk + blockIdx.x] = c[threadIdx.x];
}

__global__ void __launch_bounds__(TP_THREADS) k_tier_place(int64_t n, const uint8_t *tier, int64_t nblk,
                                                           const int32_t *boff, int32_t *tlist) {
    __shared__ int base[NUM_TIERS];
    __shared__ int wcnt[TP_THREADS / 32][NUM_TIERS];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    if (threadIdx.x < NUM_TIERS)
        base[threadIdx.x] = boff[threadIdx.x * nblk + blockIdx.x];
    __syncthreads();
    for (int r = 0; r < TP_ROUNDS; ++r) {
        const int64_t u = static_cast<int64_t>(blockIdx.x) * TP_NODES + r * TP_THREADS + threadIdx.x;
        const int t = u < n ? tier[u] : TIER_NONE;
        int rank = 0;
#pragma unroll
        for (int tt = 0; tt < NUM_TIERS; ++tt) {
            const uint32_t m = __ballot_sync(0xffffffffu, t == tt);
            if (lane == 0)
                wcnt[wid][tt] = __popc(m);
            if (t == tt)
                rank = __popc(m & lanemask_lt());
        }
        __syncthreads();
        if (t < NUM_TIERS) {
            int pre = base[t];
            for (int w = 0; w < wid; ++w)
                pre += wcnt[w][t];
            tlist[pre + rank] = static_cast<int32_t>(u);
        }
        __syncthreads();
        if (threadIdx.x < NUM_TIERS) {
            int add = 0;
            for (int w = 0; w < TP_THREADS / 32; ++w)
                add += wcnt[w][threadIdx.x];
            base[threadIdx.x] += add;
        }
        __syncthreads();
    }
}

struct HubChunkGen {
    const int32_t *hubs;
    const int64_t *off;
    __device__ int64_t operator()(int64_t h) const {
        const int64_t d = off[hubs[h] + 1] - off[hubs[h]];
        return (d + HUB_CHUNK - 1) / HUB_CHUNK;
    }
};


struct HubPartGen {
    const int32_t *hubs;
    const int64_t *off;
    __device__ int64_t operator()(int64_t h) const {
        return int64_t(1) << hub_pbits_of(off[hubs[h] + 1] - off[hubs[h]]);
    }
};

__global__ void k_hub_chunks(int64_t nh, const int32_t *hubs, const int64_t *off, const int64_t *chunk_pre,
                             const int64_t *pbase, int32_t *pbits, int32_t *chunk_hub, int32_t *chunk_part,
                             int32_t *part_hub) {
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t d = off[hubs[h] + 1] - off[hubs[h]];
        if (threadIdx.x == 0)
            pbits[h] = hub_pbits_of(d);
        const int64_t nch = (d + HUB_CHUNK - 1) / HUB_CHUNK;
        for (int64_t k = threadIdx.x; k < nch; k += blockDim.x) {
            chunk_hub[chunk_pre[h] + k] = static_cast<int32_t>(h);
            chunk_part[chunk_pre[h] + k] = static_cast<int32_t>(k);
        }
        for (int64_t q = pbase[h] + threadIdx.x; q < pbase[h + 1]; q += blockDim.x)
            part_hub[q] = static_cast<int32_t>(h);
    }
}

void graph_ensure_bins(cd_ctx *ctx, cd_graph *g) {
    if (g->binned)
        return;
    const int64_t n = g->n;
    g->tier.alloc(ctx, std::max<int64_t>(n, 1));
    DBuf<unsigned long long> counts(ctx, NUM_TIERS);
    counts.zero();
    if (n > 0)
        CD_LAUNCH(ctx, "bins", k_tiers, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n,
                  static_cast<const int64_t *>(g->off.p),
                  // distributed-smem fp64 atomics are slow: real-weight graphs keep the HUB path
                  (g->weighted && !g->int_weights) ? int64_t(0) : CLUSTER_MAX_DEG, g->tier.p, counts.p);
    unsigned long long hc[NUM_TIERS];
    CD_CUDA(cudaMemcpyAsync(hc, counts.p, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t s = 0;
    for (int t = 0; t < NUM_TIERS; ++t) {
        g->tier_nodes[t] = static_cast<int64_t>(hc[t]);
        g->tier_start[t] = s;
        s += g->tier_nodes[t];
    }
    g->tier_start[NUM_TIERS] = s;
    g->tlist.alloc(ctx, std::max<int64_t>(s, 1));
    if (s > 0) {
        // stable partition by tier (ascending id within a tier), all tiers at once
        const int64_t nblk = (n + TP_NODES - 1) / TP_NODES;
        DBuf<int32_t> bc(ctx, NUM_TIERS * nblk), boff(ctx, NUM_TIERS * nblk + 1);
        CD_LAUNCH(ctx, "bins", k_tier_blockcount, static_cast<int>(nblk), TP_THREADS, 0, n,
                  static_cast<const uint8_t *>(g->tier.p), nblk, bc.p);
        exclusive_scan<int32_t>(ctx, NUM_TIERS * nblk, ArrayGen<int32_t>{bc.p}, boff.p, boff.p + NUM_TIERS * nblk);
        CD_LAUNCH(ctx, "bins", k_tier_place, static_cast<int>(nblk), TP_THREADS, 0, n,
                  static_cast<const uint8_t *>(g->tier.p), nblk, static_cast<const int32_t *>(boff.p), g->tlist.p);
    }
    // hubs
    g->n_hubs = g->tier_nodes[TIER_HUB];
    g->n_hub_chunks = 0;
    g->n_hub_parts = 0;
    g->hub_entries = 0;
    g->hubs = g->tlist.p + g->tier_start[TIER_HUB];
    if (g->n_hubs > 0) {
        const int64_t nh = g->n_hubs;
        DBuf<int64_t> chunk_pre(ctx, nh + 1);
        g->hub_pbase.alloc(ctx, nh + 1);
        exclusive_scan<int64_t>(ctx, nh, HubChunkGen{g->hubs, g->off.p}, chunk_pre.p, chunk_pre.p + nh);
        exclusive_scan<int64_t>(ctx, nh, HubPartGen{g->hubs, g->off.p}, g->hub_pbase.p, g->hub_pbase.p + nh);
        int64_t tot[2];
        CD_CUDA(cudaMemcpyAsync(&tot[0], chunk_pre.p + nh, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaMemcpyAsync(&tot[1], g->hub_pbase.p + nh, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        g->n_hub_chunks = tot[0];
        g->n_hub_parts = tot[1];
        g->hub_pbits.alloc(ctx, nh);
        g->chunk_hub.alloc(ctx, g->n_hub_chunks);
        g->chunk_part.alloc(ctx, g->n_hub_chunks);
        g->part_hub.alloc(ctx, g->n_hub_parts);
        CD_LAUNCH(ctx, "bins", k_hub_chunks, grid_for(nh, 1, ctx->num_sms * 4), 128, 0, nh,
                  static_cast<const int32_t *>(g->hubs), static_cast<const int64_t *>(g->off.p),
                  static_cast<const int64_t *>(chunk_pre.p), static_cast<const int64_t *>(g->hub_pbase.p),
                  g->hub_pbits.p, g->chunk_hub.p, g->chunk_part.p, g->part_hub.p);
        g->hub_entries = g->n_hub_chunks * HUB_CHUNK;  // >= sum of hub degrees
        g->hp_cnt.alloc(ctx, g->n_hub_parts);
        g->hp_cur.alloc(ctx, g->n_hub_parts);
        g->hp_start.alloc(ctx, g->n_hub_parts + 1);
        g->hp_key.alloc(ctx, g->hub_entries);
        g->hp_val.alloc(ctx, g->hub_entries);
        g->st_key.alloc(ctx, g->hub_entries);
        g->st_val.alloc(ctx, g->hub_entries);
        g->chunk_np.alloc(ctx, g->n_hub_chunks);
        g->hp_best_val.alloc(ctx, g->n_hub_parts);
        g->hp_second.alloc(ctx, g->n_hub_parts);
        g->hp_best_key.alloc(ctx, g->n_hub_parts);
        g->hp_scan.alloc(ctx, 2 * scan_scratch_elems(g->n_hub_parts));
        g->hp_flag.alloc(ctx, 1);
        g->hp_flag.zero();
        g->hub_aux.alloc(ctx, nh);
        g->hub_aux.zero();
    }
    g->binned = true;
}

// Drop the work decomposition (tier lists, hub scratch: ~12 B per hub entry)
// of a graph whose move phases are over for now; graph_ensure_bins rebuilds it
// on the next use (PLMR refinement).  Used for graphs near the device's
// capacity, where the next level's contraction needs the room.
void graph_release_bins(cd_graph *g) {
    g->binned = false;
    g->tier.release();
    g->tlist.release();
    g->hubs = nullptr;
    g->n_hubs = g->n_hub_chunks = g->n_hub_parts = g->hub_entries = 0;
    for (auto *b : {&g->chunk_hub, &g->chunk_part, &g->hub_pbits, &g->part_hub, &g->hp_cnt, &g->hp_cur,
                    &g->hp_best_key, &g->hp_flag})
        b->release();
    for (auto *b : {&g->hub_pbase, &g->hp_start, &g->hp_scan})
        b->release();
    for (auto *b : {&g->hp_val, &g->hp_best_val, &g->hp_second, &g->hub_aux})
        b->release();
    g->hp_key.release();
    g->st_key.release();
    g->st_val.release();
    g->chunk_np.release();
}

HubScratch *hub_scratch_for(cd_ctx *ctx, const cd_graph *g) {
    if (!ctx->private_hubs || !g->n_hubs)
        return nullptr;
    auto &slot = ctx->hub_scratch[g];
    if (!slot) {
        auto *h = new HubScratch();
        slot = std::shared_ptr<void>(h, [](void *p) { delete static_cast<HubScratch *>(p); });
        h->hp_cnt.alloc(ctx, g->n_hub_parts);
        h->hp_cur.alloc(ctx, g->n_hub_parts);
        h->hp_start.alloc(ctx, g->n_hub_parts + 1);
        h->hp_key.alloc(ctx, g->hub_entries);
        h->hp_val.alloc(ctx, g->hub_entries);
        h->st_key.alloc(ctx, g->hub_entries);
        h->st_val.alloc(ctx, g->hub_entries);
        h->chunk_np.alloc(ctx, g->n_hub_chunks);
        h->hp_best_val.alloc(ctx, g->n_hub_parts);
        h->hp_second.alloc(ctx, g->n_hub_parts);
        h->hp_best_key.alloc(ctx, g->n_hub_parts);
        h->hp_scan.alloc(ctx, 2 * scan_scratch_elems(g->n_hub_parts));
        h->hp_flag.alloc(ctx, 1);
        h->hp_flag.zero();
        h->hub_aux.alloc(ctx, g->n_hubs);
        h->hub_aux.zero();
    }
    return static_cast<HubScratch *>(slot.get());
}

cd_ctx *ctx_child(const cd_ctx *parent) {
    auto *c = new cd_ctx();
    try {
        c->device = parent->device;
        c->pool = parent->pool;
        c->num_sms = parent->num_sms;
        c->smem_optin = parent->smem_optin;
        c->use_graphs = parent->use_graphs;
        c->private_hubs = true;
        CD_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CD_CUDA(cudaMalloc(reinterpret_cast<void **>(&c->dstats), DSTATS * sizeof(unsigned long long)));
        CD_CUDA(cudaMemsetAsync(c->dstats, 0, DSTATS * sizeof(unsigned long long), c->stream));
    } catch (...) {
        if (c->stream)
            cudaStreamDestroy(c->stream);
        delete c;
        throw;
    }
    return c;
}

void ctx_child_destroy(cd_ctx *parent, cd_ctx *child) {
    if (!child)
        return;
    cudaStreamSynchronize(child->stream);
    child->hub_scratch.clear();  // frees on the child stream
    cudaStreamSynchronize(child->stream);
    parent->launches += child->launches;
    for (auto e : child->free_events)
        cudaEventDestroy(e);
    for (auto &st : child->side)
        if (st)
            cudaStreamDestroy(st);
    if (child->fork_ev)
        cudaEventDestroy(child->fork_ev);
    for (auto e : child->join_ev)
        if (e)
            cudaEventDestroy(e);
    if (child->dstats)
        cudaFree(child->dstats);
    cudaStreamDestroy(child->stream);
    delete child;
}

}  // namespace cdk
