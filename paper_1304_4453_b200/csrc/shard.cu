// shard.cu -- 1D row sharding of a graph across ranks.
//
// Rank r of G owns nodes [b_r, b_{r+1}), the ranges splitting the CSR
// entries evenly (comm.cuh shard_bounds).  A row shard keeps the owned rows
// (global column ids) and the replicated per-node state (vol, loop); labels
// and community volumes are replicated by the drivers.  Coarsening a row
// shard gives each rank a partial coarse graph over the same coarse ids; the
// partials are allgathered and summed by the row engine into the replicated
// coarse graph (its rows sorted and duplicate-summed exactly as coarsen does
// on one device, H/louvain.hpp:154-220).
#include "comm.cuh"
#include "rows.cuh"

namespace cdk {

__global__ void k_shard_off(int64_t n, const int64_t *off, int64_t lo, int64_t hi, int64_t *out) {
    const int64_t e0 = off[lo], e1 = off[hi];
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u <= n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[u] = u <= lo ? 0 : (u >= hi ? e1 - e0 : off[u] - e0);
}

cd_graph *graph_shard_dev(cd_ctx *ctx, const cd_graph *full) {
    if (full->rows_local)
        fail(CD_EINVAL, "graph is already a row shard");
    const int G = world_size(ctx), r = world_rank(ctx);
    const int64_t n = full->n;
    std::vector<int64_t> bounds(G + 1);
    shard_bounds_dev(ctx, n, full->off.p, G, bounds.data());
    const int64_t lo = bounds[r], hi = bounds[r + 1];
    int64_t e[2] = {0, 0};
    CD_CUDA(cudaMemcpyAsync(&e[0], full->off.p + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&e[1], full->off.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    auto *sh = new cd_graph();
    try {
        sh->ctx = ctx;
        sh->n = n;
        sh->D = e[1] - e[0];
        sh->m = full->m;
        sh->total = full->total;
        sh->weighted = full->weighted;
        sh->int_weights = full->int_weights;
        sh->max_vol = full->max_vol;
        sh->max_degree = full->max_degree;
        sh->isolated = full->isolated;
        sh->rows_local = true;
        sh->shard_rank = r;
        sh->shard_size = G;
        sh->own_lo = lo;
        sh->own_hi = hi;
        sh->D_global = full->D;
        sh->off.alloc(ctx, n + 1);
        CD_LAUNCH(ctx, "shard", k_shard_off, grid_for(n + 1, 256, ctx->num_sms * 8), 256, 0, n,
                  static_cast<const int64_t *>(full->off.p), lo, hi, sh->off.p);
        sh->col.alloc(ctx, std::max<int64_t>(sh->D, 1));
        if (sh->D)
            CD_CUDA(cudaMemcpyAsync(sh->col.p, full->col.p + e[0], sh->D * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        if (full->weighted) {
            sh->w.alloc(ctx, std::max<int64_t>(sh->D, 1));
            if (sh->D)
                CD_CUDA(cudaMemcpyAsync(sh->w.p, full->w.p + e[0], sh->D * sizeof(float), cudaMemcpyDeviceToDevice,
                                        ctx->stream));
        }
        sh->vol.alloc(ctx, std::max<int64_t>(n, 1));
        sh->loop.alloc(ctx, std::max<int64_t>(n, 1));
        if (n) {
            CD_CUDA(cudaMemcpyAsync(sh->vol.p, full->vol.p, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            CD_CUDA(cudaMemcpyAsync(sh->loop.p, full->loop.p, n * sizeof(double), cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        }
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        delete sh;
        throw;
    }
    return sh;
}

cd_graph *graph_from_rows_dev(cd_ctx *ctx, int64_t n, const int64_t *off, int64_t lo, int64_t hi,
                              const int32_t *col, const float *w) {
    const int G = world_size(ctx), r = world_rank(ctx);
    DBuf<int64_t> full(ctx, n + 1);
    CD_CUDA(cudaMemcpyAsync(full.p, off, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, ctx->stream));
    std::vector<int64_t> bounds(G + 1);
    shard_bounds_dev(ctx, n, full.p, G, bounds.data());
    if (bounds[r] != lo || bounds[r + 1] != hi)
        fail(CD_EINVAL, "row range [" + std::to_string(lo) + ", " + std::to_string(hi) + ") is not this rank's " +
                            "shard range [" + std::to_string(bounds[r]) + ", " + std::to_string(bounds[r + 1]) + ")");
    int64_t e[3] = {0, 0, 0};
    CD_CUDA(cudaMemcpyAsync(&e[0], full.p + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&e[1], full.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&e[2], full.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t D = e[1] - e[0];
    if (D < 0 || e[0] < 0 || e[2] < e[1])
        fail(CD_EINPUT, "malformed CSR offsets");
    if (D && !col)
        fail(CD_EINVAL, "null column array");
    auto *g = new cd_graph();
    try {
        g->ctx = ctx;
        g->n = n;
        g->D = D;
        g->weighted = w != nullptr;
        g->off.alloc(ctx, n + 1);
        CD_LAUNCH(ctx, "shard", k_shard_off, grid_for(n + 1, 256, ctx->num_sms * 8), 256, 0, n,
                  static_cast<const int64_t *>(full.p), lo, hi, g->off.p);
        full.release();
        g->col.alloc(ctx, std::max<int64_t>(D, 1));
        if (w)
            g->w.alloc(ctx, std::max<int64_t>(D, 1));
        if (D >= UPLOAD_MIN_ENTRIES && !is_device_ptr(col)) {
            // host rows: chunked copies, each chunk checked while the next one copies
            // (as cd_graph_from_csr; the shard's node state needs the finalize below)
            graph_upload_validate(ctx, n, D, g->off.p, g->col.p, col, w ? g->w.p : nullptr, w);
        } else {
            if (D)
                CD_CUDA(cudaMemcpyAsync(g->col.p, col, D * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
            if (w && D)
                CD_CUDA(cudaMemcpyAsync(g->w.p, w, D * sizeof(float), cudaMemcpyDefault, ctx->stream));
            graph_validate_csr(ctx, n, g->off.p, g->col.p, g->weighted ? g->w.p : nullptr, D);
        }
        graph_finalize(ctx, g);  // over the owned rows: each edge counted once, by its smaller endpoint's owner
        if (G > 1)
            shard_globalize(ctx, g, lo, hi);
    } catch (...) {
        delete g;
        throw;
    }
    return g;
}

// transposed block: for every node v, the owned u with (u, v) an entry
__global__ void k_tcount(int64_t lo, int64_t hi, const int64_t *off, const int32_t *col, int32_t *cnt) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = lo + gw; u < hi; u += nw)
        for (int64_t e = off[u] + lane_id(); e < off[u + 1]; e += 32)
            atomicAdd(&cnt[col[e]], 1);
}

__global__ void k_tscatter(int64_t lo, int64_t hi, const int64_t *off, const int32_t *col, int64_t *cursor,
                           int32_t *tcol) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = lo + gw; u < hi; u += nw)
        for (int64_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) {
            const int64_t p = static_cast<int64_t>(
                atomicAdd(reinterpret_cast<unsigned long long *>(&cursor[col[e]]), 1ULL));
            tcol[p] = static_cast<int32_t>(u);
        }
}

struct Cnt32Gen {
    const int32_t *c;
    __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

void graph_ensure_transpose(cd_ctx *ctx, cd_graph *g) {
    if (!g->rows_local || g->toff.p)
        return;
    const int64_t n = g->n;
    DBuf<int32_t> cnt(ctx, std::max<int64_t>(n, 1));
    cnt.zero();
    const int grid = grid_for(std::max<int64_t>(g->own_hi - g->own_lo, 1), 8, ctx->num_sms * 8);
    CD_LAUNCH(ctx, "shard", k_tcount, grid, 256, 0, g->own_lo, g->own_hi, static_cast<const int64_t *>(g->off.p),
              static_cast<const int32_t *>(g->col.p), cnt.p);
    g->toff.alloc(ctx, n + 1);
    exclusive_scan<int64_t>(ctx, n, Cnt32Gen{cnt.p}, g->toff.p, g->toff.p + n);
    DBuf<int64_t> cursor(ctx, n + 1);
    CD_CUDA(cudaMemcpyAsync(cursor.p, g->toff.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    g->tcol.alloc(ctx, std::max<int64_t>(g->D, 1));
    CD_LAUNCH(ctx, "shard", k_tscatter, grid, 256, 0, g->own_lo, g->own_hi, static_cast<const int64_t *>(g->off.p),
              static_cast<const int32_t *>(g->col.p), cursor.p, g->tcol.p);
}

void owned_range(cd_ctx *ctx, const cd_graph *g, int64_t &lo, int64_t &hi) {
    const int G = world_size(ctx);
    if (G == 1) {
        lo = 0;
        hi = g->n;
        return;
    }
    if (g->rows_local) {
        if (g->shard_size != G || g->shard_rank != world_rank(ctx))
            fail(CD_EINVAL, "row shard was built for another communicator");
        lo = g->own_lo;
        hi = g->own_hi;
        return;
    }
    std::vector<int64_t> b(G + 1);
    shard_bounds_dev(ctx, g->n, g->off.p, G, b.data());
    lo = b[world_rank(ctx)];
    hi = b[world_rank(ctx) + 1];
}

// ---------------------------------------------------------------------------
// coarsening a row shard
// ---------------------------------------------------------------------------
// coarse row c = concatenation over ranks of the partial rows c
struct SrcStack {
    const int64_t *roff;  // [G][nc+1]
    const int32_t *rcol;  // [G][cstride]
    const float *rw;      // [G][cstride]
    const int64_t *fpre;  // [nc+1] prefix of the merged row lengths
    int G;
    int64_t ostride, cstride;
    struct Cursor {};
    __device__ Cursor init(int64_t, int64_t) const { return {}; }
    __device__ void load(int64_t c, int64_t f0, int64_t fend, Cursor &, int32_t &k, double &wt, bool &valid) const {
        const int64_t f = f0 + lane_id();
        valid = f < fend;
        k = 0;
        wt = 1.0;
        if (!valid)
            return;
        int64_t rel = f - fpre[c];
        for (int r = 0; r < G; ++r) {
            const int64_t a = roff[r * ostride + c], len = roff[r * ostride + c + 1] - a;
            if (rel < len) {
                const int64_t e = r * cstride + a + rel;
                k = rcol[e];
                wt = static_cast<double>(rw[e]);
                return;
            }
            rel -= len;
        }
    }
};

__global__ void k_stack_fpre(int64_t nc, const int64_t *roff, int G, int64_t ostride, int64_t *fpre) {
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c <= nc;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t s = 0;
        for (int r = 0; r < G; ++r)
            s += roff[r * ostride + c];
        fpre[c] = s;
    }
}

__global__ void k_row_len(int64_t n, const int64_t *off, int64_t *len) {
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
        len[c] = off[c + 1] - off[c];
}

struct Len64Gen {
    const int64_t *a;
    __device__ int64_t operator()(int64_t i) const { return a[i]; }
};

// Coarse graphs too large to replicate (C5's level 1 keeps ~98 % of the
// entries) stay row-sharded: coarse rows are owned by degree-balanced ranges
// of the summed partial row lengths, every rank sends each owner the slab of
// its partial in the owner's range (one all-to-all for the row lengths, two
// for the entries), and the owner merges its G slabs with the row engine.
// The result is a row shard exactly like cd_graph_shard's (global node state
// summed over the ranks by shard_globalize).
static int64_t shard_coarse_min_entries() { return env_i64("CD_SHARD_COARSE_MIN_ENTRIES", int64_t(1) << 30); }

static cd_graph *coarse_shard_from_partials(cd_ctx *ctx, cd_graph *part, int64_t nc, bool sorted) {
    Comm *comm = ctx->comm;
    const int G = world_size(ctx), me = world_rank(ctx);
    const int grid = grid_for(std::max<int64_t>(nc, 1), 256, ctx->num_sms * 8);
    // ownership of coarse rows
    std::vector<int64_t> cb(G + 1);
    {
        DBuf<int64_t> len(ctx, std::max<int64_t>(nc, 1)), pre(ctx, nc + 1);
        if (nc)
            CD_LAUNCH(ctx, "coarsen.prep", k_row_len, grid, 256, 0, nc, static_cast<const int64_t *>(part->off.p), len.p);
        comm->allreduce_sum_i64(ctx, len.p, static_cast<size_t>(std::max<int64_t>(nc, 1)));
        exclusive_scan<int64_t>(ctx, nc, Len64Gen{len.p}, pre.p, pre.p + nc);
        shard_bounds_dev(ctx, nc, pre.p, G, cb.data());
    }
    const int64_t clo = cb[me], chi = cb[me + 1], nloc = chi - clo;
    // my partial's slab offsets at every owner boundary
    std::vector<int64_t> ob(G + 1);
    for (int d = 0; d <= G; ++d)
        CD_CUDA(cudaMemcpyAsync(&ob[d], part->off.p + cb[d], sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    // G x G entry counts: row s = what rank s sends to each owner
    std::vector<int64_t> mat(size_t(G) * G);
    {
        DBuf<int64_t> mine(ctx, G), all(ctx, size_t(G) * G);
        std::vector<int64_t> cnt(G);
        for (int d = 0; d < G; ++d)
            cnt[d] = ob[d + 1] - ob[d];
        CD_CUDA(cudaMemcpyAsync(mine.p, cnt.data(), G * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        comm->allgather(ctx, mine.p, all.p, G * sizeof(int64_t));
        CD_CUDA(cudaMemcpyAsync(mat.data(), all.p, mat.size() * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    int64_t cstride = 1, floc = 0;
    for (int s = 0; s < G; ++s) {
        cstride = std::max(cstride, mat[size_t(s) * G + me]);
        floc += mat[size_t(s) * G + me];
    }
    const int64_t ostride = nloc + 1;
    // row lengths of every source's slab for my rows; entries padded to cstride
    DBuf<int64_t> slen(ctx, std::max<int64_t>(nc, 1)), rlen(ctx, size_t(G) * std::max<int64_t>(nloc, 1));
    if (nc)
        CD_LAUNCH(ctx, "coarsen.prep", k_row_len, grid, 256, 0, nc, static_cast<const int64_t *>(part->off.p), slen.p);
    DBuf<int32_t> rcol(ctx, size_t(G) * cstride);
    DBuf<float> rw(ctx, size_t(G) * cstride);
    {
        std::vector<size_t> sd(G), sc(G), rd(G), rc(G);
        for (int d = 0; d < G; ++d) {
            sd[d] = size_t(cb[d]) * sizeof(int64_t);
            sc[d] = size_t(cb[d + 1] - cb[d]) * sizeof(int64_t);
            rd[d] = size_t(d) * std::max<int64_t>(nloc, 1) * sizeof(int64_t);
            rc[d] = size_t(nloc) * sizeof(int64_t);
        }
        comm->alltoallv(ctx, slen.p, sd.data(), sc.data(), rlen.p, rd.data(), rc.data());
        for (int d = 0; d < G; ++d) {
            sd[d] = size_t(ob[d]) * sizeof(int32_t);
            sc[d] = size_t(ob[d + 1] - ob[d]) * sizeof(int32_t);
            rd[d] = size_t(d) * cstride * sizeof(int32_t);
            rc[d] = size_t(mat[size_t(d) * G + me]) * sizeof(int32_t);
        }
        comm->alltoallv(ctx, part->col.p, sd.data(), sc.data(), rcol.p, rd.data(), rc.data());
        comm->alltoallv(ctx, part->w.p, sd.data(), sc.data(), rw.p, rd.data(), rc.data());  // float = int32 size
    }
    slen.release();
    // per-source exclusive prefixes -> SrcStack layout [G][nloc+1]
    DBuf<int64_t> roff(ctx, size_t(G) * ostride), fpre(ctx, ostride);
    for (int s = 0; s < G; ++s)
        exclusive_scan<int64_t>(ctx, nloc, Len64Gen{rlen.p + size_t(s) * std::max<int64_t>(nloc, 1)},
                                roff.p + size_t(s) * ostride, roff.p + size_t(s) * ostride + nloc);
    CD_LAUNCH(ctx, "coarsen.prep", k_stack_fpre, grid_for(ostride, 256, ctx->num_sms * 8), 256, 0, nloc,
              static_cast<const int64_t *>(roff.p), G, ostride, fpre.p);
    auto *cg = new cd_graph();
    try {
        cg->ctx = ctx;
        cg->n = nc;
        cg->weighted = true;
        DBuf<int64_t> loff;
        bool want_w = true;
        SrcStack src{roff.p, rcol.p, rw.p, fpre.p, G, ostride, cstride};
        const int64_t dloc = run_row_engine(ctx, src, nloc, fpre.p, floc, std::max<int64_t>(nc, 1), DUP_SUM, want_w,
                                            loff, cg->col, cg->w, nullptr, "coarsen", sorted);
        cg->D = dloc;
        cg->off.alloc(ctx, nc + 1);
        if (clo > 0)
            CD_LAUNCH(ctx, "coarsen.prep", k_fill_i64, grid_for(clo, 256, ctx->num_sms * 8), 256, 0, clo, int64_t(0),
                      cg->off.p);
        if (nloc > 0)
            CD_LAUNCH(ctx, "coarsen.prep", k_rebase, grid_for(nloc, 256, ctx->num_sms * 8), 256, 0, nloc,
                      static_cast<const int64_t *>(loff.p), int64_t(0), int64_t(0), cg->off.p + clo);
        CD_LAUNCH(ctx, "coarsen.prep", k_fill_i64, grid_for(nc + 1 - chi, 256, ctx->num_sms * 8), 256, 0, nc + 1 - chi,
                  dloc, cg->off.p + chi);
        graph_finalize(ctx, cg);
        shard_globalize(ctx, cg, clo, chi);
    } catch (...) {
        delete cg;
        throw;
    }
    return cg;
}

cd_graph *coarsen_sharded_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc, bool sorted) {
    Comm *comm = ctx->comm;
    const int G = world_size(ctx);
    if (!g->rows_local || G == 1)
        return coarsen_dev(ctx, g, z, nc, sorted);
    cd_graph *part = coarsen_dev(ctx, g, z, nc, false);  // this rank's rows only (merged below)
    cd_graph *cg = nullptr;
    try {
        DBuf<int64_t> dcount(ctx, 1), rcount(ctx, G);
        CD_CUDA(cudaMemcpyAsync(dcount.p, &part->D, sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
        comm->allgather(ctx, dcount.p, rcount.p, sizeof(int64_t));
        std::vector<int64_t> hc(G);
        CD_CUDA(cudaMemcpyAsync(hc.data(), rcount.p, G * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        int64_t maxd = 1, ftotal = 0;
        for (int r = 0; r < G; ++r) {
            maxd = std::max(maxd, hc[r]);
            ftotal += hc[r];
        }
        if (ftotal >= shard_coarse_min_entries()) {
            cg = coarse_shard_from_partials(ctx, part, nc, sorted);
            delete part;
            return cg;
        }
        const int64_t ostride = nc + 1;
        DBuf<int64_t> roff(ctx, G * ostride);
        comm->allgather(ctx, part->off.p, roff.p, ostride * sizeof(int64_t));
        // padded send blocks (the allgather reads maxd entries from every rank)
        DBuf<int32_t> scol(ctx, maxd), rcol(ctx, G * maxd);
        DBuf<float> sw(ctx, maxd), rw(ctx, G * maxd);
        if (part->D) {
            CD_CUDA(cudaMemcpyAsync(scol.p, part->col.p, part->D * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                    ctx->stream));
            CD_CUDA(cudaMemcpyAsync(sw.p, part->w.p, part->D * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
        }
        delete part;
        part = nullptr;
        comm->allgather(ctx, scol.p, rcol.p, maxd * sizeof(int32_t));
        comm->allgather(ctx, sw.p, rw.p, maxd * sizeof(float));
        DBuf<int64_t> fpre(ctx, nc + 1);
        CD_LAUNCH(ctx, "coarsen.prep", k_stack_fpre, grid_for(nc + 1, 256, ctx->num_sms * 8), 256, 0, nc,
                  static_cast<const int64_t *>(roff.p), G, ostride, fpre.p);
        cg = new cd_graph();
        cg->ctx = ctx;
        cg->n = nc;
        cg->weighted = true;
        SrcStack src{roff.p, rcol.p, rw.p, fpre.p, G, ostride, maxd};
        bool want_w = true;
        cg->D = run_row_engine(ctx, src, nc, fpre.p, ftotal, std::max<int64_t>(nc, 1), DUP_SUM, want_w, cg->off,
                               cg->col, cg->w, nullptr, "coarsen", sorted);
        graph_finalize(ctx, cg);
    } catch (...) {
        delete part;
        delete cg;
        throw;
    }
    return cg;
}

}  // namespace cdk
