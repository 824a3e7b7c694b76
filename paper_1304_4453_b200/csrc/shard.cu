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
        CD_LAUNCH(ctx, "coarsen", k_stack_fpre, grid_for(nc + 1, 256, ctx->num_sms * 8), 256, 0, nc,
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
