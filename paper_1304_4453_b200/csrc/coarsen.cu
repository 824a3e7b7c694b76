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

cd_graph *coarsen_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc) {
    const int64_t n = g->n;
    const int grid = grid_for(n, 256, ctx->num_sms * 8);
    DBuf<int32_t> csz(ctx, std::max<int64_t>(nc, 1));
    csz.zero();
    if (n > 0)
        CD_LAUNCH(ctx, "coarsen", k_member_count, grid, 256, 0, n, z, csz.p);
    DBuf<int64_t> moff(ctx, nc + 1);
    exclusive_scan<int64_t>(ctx, nc, CszGen{csz.p}, moff.p, moff.p + nc);
    DBuf<int32_t> mem(ctx, std::max<int64_t>(n, 1));
    {
        DBuf<int64_t> cursor(ctx, nc + 1);
        CD_CUDA(cudaMemcpyAsync(cursor.p, moff.p, (nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (n > 0)
            CD_LAUNCH(ctx, "coarsen", k_member_scatter, grid, 256, 0, n, z, cursor.p, mem.p);
    }
    DBuf<int64_t> mpre(ctx, n + 1);
    exclusive_scan<int64_t>(ctx, n, MemDegGen{mem.p, g->off.p}, mpre.p, mpre.p + n);
    DBuf<int64_t> fpre(ctx, nc + 1);
    CD_LAUNCH(ctx, "coarsen", k_row_fpre, grid_for(nc + 1, 256, ctx->num_sms * 8), 256, 0, nc,
              static_cast<const int64_t *>(moff.p), static_cast<const int64_t *>(mpre.p), fpre.p);
    auto *cg = new cd_graph();
    cg->ctx = ctx;
    cg->n = nc;
    cg->weighted = true;
    try {
        SrcCoarsen src{moff.p, mem.p, mpre.p, g->off.p, g->col.p, g->weighted ? g->w.p : nullptr, z};
        bool want_w = true;
        cg->D = run_row_engine(ctx, src, nc, fpre.p, g->D, std::max<int64_t>(nc, 1), DUP_SUM, want_w, cg->off,
                               cg->col, cg->w, nullptr, "coarsen");
        graph_finalize(ctx, cg);
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
        CD_LAUNCH(ctx, "coarsen", k_member_count, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n, z, csz.p);
    CD_LAUNCH(ctx, "coarsen", k_check_used, grid_for(nc, 256, ctx->num_sms * 8), 256, 0, nc,
              static_cast<const int32_t *>(csz.p), flag.p);
    int h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return h == 0;
}

}  // namespace cdk
