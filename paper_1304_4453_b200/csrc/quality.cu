// quality.cu -- modularity / coverage (H/quality.hpp:21-51) and community
// volumes (H/louvain.hpp:27-31).  Every accumulator is fp64: Q is a
// difference of O(1) terms that cancel to ~1e-5 on R-MAT (SURVEY.md finding 11).
#include "comm.cuh"
#include "graph.cuh"

namespace cdk {

constexpr int MOD_ITEMS = 8;

// intra-community weight over for_edges (u <= v, loops once): entry-parallel,
// each thread owns MOD_ITEMS consecutive CSR entries and locates its row by
// binary search, so hubs are split evenly across threads.
__global__ void __launch_bounds__(256) k_mod_intra(int64_t n, int64_t D, const int64_t *off, const int32_t *col,
                                                   const float *w, const int32_t *z, double *acc) {
    __shared__ double red[8];
    double sum = 0.0;
    for (int64_t e0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * MOD_ITEMS; e0 < D;
         e0 += static_cast<int64_t>(gridDim.x) * blockDim.x * MOD_ITEMS) {
        int64_t lo = 0, hi = n - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (off[mid] <= e0)
                lo = mid;
            else
                hi = mid - 1;
        }
        int64_t u = lo;
        int64_t next = off[u + 1];
        int32_t zu = z[u];
        const int64_t e1 = min(D, e0 + MOD_ITEMS);
        for (int64_t e = e0; e < e1; ++e) {
            if (e >= next) {
                int steps = 0;
                while (e >= next && steps < 4) {
                    ++u;
                    next = off[u + 1];
                    ++steps;
                }
                if (e >= next) {
                    int64_t a = u, b = n - 1;
                    while (a < b) {
                        const int64_t mid = (a + b + 1) >> 1;
                        if (off[mid] <= e)
                            a = mid;
                        else
                            b = mid - 1;
                    }
                    u = a;
                    next = off[u + 1];
                }
                zu = z[u];
            }
            const int32_t v = col[e];
            if (v >= u && z[v] == zu)
                sum += w ? static_cast<double>(w[e]) : 1.0;
        }
    }
    sum = warp_sum(sum);
    if (lane_id() == 0)
        red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
            t += red[q];
        if (t != 0.0)
            atomicAdd(acc, t);
    }
}

// vols[z[u]] += vol[u], warp-aggregated by label; flags labels outside [0, ub)
__global__ void __launch_bounds__(256) k_comm_vol(int64_t n, const int32_t *z, const double *vol, int64_t ub,
                                                  double *vols, int32_t *csize, int64_t *flag) {
    __shared__ double scratch[8][32];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < n;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u = base + threadIdx.x;
        bool valid = u < n;
        int32_t c = valid ? z[u] : 0;
        if (valid && (c < 0 || c >= ub)) {
            if (flag)
                flag[0] = 1;
            valid = false;
        }
        const double vu = valid ? vol[u] : 0.0;
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t peers = __match_any_sync(0xffffffffu, c) & vmask;
        const bool leader = valid && (__ffs(peers) - 1) == lane;
        scratch[wid][lane] = vu;
        __syncwarp();
        if (leader) {
            double s = 0.0;
            for (uint32_t m = peers; m; m &= m - 1)
                s += scratch[wid][__ffs(m) - 1];
            atomicAdd(&vols[c], s);
            if (csize)
                atomicAdd(&csize[c], __popc(peers));
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_sum_sq(int64_t ub, const double *vols, double *acc) {
    __shared__ double red[8];
    double s = 0.0;
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < ub;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s += vols[c] * vols[c];
    s = warp_sum(s);
    if (lane_id() == 0)
        red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
            t += red[q];
        atomicAdd(acc, t);
    }
}

static void comm_vol_launch(cd_ctx *ctx, const cd_graph *g, const int32_t *z, double *vols, int32_t *csize,
                            int64_t ub, int64_t *flag) {
    CD_CUDA(cudaMemsetAsync(vols, 0, ub * sizeof(double), ctx->stream));
    if (csize)
        CD_CUDA(cudaMemsetAsync(csize, 0, ub * sizeof(int32_t), ctx->stream));
    if (g->n > 0)
        CD_LAUNCH(ctx, "comm_volumes", k_comm_vol, grid_for(g->n, 256, ctx->num_sms * 8), 256, 0, g->n, z,
                  static_cast<const double *>(g->vol.p), ub, vols, csize, flag);
}

void community_volumes_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, double *vols, int64_t ub) {
    DBuf<int64_t> flag(ctx, 1);
    flag.zero();
    comm_vol_launch(ctx, g, z, vols, nullptr, ub, flag.p);
    int64_t h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h)
        fail(CD_ERANGE, "community id outside [0, upper_bound)");
}

void community_volumes_sizes_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, double *vols, int32_t *csize,
                                 int64_t ub) {
    comm_vol_launch(ctx, g, z, vols, csize, ub, nullptr);
}

void modularity_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double gamma, double *q,
                    double *cov) {
    DBuf<double> vols(ctx, std::max<int64_t>(ub, 1));
    DBuf<double> acc(ctx, 2);
    DBuf<int64_t> flag(ctx, 1);
    acc.zero();
    flag.zero();
    comm_vol_launch(ctx, g, z, vols.p, nullptr, ub, flag.p);
    if (g->D > 0)
        CD_LAUNCH(ctx, "modularity", k_mod_intra, grid_for(g->D, 256 * MOD_ITEMS, ctx->num_sms * 8), 256, 0, g->n,
                  g->D, static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p),
                  static_cast<const float *>(g->weighted ? g->w.p : nullptr), z, acc.p);
    // a row shard holds only its rows' intra-community entries
    if (g->rows_local && world_size(ctx) > 1)
        ctx->comm->allreduce_sum_f64(ctx, acc.p, 1);
    CD_LAUNCH(ctx, "modularity", k_sum_sq, grid_for(ub, 256, ctx->num_sms * 8), 256, 0, ub,
              static_cast<const double *>(vols.p), acc.p + 1);
    double h[2];
    int64_t hf = 0;
    CD_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&hf, flag.p, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hf)
        fail(CD_ERANGE, "community id outside [0, upper_bound)");
    const double total = g->total;
    if (cov)
        *cov = total == 0.0 ? 0.0 : h[0] / total;
    if (total == 0.0) {
        if (q)
            fail(CD_EDOMAIN, "modularity undefined for graph with zero total edge weight");
        return;
    }
    if (q)
        *q = h[0] / total - gamma * h[1] / (4.0 * total * total);
}

// graph_rand_index (H/quality.hpp:56-69): edges {u <= v} on which the two
// partitions agree (both join or both separate the endpoints; loops agree)
__global__ void k_rand_agree(int64_t n, const int64_t *off, const int32_t *col, const int32_t *a, const int32_t *b,
                             unsigned long long *agree) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long c = 0;
    for (int64_t u = gw; u < n; u += nw) {
        const int32_t au = a[u], bu = b[u];
        for (int64_t e = off[u] + lane; e < off[u + 1]; e += 32) {
            const int32_t v = col[e];
            if (v >= u)
                c += ((au == a[v]) == (bu == b[v])) ? 1 : 0;
        }
    }
    c = warp_sum(c);
    if (lane == 0 && c)
        atomicAdd(agree, c);
}

double rand_index_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *a, const int32_t *b) {
    if (g->m == 0)
        fail(CD_EDOMAIN, "graph-structural Rand index undefined for edgeless graph");
    DBuf<unsigned long long> agree(ctx, 1);
    agree.zero();
    if (g->n)
        CD_LAUNCH(ctx, "quality", k_rand_agree, grid_for(g->n, 8, ctx->num_sms * 16), 256, 0, g->n,
                  static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p), a, b, agree.p);
    if (g->rows_local && world_size(ctx) > 1)
        ctx->comm->allreduce_sum_i64(ctx, reinterpret_cast<int64_t *>(agree.p), 1);
    unsigned long long h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, agree.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return static_cast<double>(h) / static_cast<double>(g->m);
}

}  // namespace cdk
