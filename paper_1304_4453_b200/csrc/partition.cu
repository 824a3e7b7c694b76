// partition.cu -- Partition::compacted (H/partition.hpp:39-53, first
// appearance order), prolong (H/louvain.hpp:223-233) and combine_hashed
// (H/ensemble.hpp:86-107) on the device.
#include "graph.cuh"
#include "scan.cuh"

namespace cdk {

__global__ void k_iota(int32_t *z, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        z[i] = static_cast<int32_t>(i);
}

void iota_dev(cd_ctx *ctx, int32_t *z, int64_t n) {
    if (n > 0)
        CD_LAUNCH(ctx, "iota", k_iota, grid_for(n, 256, ctx->num_sms * 8), 256, 0, z, n);
}

__global__ void k_max_label(int64_t n, const int32_t *z, int *mx, int *neg) {
    int m = 0;
    bool bad = false;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        m = max(m, z[i]);
        bad |= z[i] < 0;
    }
    for (int o = 16; o > 0; o >>= 1)
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane_id() == 0)
        atomicMax(mx, m);
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0)
        *neg = 1;
}

int64_t max_label_dev(cd_ctx *ctx, int64_t n, const int32_t *z) {
    DBuf<int> r(ctx, 2);
    r.zero();
    if (n > 0)
        CD_LAUNCH(ctx, "max_label", k_max_label, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n, z, r.p, r.p + 1);
    int h[2];
    CD_CUDA(cudaMemcpyAsync(h, r.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h[1])
        return -1;
    return static_cast<int64_t>(h[0]) + 1;
}

// ---- first-appearance compaction ------------------------------------------
// A flooded label (R-MAT PLP: half the nodes share one) would serialise its
// members on one address: only the warp's smallest member of each label
// competes, and only while the stored member is larger.
__global__ void k_first_member(int64_t n, const int32_t *z, int32_t *first) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x; b < n; b += stride) {
        const int64_t u = b + threadIdx.x;
        const bool in = u < n;
        const int32_t k = in ? z[u] : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, k);
        if (in && (threadIdx.x & 31) == __ffs(peers) - 1 && __ldcg(&first[k]) > static_cast<int32_t>(u))
            atomicMin(&first[k], static_cast<int32_t>(u));
    }
}

struct FirstFlag {
    const int32_t *z;
    const int32_t *first;
    __device__ int32_t operator()(int64_t u) const { return first[z[u]] == static_cast<int32_t>(u) ? 1 : 0; }
};

__global__ void k_compact_out(int64_t n, const int32_t *z, const int32_t *first, const int32_t *rank,
                              int32_t *out) {
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[u] = rank[first[z[u]]];
}

// out[u] = rank of z[u]'s first member among all first members.  out may
// alias z only through the caller's copy (it is written last).  Returns k.
int64_t compact_dev(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t ub, int32_t *out) {
    if (n == 0)
        return 0;
    DBuf<int32_t> first(ctx, ub);
    first.fill_bytes(0x7f);
    const int grid = grid_for(n, 256, ctx->num_sms * 8);
    CD_LAUNCH(ctx, "compact", k_first_member, grid, 256, 0, n, z, first.p);
    DBuf<int32_t> rank(ctx, n + 1);
    exclusive_scan<int32_t>(ctx, n, FirstFlag{z, first.p}, rank.p, rank.p + n);
    int32_t k = 0;
    CD_CUDA(cudaMemcpyAsync(&k, rank.p + n, sizeof(k), cudaMemcpyDeviceToHost, ctx->stream));
    CD_LAUNCH(ctx, "compact", k_compact_out, grid, 256, 0, n, z, static_cast<const int32_t *>(first.p),
              static_cast<const int32_t *>(rank.p), out);
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return k;
}

// ---- prolongation ------------------------------------------------------------
__global__ void k_prolong(int64_t nc, const int32_t *zc, int64_t n, const int32_t *pi, int32_t *out, int *flag) {
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p = pi[v];
        if (p < 0 || p >= nc) {
            *flag = 1;
            continue;
        }
        out[v] = zc[p];
    }
}

void prolong_dev(cd_ctx *ctx, int64_t nc, const int32_t *zc, int64_t n, const int32_t *pi, int32_t *out) {
    if (n == 0)
        return;
    DBuf<int> flag(ctx, 1);
    flag.zero();
    CD_LAUNCH(ctx, "prolong", k_prolong, grid_for(n, 256, ctx->num_sms * 8), 256, 0, nc, zc, n, pi, out, flag.p);
    int h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h)
        fail(CD_ERANGE, "prolong: contraction map entry out of range");
}

// ---- combine_hashed -----------------------------------------------------------
constexpr unsigned long long HEMPTY = ~0ULL;

__device__ __forceinline__ unsigned long long djb2_labels(const int32_t *const *sols, int64_t b, int64_t v) {
    unsigned long long h = 5381ULL;
    for (int64_t i = 0; i < b; ++i) {
        unsigned long long id = static_cast<unsigned long long>(static_cast<uint32_t>(sols[i][v]));
#pragma unroll
        for (int byte = 0; byte < 8; ++byte) {
            h = h * 33ULL + (id & 0xffULL);
            id >>= 8;
        }
    }
    return h == HEMPTY ? (HEMPTY ^ 1ULL) : h;
}

__device__ __forceinline__ uint64_t hslot64(unsigned long long h, uint64_t mask) {
    return (splitmix64(h)) & mask;
}

__global__ void k_combine_insert(int64_t b, int64_t n, const int32_t *const *sols, unsigned long long *hv,
                                 unsigned long long *tkeys, int32_t *tmin, uint64_t mask) {
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long h = djb2_labels(sols, b, v);
        hv[v] = h;
        uint64_t s = hslot64(h, mask);
        while (true) {
            const unsigned long long old = atomicCAS(&tkeys[s], HEMPTY, h);
            if (old == HEMPTY || old == h) {
                atomicMin(&tmin[s], static_cast<int32_t>(v));
                break;
            }
            s = (s + 1) & mask;
        }
    }
}

__global__ void k_combine_rep(int64_t n, const unsigned long long *hv, const unsigned long long *tkeys,
                              const int32_t *tmin, uint64_t mask, int32_t *rep) {
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long h = hv[v];
        uint64_t s = hslot64(h, mask);
        while (tkeys[s] != h)
            s = (s + 1) & mask;
        rep[v] = tmin[s];
    }
}

struct RepFlag {
    const int32_t *rep;
    __device__ int32_t operator()(int64_t v) const { return rep[v] == static_cast<int32_t>(v) ? 1 : 0; }
};

__global__ void k_combine_out(int64_t n, const int32_t *rep, const int32_t *rank, int32_t *out) {
    for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[v] = rank[rep[v]];
}

int64_t combine_hashed_dev(cd_ctx *ctx, int64_t b, int64_t n, const int32_t *const *sols_dev, int32_t *out) {
    if (n == 0)
        return 0;
    const uint64_t cap = next_pow2(static_cast<uint64_t>(2 * n));
    DBuf<unsigned long long> hv(ctx, n), tkeys(ctx, cap);
    DBuf<int32_t> tmin(ctx, cap), rep(ctx, n), rank(ctx, n + 1);
    tkeys.fill_bytes(0xff);
    tmin.fill_bytes(0x7f);
    const int grid = grid_for(n, 256, ctx->num_sms * 8);
    CD_LAUNCH(ctx, "combine", k_combine_insert, grid, 256, 0, b, n, sols_dev, hv.p, tkeys.p, tmin.p, cap - 1);
    CD_LAUNCH(ctx, "combine", k_combine_rep, grid, 256, 0, n, static_cast<const unsigned long long *>(hv.p),
              static_cast<const unsigned long long *>(tkeys.p), static_cast<const int32_t *>(tmin.p), cap - 1,
              rep.p);
    exclusive_scan<int32_t>(ctx, n, RepFlag{rep.p}, rank.p, rank.p + n);
    CD_LAUNCH(ctx, "combine", k_combine_out, grid, 256, 0, n, static_cast<const int32_t *>(rep.p),
              static_cast<const int32_t *>(rank.p), out);
    int32_t k = 0;
    CD_CUDA(cudaMemcpyAsync(&k, rank.p + n, sizeof(k), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return k;
}

}  // namespace cdk
