// scan.cuh -- device-wide exclusive prefix sums (reduce-then-scan, 3 kernels)
// over a generator functor.  Used for CSR offsets, compaction ranks and
// member prefixes.  Tile = 256 threads x 8 items.
#pragma once

#include "common.cuh"

namespace cdk {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_tot, T &block_total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o)
            incl += t;
    }
    if (lane == 31)
        warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        T t = lane < nw ? warp_tot[lane] : T(0);
        T ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T u = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o)
                ti += u;
        }
        if (lane < nw)
            warp_tot[lane] = ti - t;  // exclusive warp offsets
        if (lane == nw - 1)
            warp_tot[32] = ti;
    }
    __syncthreads();
    block_total = warp_tot[32];
    T r = warp_tot[wid] + incl - v;
    __syncthreads();
    return r;
}

template <class T, class F>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(int64_t n, F f, T *partial) {
    __shared__ T wt[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i)
        if (base + i < n)
            s += f(base + i);
    T tot;
    block_exclusive_scan<T>(s, wt, tot);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = tot;
}

template <class T, class F>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(int64_t n, F f, const T *partial_scanned, T *out,
                                                            T *total) {
    __shared__ T wt[33];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    T vals[SCAN_ITEMS];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        vals[i] = (base + i < n) ? f(base + i) : T(0);
        s += vals[i];
    }
    T tot;
    T pre = block_exclusive_scan<T>(s, wt, tot) + (partial_scanned ? partial_scanned[blockIdx.x] : T(0));
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n)
            out[base + i] = pre;
        pre += vals[i];
    }
    if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1)
        *total = pre;
}

template <class T>
struct ArrayGen {
    const T *a;
    __device__ T operator()(int64_t i) const { return a[i]; }
};

// Two-level exclusive scan on an explicit stream with caller-provided
// Scratch elements exclusive_scan_on needs in EACH of `partial` and `pscan`
// for n items (the tile partials of every recursion level).
inline int64_t scan_scratch_elems(int64_t n) {
    int64_t s = 0, t = (n + SCAN_TILE - 1) / SCAN_TILE;
    while (t > 1) {
        s += t;
        t = (t + SCAN_TILE - 1) / SCAN_TILE;
    }
    return s + 1;
}

// scratch (no allocation: safe inside CUDA-graph capture); any n.
// partial / pscan: >= scan_scratch_elems(n) elements each.
template <class T, class F>
void exclusive_scan_on(cd_ctx *ctx, cudaStream_t s, int64_t n, F f, T *out, T *total, T *partial, T *pscan,
                       const char *family) {
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles <= 1) {
        CD_LAUNCH_S(ctx, s, family, (k_scan_apply<T, F>), 1, SCAN_THREADS, 0, n, f, static_cast<const T *>(nullptr),
                    out, total);
        return;
    }
    CD_LAUNCH_S(ctx, s, family, (k_scan_reduce<T, F>), static_cast<int>(tiles), SCAN_THREADS, 0, n, f, partial);
    // the tile partials: one block, or (beyond SCAN_TILE tiles) recursively
    // with the scratch that follows this level's
    exclusive_scan_on<T>(ctx, s, tiles, ArrayGen<T>{partial}, pscan, static_cast<T *>(nullptr), partial + tiles,
                         pscan + tiles, family);
    CD_LAUNCH_S(ctx, s, family, (k_scan_apply<T, F>), static_cast<int>(tiles), SCAN_THREADS, 0, n, f,
                static_cast<const T *>(pscan), out, total);
}

// out[i] = sum_{j<i} f(j) for i in [0, n); *total (device) = sum of all.
// out may alias nothing read by f.
template <class T, class F>
void exclusive_scan(cd_ctx *ctx, int64_t n, F f, T *out, T *total) {
    if (n <= 0) {
        if (total)
            CD_CUDA(cudaMemsetAsync(total, 0, sizeof(T), ctx->stream));
        return;
    }
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 1) {
        CD_LAUNCH(ctx, "scan", (k_scan_apply<T, F>), 1, SCAN_THREADS, 0, n, f, static_cast<const T *>(nullptr), out,
                  total);
        return;
    }
    DBuf<T> partial(ctx, tiles);
    DBuf<T> pscan(ctx, tiles);
    CD_LAUNCH(ctx, "scan", (k_scan_reduce<T, F>), static_cast<int>(tiles), SCAN_THREADS, 0, n, f, partial.p);
    exclusive_scan<T>(ctx, tiles, ArrayGen<T>{partial.p}, pscan.p, static_cast<T *>(nullptr));
    CD_LAUNCH(ctx, "scan", (k_scan_apply<T, F>), static_cast<int>(tiles), SCAN_THREADS, 0, n, f,
              static_cast<const T *>(pscan.p), out, total);
}

}  // namespace cdk
