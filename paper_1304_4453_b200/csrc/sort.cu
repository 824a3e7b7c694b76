// sort.cu -- device radix sort (sort.cuh).
#include "sort.cuh"

#include "scan.cuh"

namespace cdk {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 8;  // a tile = RS_ROUNDS x RS_THREADS keys, round-major
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr int RS_WARPS = RS_THREADS / 32;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint64_t *keys, int64_t n, int shift, int64_t ntiles,
                                                        int64_t *hist) {
    __shared__ int bins[256];
    bins[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t i = base + r * RS_THREADS + threadIdx.x;
        if (i < n)
            atomicAdd(&bins[(keys[i] >> shift) & 0xff], 1);
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = bins[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint64_t *keys, const uint32_t *vals, int64_t n,
                                                           int shift, int64_t ntiles, const int64_t *offs,
                                                           uint64_t *okeys, uint32_t *ovals) {
    __shared__ int cnt[RS_WARPS][256];
    __shared__ int64_t run[256];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    run[threadIdx.x] = offs[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * RS_TILE;
    for (int r = 0; r < RS_ROUNDS; ++r) {
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w)
            cnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = base + r * RS_THREADS + threadIdx.x;
        const bool valid = i < n;
        const uint64_t k = valid ? keys[i] : 0;
        const int d = valid ? static_cast<int>((k >> shift) & 0xff) : 256 + lane;  // invalid: unique dummy
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lanemask_lt());
        if (valid && rank == 0)
            cnt[wid][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int64_t pos = run[d] + rank;
            for (int w = 0; w < wid; ++w)
                pos += cnt[w][d];
            okeys[pos] = k;
            if (vals)
                ovals[pos] = vals[i];
        }
        __syncthreads();
        int s = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; ++w)
            s += cnt[w][threadIdx.x];
        run[threadIdx.x] += s;
        __syncthreads();
    }
}

}  // namespace

void radix_sort_pairs(cd_ctx *ctx, uint64_t *keys, uint32_t *vals, int64_t n, int end_bit) {
    if (n <= 1 || end_bit <= 0)
        return;
    const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    if (ntiles > INT32_MAX)
        fail(CD_EINVAL, "radix sort: too many keys");
    DBuf<uint64_t> k2(ctx, n);
    DBuf<uint32_t> v2(ctx, vals ? n : 0);
    DBuf<int64_t> hist(ctx, 256 * ntiles + 1), offs(ctx, 256 * ntiles + 1);
    uint64_t *ka = keys, *kb = k2.p;
    uint32_t *va = vals, *vb = vals ? v2.p : nullptr;
    int passes = 0;
    for (int shift = 0; shift < end_bit; shift += 8, ++passes) {
        CD_LAUNCH(ctx, "sort", k_rs_hist, static_cast<int>(ntiles), RS_THREADS, 0, static_cast<const uint64_t *>(ka),
                  n, shift, ntiles, hist.p);
        exclusive_scan<int64_t>(ctx, 256 * ntiles, ArrayGen<int64_t>{hist.p}, offs.p, offs.p + 256 * ntiles);
        CD_LAUNCH(ctx, "sort", k_rs_scatter, static_cast<int>(ntiles), RS_THREADS, 0,
                  static_cast<const uint64_t *>(ka), static_cast<const uint32_t *>(va), n, shift, ntiles,
                  static_cast<const int64_t *>(offs.p), kb, vb);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (passes & 1) {  // result sits in the scratch buffers
        CD_CUDA(cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        if (vals)
            CD_CUDA(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    }
}

}  // namespace cdk
