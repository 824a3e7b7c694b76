// common.cuh -- context, device buffers, launch accounting and device
// utilities shared by every kernel file of libcommdet_cuda.so (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "commdet_cuda.h"

namespace cdk {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
    cd_status code;
    Error(cd_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(cd_status c, const std::string &m) { throw Error(c, m); }

#define CD_CUDA(x)                                                                                   \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            ::cdk::fail(e_ == cudaErrorMemoryAllocation ? CD_ENOMEM : CD_ECUDA,                      \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                            \
    } while (0)

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct KStat {
    int64_t launches = 0;
    double total_ms = 0.0;
    double bytes = 0.0;
    double items = 0.0;
};

struct PendingEvent {
    std::string name;
    cudaEvent_t a, b;
};

class Comm;

}  // namespace cdk

struct cd_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaMemPool_t pool = nullptr;
    int num_sms = 148;
    size_t smem_optin = 0;
    // 0 off; 1 every launch timed, sweep tiers serialised on the library
    // stream; 2 sweep tiers as concurrent branches (as in the timed run), one
    // event pair around each sub-sweep's tier group ("<mode>.group")
    int profiling = 0;
    int64_t launches = 0;
    std::map<std::string, cdk::KStat> stats;
    std::vector<cdk::PendingEvent> pending;
    std::vector<cudaEvent_t> free_events;
    // small pinned staging area for scalar read-backs
    int64_t *pinned = nullptr;
    // device work counters of the sweep kernels (algorithmic-byte model):
    // [mode * STAT_MODE_STRIDE + slot * 3 + {0: nodes, 1: entries unweighted,
    // 2: entries weighted}], slot = degree tier, STAT_SLOT_SMALL or STAT_SLOT_FUSED
    unsigned long long *dstats = nullptr;
    // side streams + events used to capture independent kernels as parallel
    // branches of a CUDA graph
    static constexpr int NSIDE = 10;  // >= number of degree tiers
    cudaStream_t side[NSIDE] = {};
    cudaEvent_t fork_ev = nullptr;
    cudaEvent_t join_ev[NSIDE] = {};
    bool use_graphs = true;
    // host -> device uploads in chunks, overlapped with their validation
    cudaStream_t copy_stream = nullptr;
    // sharded execution (comm.cuh); nullptr = one device, no exchange
    cdk::Comm *comm = nullptr;
    // child context of a concurrent run on the same device (EPP bases): the
    // per-sub-sweep hub scratch is private to the context, keyed by graph
    // (graph.cuh hub_scratch_for); everything else a run writes is its own
    bool private_hubs = false;
    std::map<const void *, std::shared_ptr<void>> hub_scratch;
};

namespace cdk {

constexpr int STAT_SLOTS = 11;  // NUM_TIERS (9) + small + fused
constexpr int STAT_SLOT_SMALL = 9;
constexpr int STAT_SLOT_FUSED = 10;
constexpr int STAT_MODE_STRIDE = 3 * STAT_SLOTS;
constexpr int DSTATS = 2 * STAT_MODE_STRIDE;

// ---------------------------------------------------------------------------
// device buffers (stream-ordered pool allocations on the context stream)
// ---------------------------------------------------------------------------
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;

    DBuf() = default;
    DBuf(cd_ctx *ctx, size_t count) { alloc(ctx, count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }

    void alloc(cd_ctx *ctx, size_t count) {
        release();
        s = ctx->stream;
        n = count;
        if (count) {
            static const bool trace = std::getenv("CD_TRACE_ALLOC") != nullptr;
            if (trace && count * sizeof(T) >= (size_t(1) << 28)) {
                size_t fr = 0, tot = 0;
                cudaMemGetInfo(&fr, &tot);
                std::fprintf(stderr, "[alloc] %.2f GB (free %.2f GB)\n", count * sizeof(T) / 1e9, fr / 1e9);
            }
            cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&p), count * sizeof(T), s);
            if (e != cudaSuccess) {
                // the pool keeps freed blocks (release threshold = max): hand
                // them back to the device and retry once before failing
                cudaGetLastError();
                cudaMemPool_t pool;
                int dev = 0;
                if (cudaStreamSynchronize(s) == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
                    cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
                    cudaMemPoolTrimTo(pool, 0) == cudaSuccess)
                    e = cudaMallocAsync(reinterpret_cast<void **>(&p), count * sizeof(T), s);
            }
            if (e != cudaSuccess) {
                p = nullptr;
                n = 0;
                cudaGetLastError();
                size_t fr = 0, tot = 0;
                cudaMemGetInfo(&fr, &tot);
                cudaGetLastError();
                fail(CD_ENOMEM, "device allocation of " + std::to_string(count * sizeof(T)) + " bytes failed (" +
                                    std::to_string(fr) + " of " + std::to_string(tot) + " bytes free)");
            }
        }
    }
    void release() {
        if (p)
            cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    void zero() {
        if (p)
            CD_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void fill_bytes(int v) {
        if (p)
            CD_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), s));
    }
    T *get() const { return p; }
    size_t bytes() const { return n * sizeof(T); }
};

// ---------------------------------------------------------------------------
// launch accounting
// ---------------------------------------------------------------------------
cudaEvent_t ctx_event(cd_ctx *ctx);
void ctx_flush_stats(cd_ctx *ctx);  // resolves pending events (after sync)
void ctx_sync(cd_ctx *ctx);
int64_t read_counter(cd_ctx *ctx, int idx);  // syncs
void read_counters(cd_ctx *ctx, int first, int count, int64_t *out);  // syncs

struct LaunchScope {
    cd_ctx *ctx;
    const char *name;
    cudaEvent_t a = nullptr;
    LaunchScope(cd_ctx *c, const char *nm) : ctx(c), name(nm) {
        ctx->launches++;
        if (ctx->profiling) {
            a = ctx_event(ctx);
            cudaEventRecord(a, ctx->stream);
        }
    }
    ~LaunchScope() {
        if (ctx->profiling) {
            cudaEvent_t b = ctx_event(ctx);
            cudaEventRecord(b, ctx->stream);
            ctx->pending.push_back({name, a, b});
        }
    }
};

inline void check_launch(const char *name) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        fail(CD_ECUDA, std::string("launch of ") + name + ": " + cudaGetErrorString(e));
}

// LAUNCH(ctx, "family", kernel, grid, block, smem)(args...)
#define CD_LAUNCH(ctx, family, kernel, grid, block, smem, ...)                                       \
    do {                                                                                             \
        ::cdk::LaunchScope ls_((ctx), (family));                                                     \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                            \
        ::cdk::check_launch(family);                                                                 \
    } while (0)

// same on an explicit stream (graph capture branches; never profiled)
#define CD_LAUNCH_S(ctx, strm, family, kernel, grid, block, smem, ...)                               \
    do {                                                                                             \
        (ctx)->launches++;                                                                           \
        kernel<<<(grid), (block), (smem), (strm)>>>(__VA_ARGS__);                                   \
        ::cdk::check_launch(family);                                                                 \
    } while (0)

inline void add_stat_work(cd_ctx *ctx, const char *family, double bytes, double items) {
    auto &s = ctx->stats[family];
    s.bytes += bytes;
    s.items += items;
}

// integer tuning knob from the environment (default when unset / malformed)
inline int64_t env_i64(const char *name, int64_t dflt) {
    const char *e = std::getenv(name);
    if (!e || !*e)
        return dflt;
    char *end = nullptr;
    const long long v = std::strtoll(e, &end, 10);
    return (end && *end == '\0') ? static_cast<int64_t>(v) : dflt;
}

inline int grid_for(int64_t items, int per_block, int cap_blocks) {
    int64_t g = (items + per_block - 1) / per_block;
    if (g < 1)
        g = 1;
    if (g > cap_blocks)
        g = cap_blocks;
    return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// host <-> device argument handling: every ABI array may be host or device
// ---------------------------------------------------------------------------
bool is_device_ptr(const void *p);

template <class T>
struct InArr {
    const T *d = nullptr;
    DBuf<T> own;
    InArr(cd_ctx *ctx, const T *p, size_t count) {
        if (!p || count == 0) {
            d = p;
            return;
        }
        if (is_device_ptr(p)) {
            d = p;
        } else {
            own.alloc(ctx, count);
            CD_CUDA(cudaMemcpyAsync(own.p, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
            d = own.p;
        }
    }
};

template <class T>
struct OutArr {
    T *host = nullptr;
    T *d = nullptr;
    DBuf<T> own;
    size_t count = 0;
    cd_ctx *ctx;
    OutArr(cd_ctx *c, T *p, size_t cnt) : ctx(c), count(cnt) {
        if (!p || cnt == 0) {
            d = p;
            return;
        }
        if (is_device_ptr(p)) {
            d = p;
        } else {
            host = p;
            own.alloc(ctx, cnt);
            d = own.p;
        }
    }
    void finish() {
        if (host && count)
            CD_CUDA(cudaMemcpyAsync(host, d, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    }
};

// ---------------------------------------------------------------------------
// device utilities
// ---------------------------------------------------------------------------
constexpr int32_t EMPTY_KEY = -1;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// Bucket schedule shared by every driver (ported in oracle/commdet_oracle.c:
// cdo_bucket_key / cdo_bucket_of).
__host__ __device__ __forceinline__ uint64_t bucket_key(uint64_t seed, uint64_t salt) {
    return splitmix64(seed ^ splitmix64(salt ^ 0xb5ad4eceda1ce2a9ULL));
}
__host__ __device__ __forceinline__ int32_t bucket_of(uint64_t key, int32_t u, int32_t buckets) {
    return static_cast<int32_t>(static_cast<uint32_t>(splitmix64(key ^ static_cast<uint64_t>(static_cast<uint32_t>(u))) >> 32) %
                                static_cast<uint32_t>(buckets));
}

// Open-addressing slot of a label: Fibonacci hashing proper -- the TOP
// bits of key * C (multiply-high by the table size).  They depend on every
// key bit, and consecutive keys (compacted community ids) land nearly evenly
// spaced.  The low bits of the product (the old slot) depend only on the
// key's low bits, and R-MAT ids share low bits heavily (each id bit is 0
// with probability a+b = 0.76): a hub's probe chains grew to hundreds of
// slots (C3 PLM 371 -> 295 ms, C3 PLP 38 -> 28 ms with this hash).  The
// multiplier differs from the owner / partition hash (top bits of
// key * 0x9E3779B1), so a CTA's or partition's keys spread over its table.
__device__ __forceinline__ uint32_t hash_slot(int32_t key, uint32_t mask) {
    return __umulhi(static_cast<uint32_t>(key) * 0x2545F491u, mask + 1u);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// warp-aggregated append: returns the slot for this lane (only lanes with
// pred == true get a valid slot).
__device__ __forceinline__ int32_t warp_append(int32_t *counter, bool pred) {
    const uint32_t mask = __ballot_sync(0xffffffffu, pred);
    if (!mask)
        return -1;
    const int leader = __ffs(mask) - 1;
    int32_t base = 0;
    if (lane_id() == leader)
        base = atomicAdd(counter, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(mask & lanemask_lt());
}

// Sum v over the lanes (with pred) sharing `key`; returns true on the group
// leader (lowest lane), which receives the sum in `out`.  scratch is 32
// doubles private to the calling warp.  Must be called by the full warp.
__device__ __forceinline__ bool warp_aggregate_sum(int32_t key, double v, bool pred, double *scratch, double &out) {
    const int lane = lane_id();
    const uint32_t vm = __ballot_sync(0xffffffffu, pred);
    const uint32_t peers = __match_any_sync(0xffffffffu, key) & vm;
    scratch[lane] = v;
    __syncwarp();
    const bool leader = pred && (__ffs(peers) - 1) == lane;
    if (leader) {
        double s = 0.0;
        for (uint32_t p = peers; p; p &= p - 1)
            s += scratch[__ffs(p) - 1];
        out = s;
    }
    __syncwarp();
    return leader;
}

inline uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x)
        p <<= 1;
    return p;
}

}  // namespace cdk
