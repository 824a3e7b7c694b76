// Microbenchmark of per-node label tallies (PLP count tallies: argmax count,
// ties -> smallest label), warp per row, rows of D <= 256 labels.  Decides
// how the sweep kernels aggregate: shared-memory atomics cost one L1 data-pipe
// wavefront per lane, plain LDS/STS one per warp instruction (per bank-
// conflict degree), so the variants trade atomics for warp collectives.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tally_bench tools/microbench/tally_bench.cu
//   ./tally_bench [rows] [deg] [universe]
//
// Variants:
//   cas    atomicCAS claim + atomicAdd count per entry (the round-1 WARP tier)
//   pack   one 64-bit word per slot (key << 32 | count): claim-with-count-1 CAS,
//          atomicAdd on a hit
//   match  __match_any_sync per 32-entry round, leaders insert (packed)
//   sort   warp bitonic sort of the row (8 keys per lane), run-length argmax
// Labels are pre-gathered (coalesced), so only the tally is timed; `gather`
// times the random z[v] gather alone for scale.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int CAP = 512;
constexpr int ITEMS = 8;
constexpr int32_t EMPTY = -1;

__device__ __forceinline__ uint32_t hslot(int32_t key, uint32_t mask) {
    return __umulhi(static_cast<uint32_t>(key) * 0x2545F491u, mask + 1u);
}
__device__ __forceinline__ bool better(uint32_t a, int32_t ka, uint32_t b, int32_t kb) {
    return a > b || (a == b && ka < kb);
}
__device__ __forceinline__ void warp_argmax(uint32_t &v, int32_t &k) {
    for (int o = 16; o > 0; o >>= 1) {
        uint32_t ov = __shfl_xor_sync(~0u, v, o);
        int32_t ok = __shfl_xor_sync(~0u, k, o);
        if (better(ov, ok, v, k)) { v = ov; k = ok; }
    }
}
__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

// ---- cas: 32-bit keys + 32-bit counts, CAS then add -------------------------
template <bool SKIP>
__global__ void __launch_bounds__(128, 8) k_cas(int64_t rows, int deg, const int32_t *lab, int32_t *out) {
    __shared__ int32_t skeys[4][CAP];
    __shared__ uint32_t svals[4][CAP];
    __shared__ uint16_t sdist[4][CAP / 2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *keys = skeys[w]; uint32_t *vals = svals[w]; uint16_t *dist = sdist[w];
    for (int t = lane; t < CAP; t += 32) { keys[t] = EMPTY; vals[t] = 0; }
    __syncwarp();
    uint32_t cap = 64; while (cap < 2u * deg) cap <<= 1;
    const uint32_t mask = cap - 1;
    for (int64_t r = (blockIdx.x * 4 + w); r < rows; r += gridDim.x * 4) {
        const int32_t *row = lab + r * deg;
        int32_t kk[ITEMS];
#pragma unroll
        for (int c = 0; c < ITEMS; ++c) kk[c] = c * 32 + lane < deg ? row[c * 32 + lane] : EMPTY;
        int nd = 0;
#pragma unroll
        for (int c = 0; c < ITEMS; ++c) {
            if (c * 32 >= deg) break;
            bool claimed = false; uint32_t slot = 0;
            if (kk[c] != EMPTY) {
                uint32_t s = hslot(kk[c], mask);
                while (true) {
                    int32_t old = atomicCAS(&keys[s], EMPTY, kk[c]);
                    if (old == EMPTY || old == kk[c]) {
                        claimed = old == EMPTY;
                        if (!SKIP || !claimed) atomicAdd(&vals[s], 1u);  // SKIP: a claim counts 1 implicitly
                        slot = s; break; }
                    s = (s + 1) & mask;
                }
            }
            uint32_t cm = __ballot_sync(~0u, claimed);
            if (claimed) dist[nd + __popc(cm & lanemask_lt())] = (uint16_t)slot;
            nd += __popc(cm);
        }
        __syncwarp();
        uint32_t bv = 0; int32_t bk = INT32_MAX;
        for (int j = lane; j < nd; j += 32) {
            uint32_t t = dist[j];
            const uint32_t v = vals[t] + (SKIP ? 1u : 0u);
            if (better(v, keys[t], bv, bk)) { bv = v; bk = keys[t]; }
            keys[t] = EMPTY; vals[t] = 0;
        }
        warp_argmax(bv, bk);
        if (lane == 0) out[r] = bk;
        __syncwarp();
    }
}

// ---- pack: one 64-bit slot = key << 32 | count ------------------------------
__device__ __forceinline__ bool pinsert(unsigned long long *tab, uint32_t mask, int32_t key, uint32_t cnt, uint32_t *slot) {
    uint32_t s = hslot(key, mask);
    const unsigned long long mine = (static_cast<unsigned long long>(static_cast<uint32_t>(key)) << 32) | cnt;
    while (true) {
        unsigned long long old = atomicCAS(&tab[s], ~0ULL, mine);
        if (old == ~0ULL) { *slot = s; return true; }
        if (static_cast<int32_t>(old >> 32) == key) { atomicAdd(&tab[s], static_cast<unsigned long long>(cnt)); return false; }
        s = (s + 1) & mask;
    }
}

template <bool MATCH>
__global__ void __launch_bounds__(128, 8) k_pack(int64_t rows, int deg, const int32_t *lab, int32_t *out) {
    __shared__ unsigned long long stab[4][CAP];
    __shared__ uint16_t sdist[4][CAP / 2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long *tab = stab[w]; uint16_t *dist = sdist[w];
    for (int t = lane; t < CAP; t += 32) tab[t] = ~0ULL;
    __syncwarp();
    uint32_t cap = 64; while (cap < 2u * deg) cap <<= 1;
    const uint32_t mask = cap - 1;
    for (int64_t r = (blockIdx.x * 4 + w); r < rows; r += gridDim.x * 4) {
        const int32_t *row = lab + r * deg;
        int32_t kk[ITEMS];
#pragma unroll
        for (int c = 0; c < ITEMS; ++c) kk[c] = c * 32 + lane < deg ? row[c * 32 + lane] : EMPTY;
        int nd = 0;
#pragma unroll
        for (int c = 0; c < ITEMS; ++c) {
            if (c * 32 >= deg) break;
            bool claimed = false; uint32_t slot = 0;
            const bool valid = kk[c] != EMPTY;
            if (MATCH) {
                const uint32_t vm = __ballot_sync(~0u, valid);
                const uint32_t peers = __match_any_sync(~0u, kk[c]) & vm;
                if (valid && (__ffs(peers) - 1) == lane) claimed = pinsert(tab, mask, kk[c], __popc(peers), &slot);
            } else if (valid) {
                claimed = pinsert(tab, mask, kk[c], 1u, &slot);
            }
            uint32_t cm = __ballot_sync(~0u, claimed);
            if (claimed) dist[nd + __popc(cm & lanemask_lt())] = (uint16_t)slot;
            nd += __popc(cm);
        }
        __syncwarp();
        uint32_t bv = 0; int32_t bk = INT32_MAX;
        for (int j = lane; j < nd; j += 32) {
            uint32_t t = dist[j];
            unsigned long long x = tab[t];
            int32_t k = static_cast<int32_t>(x >> 32); uint32_t v = static_cast<uint32_t>(x);
            if (better(v, k, bv, bk)) { bv = v; bk = k; }
            tab[t] = ~0ULL;
        }
        warp_argmax(bv, bk);
        if (lane == 0) out[r] = bk;
        __syncwarp();
    }
}

// ---- sort: bitonic over 256 = 8 regs x 32 lanes, element e = c*32 + lane ----
__device__ __forceinline__ void cswap(int32_t &a, int32_t &b, bool up) {
    int32_t lo = min(a, b), hi = max(a, b);
    a = up ? lo : hi; b = up ? hi : lo;
}
template <int NREG>
__device__ __forceinline__ void warp_bitonic(int32_t (&x)[ITEMS]) {
    const int lane = threadIdx.x & 31;
    constexpr int N = NREG * 32;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                // in-register: element e = c*32+lane, partner e^j differs in c
                const int jc = j >> 5;
#pragma unroll
                for (int c = 0; c < NREG; ++c) {
                    const int pc = c ^ jc;
                    if (pc > c) {
                        const int e = c * 32 + lane;
                        const bool up = (e & k) == 0;
                        cswap(x[c], x[pc], up);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < NREG; ++c) {
                    const int e = c * 32 + lane;
                    const int32_t o = __shfl_xor_sync(~0u, x[c], j);
                    const bool up = (e & k) == 0;
                    const bool lower = (lane & j) == 0;
                    // lower element keeps min if ascending
                    x[c] = (lower == up) ? min(x[c], o) : max(x[c], o);
                }
            }
        }
    }
}

template <int NREG>
__device__ __forceinline__ void sort_row(const int32_t *row, int deg, int lane, int32_t &bk_out) {
    int32_t x[ITEMS];
#pragma unroll
    for (int c = 0; c < ITEMS; ++c) x[c] = (c < NREG && c * 32 + lane < deg) ? row[c * 32 + lane] : INT32_MAX;
    warp_bitonic<NREG>(x);
    // run-length: element e = c*32+lane sorted ascending; run starts where x[e] != x[e-1]
    // count of a run = (next start) - start; find via per-element "distance to run end"
    uint32_t bv = 0; int32_t bk = INT32_MAX;
    // prev element of e: if lane>0 same c, lane-1; else c-1, lane 31
    int32_t prev[ITEMS], next_start_pos[ITEMS];
#pragma unroll
    for (int c = 0; c < NREG; ++c) {
        int32_t p = __shfl_up_sync(~0u, x[c], 1);
        int32_t last_prev = c > 0 ? __shfl_sync(~0u, x[c - 1], 31) : INT32_MIN;
        prev[c] = lane == 0 ? last_prev : p;
    }
    // run starts; for each start, its run length = position of the next start - pos.
    // suffix-min of start positions: compute via ballots
    uint32_t startmask[ITEMS];
#pragma unroll
    for (int c = 0; c < NREG; ++c) startmask[c] = __ballot_sync(~0u, x[c] != prev[c]);
#pragma unroll
    for (int c = 0; c < NREG; ++c) {
        const bool st = x[c] != prev[c] && x[c] != INT32_MAX;
        if (st) {
            // next start after e = c*32+lane
            int nxt = -1;
            uint32_t after = startmask[c] & ~((2u << lane) - 1u);
            if (lane == 31) after = 0;
            if (after) nxt = c * 32 + __ffs(after) - 1;
            else {
#pragma unroll
                for (int cc = 0; cc < NREG; ++cc)
                    if (cc > c && nxt < 0 && startmask[cc]) nxt = cc * 32 + __ffs(startmask[cc]) - 1;
                if (nxt < 0) nxt = NREG * 32;
            }
            const uint32_t cnt = nxt - (c * 32 + lane);
            if (better(cnt, x[c], bv, bk)) { bv = cnt; bk = x[c]; }
        }
        next_start_pos[c] = 0;
    }
    warp_argmax(bv, bk);
    bk_out = bk;
}

__global__ void __launch_bounds__(128, 8) k_sort(int64_t rows, int deg, const int32_t *lab, int32_t *out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t r = (blockIdx.x * 4 + w); r < rows; r += gridDim.x * 4) {
        const int32_t *row = lab + r * deg;
        int32_t bk;
        if (deg <= 64) sort_row<2>(row, deg, lane, bk);
        else if (deg <= 128) sort_row<4>(row, deg, lane, bk);
        else sort_row<8>(row, deg, lane, bk);
        if (lane == 0) out[r] = bk;
    }
}

// random gather z[idx] for scale: D entries per row, warp per row
__global__ void __launch_bounds__(128, 8) k_gather(int64_t rows, int deg, const int32_t *idx, const int32_t *z, int32_t *out) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t r = (blockIdx.x * 4 + w); r < rows; r += gridDim.x * 4) {
        int32_t acc = 0;
#pragma unroll
        for (int c = 0; c < ITEMS; ++c)
            if (c * 32 + lane < deg) acc ^= z[idx[r * deg + c * 32 + lane]];
        acc = __reduce_xor_sync(~0u, acc);
        if (lane == 0) out[r] = acc;
    }
}

int main(int argc, char **argv) {
    const int64_t rows = argc > 1 ? atoll(argv[1]) : 1 << 20;
    const int deg = argc > 2 ? atoi(argv[2]) : 64;
    const int64_t universe = argc > 3 ? atoll(argv[3]) : 1 << 24;
    const int64_t N = rows * deg;
    std::vector<int32_t> h(N);
    std::mt19937_64 rng(1);
    // skewed labels: universe controls duplicates within a row
    for (int64_t i = 0; i < N; ++i) h[i] = static_cast<int32_t>(rng() % universe);
    int32_t *lab, *o1, *o2, *o3, *o4, *o5, *z;
    CK(cudaMalloc(&lab, N * 4)); CK(cudaMalloc(&o1, rows * 4)); CK(cudaMalloc(&o2, rows * 4));
    CK(cudaMalloc(&o3, rows * 4)); CK(cudaMalloc(&o4, rows * 4)); CK(cudaMalloc(&o5, rows * 4));
    const int64_t nz = 1 << 24;
    CK(cudaMalloc(&z, nz * 4));
    CK(cudaMemset(z, 0, nz * 4));
    CK(cudaMemcpy(lab, h.data(), N * 4, cudaMemcpyHostToDevice));
    // gather indices: labels mod nz
    int32_t *idx; CK(cudaMalloc(&idx, N * 4));
    for (auto &v : h) v = static_cast<int32_t>(rng() % nz);
    CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = sms * 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto time = [&](const char *name, auto launch) {
        launch(); CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) launch();
        cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("%-8s deg %3d universe %10lld : %8.3f ms  %6.3f ns/entry  %7.1f G entries/s\n", name, deg,
               (long long)universe, ms, ms * 1e6 / N, N / (ms * 1e-3) / 1e9);
    };
    time("cas", [&] { k_cas<false><<<grid, 128>>>(rows, deg, lab, o1); });
    time("cas1", [&] { k_cas<true><<<grid, 128>>>(rows, deg, lab, o5); });
    {
        std::vector<int32_t> x(rows), y(rows);
        CK(cudaMemcpy(x.data(), o1, rows * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(y.data(), o5, rows * 4, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (int64_t r = 0; r < rows; ++r) bad += x[r] != y[r];
        printf("cas1 mismatches %lld\n", (long long)bad);
    }
    time("pack", [&] { k_pack<false><<<grid, 128>>>(rows, deg, lab, o2); });
    time("match", [&] { k_pack<true><<<grid, 128>>>(rows, deg, lab, o3); });
    time("sort", [&] { k_sort<<<grid, 128>>>(rows, deg, lab, o4); });
    time("gather", [&] { k_gather<<<grid, 128>>>(rows, deg, idx, z, o5); });
    std::vector<int32_t> r1(rows), r2(rows), r3(rows), r4(rows);
    CK(cudaMemcpy(r1.data(), o1, rows * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r2.data(), o2, rows * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r3.data(), o3, rows * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r4.data(), o4, rows * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t r = 0; r < rows; ++r) bad += (r1[r] != r2[r]) + (r1[r] != r3[r]) + (r1[r] != r4[r]);
    printf("mismatches %lld\n", (long long)bad);
    return 0;
}
