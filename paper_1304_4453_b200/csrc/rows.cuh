// rows.cuh -- the row engine: for every output row r, reduce its source
// entries (key, weight) by key (hash tally; duplicates summed / detected) and
// emit the distinct keys sorted ascending as a CSR row.
//
// This one engine is both
//   * the CSR builder behind Graph::from_edges (H/graph.hpp:48-81,
//     sort_and_merge :169-204): rows = scattered raw adjacency, and
//   * the contraction of coarsen (H/louvain.hpp:154-220): row c = the fine
//     rows of c's members, keyed by the neighbour's community, intra-community
//     entries kept once (v >= u).
//
// Reduce tiers by source length F_r:   <=32 warp+match_any | <=256 warp smem
// hash | <=4096 block smem hash | >4096 multi-block global hash.
// Sort tiers by distinct length L_r:   <=32 warp bitonic | <=8192 block
// bitonic in smem | >8192 block-local LSD radix sort in global memory.
#pragma once

#include <algorithm>

#include "graph.cuh"
#include "scan.cuh"

namespace cdk {

constexpr int ENG_WARP_F = 256;
constexpr int ENG_BLOCK_F = 4096;
constexpr int ENG_GLOBAL_CHUNK = 4096;
constexpr int ENG_SORT_BLOCK = 8192;

// -------------------------------------------------------------------------
// sources: warp-collective loaders.  Every lane of the warp calls load() with
// the same (r, f0); lane i handles flat entry f0 + i.
// -------------------------------------------------------------------------
struct SrcFlat {
    const int64_t *fpre;  // row r's entries: [fpre[r], fpre[r+1])
    const int32_t *key;
    const float *w;       // nullable
    struct Cursor {};
    __device__ Cursor init(int64_t, int64_t) const { return {}; }
    __device__ void load(int64_t, int64_t f0, int64_t fend, Cursor &, int32_t &k, double &wt, bool &valid) const {
        const int64_t f = f0 + lane_id();
        valid = f < fend;
        k = valid ? key[f] : 0;
        wt = (valid && w) ? static_cast<double>(w[f]) : 1.0;
    }
};

// coarse row c = concatenation of the fine rows of its members (member
// order), mapped through z; entry (u -> v) with z[v] == c kept iff v >= u.
struct SrcCoarsen {
    const int64_t *moff;  // [nc+1] member ranges
    const int32_t *mem;   // members grouped by community
    const int64_t *mpre;  // [n+1] exclusive prefix of member degrees (member order)
    const int64_t *off;
    const int32_t *col;
    const float *w;  // nullable
    const int32_t *z;
    struct Cursor {
        int64_t p;
    };
    __device__ Cursor init(int64_t c, int64_t f0) const {
        int64_t lo = moff[c], hi = moff[c + 1] - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (mpre[mid] <= f0)
                lo = mid;
            else
                hi = mid - 1;
        }
        return {lo};
    }
    __device__ void load(int64_t c, int64_t f0, int64_t fend, Cursor &cur, int32_t &k, double &wt,
                         bool &valid) const {
        const int lane = lane_id();
        const int64_t f = f0 + lane;
        const int64_t pe = moff[c + 1];
        bool done = !(f < fend);
        int64_t p = cur.p;
        int64_t base = cur.p;
        while (true) {
            const int64_t q = base + 1 + lane;
            const int64_t bnd = q < pe ? mpre[q] : INT64_MAX;
            const int64_t last = __shfl_sync(0xffffffffu, bnd, 31);
            // number of lanes j with bnd_j <= f (bnd ascending across lanes)
            int cnt = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int64_t v = __shfl_sync(0xffffffffu, bnd, cnt + step - 1);
                if (v <= f)
                    cnt += step;
            }
            if (!done && !(last <= f)) {
                p = base + cnt;
                done = true;
            }
            if (__all_sync(0xffffffffu, done))
                break;
            base += 32;
        }
        valid = f < fend;
        k = 0;
        wt = 1.0;
        int32_t u = 0, v = 0;
        if (valid) {
            u = mem[p];
            const int64_t e = off[u] + (f - mpre[p]);
            v = __ldcs(col + e);  // streamed once: evict-first keeps z cached
            wt = w ? static_cast<double>(__ldcs(w + e)) : 1.0;
            k = z[v];
            if (k == static_cast<int32_t>(c) && v < u)
                valid = false;
        }
        // next chunk starts at the member of the highest in-range lane (p is
        // monotone across lanes; out-of-range lanes kept the old cursor)
        int64_t pm = p;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            pm = max(pm, __shfl_xor_sync(0xffffffffu, pm, o));
        cur.p = pm;
    }
};

// rows [r0, r0 + rows) of another source, renumbered from 0, with flat
// entry indices rebased by f0 (= the source's prefix at r0): one batch of a
// row engine run split to bound its scratch
template <class Src>
struct SrcWindow {
    Src s;
    int64_t r0, f0;
    using Cursor = typename Src::Cursor;
    __device__ Cursor init(int64_t r, int64_t f) const { return s.init(r + r0, f + f0); }
    __device__ void load(int64_t r, int64_t f, int64_t fend, Cursor &cur, int32_t &k, double &wt,
                         bool &valid) const {
        s.load(r + r0, f + f0, fend + f0, cur, k, wt, valid);
    }
};

// -------------------------------------------------------------------------
// warp aggregation: lanes with equal keys combine; the lowest lane of each
// group is the leader and receives the group's weight sum (summed in lane
// order) and count.
// -------------------------------------------------------------------------
__device__ __forceinline__ bool warp_aggregate(int32_t key, double w, bool valid, uint32_t group_mask,
                                               double *scratch32, double &sum, uint32_t &cnt) {
    const int lane = lane_id();
    const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    const uint32_t peers = __match_any_sync(0xffffffffu, key) & vmask & group_mask;
    const bool leader = valid && ((__ffs(peers) - 1) == lane);
    cnt = __popc(peers);
    scratch32[lane] = w;
    __syncwarp();
    double s = 0.0;
    if (leader)
        for (uint32_t m = peers; m; m &= m - 1)
            s += scratch32[__ffs(m) - 1];
    __syncwarp();
    sum = s;
    return leader;
}

// open-addressing insert (linear probing) into a table of any `cap` slots
// (the global tier sizes tables at exactly 2x the row's entries)
__device__ __forceinline__ void table_insert_n(int32_t *keys, double *vals, uint32_t *cnts, uint32_t cap,
                                               int32_t key, double w, uint32_t c) {
    uint32_t s = hash_slot(key, cap - 1);  // multiply-high by cap: any table size
    while (true) {
        const int32_t old = atomicCAS(&keys[s], EMPTY_KEY, key);
        if (old == EMPTY_KEY || old == key) {
            atomicAdd(&vals[s], w);
            if (cnts)
                atomicAdd(&cnts[s], c);
            return;
        }
        s = (s + 1 == cap) ? 0 : s + 1;
    }
}

// open-addressing insert (linear probing) into a table with 2^k slots
__device__ __forceinline__ void table_insert(int32_t *keys, double *vals, uint32_t *cnts, uint32_t mask,
                                             int32_t key, double w, uint32_t c) {
    uint32_t s = hash_slot(key, mask);
    while (true) {
        const int32_t old = atomicCAS(&keys[s], EMPTY_KEY, key);
        if (old == EMPTY_KEY || old == key) {
            atomicAdd(&vals[s], w);
            if (cnts)
                atomicAdd(&cnts[s], c);
            return;
        }
        s = (s + 1) & mask;
    }
}

struct EngineOut {
    int32_t *tkey;   // [F_total] reduced keys (row r at fpre[r])
    double *tval;    // [F_total]
    int64_t *deg2;   // [nrows] distinct count
    int64_t *flag;   // duplicates seen (nullptr: not tracked); written once
};

// ---- reduce kernels -------------------------------------------------------

template <class Src>
static __global__ void __launch_bounds__(256) k_eng_reduce_direct(Src src, const int64_t *fpre, const int32_t *rows,
                                                           int64_t nrows, int mode, EngineOut out) {
    __shared__ double scratch[8][32];
    const int wid = threadIdx.x >> 5, lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = gw; i < nrows; i += nw) {
        const int64_t r = rows[i];
        const int64_t f0 = fpre[r], f1 = fpre[r + 1];
        auto cur = src.init(r, f0);
        int32_t k;
        double w;
        bool valid;
        src.load(r, f0, f1, cur, k, w, valid);
        double sum;
        uint32_t cnt;
        const bool leader = warp_aggregate(k, w, valid, 0xffffffffu, scratch[wid], sum, cnt);
        const uint32_t lm = __ballot_sync(0xffffffffu, leader);
        if (leader) {
            const int rank = __popc(lm & lanemask_lt());
            out.tkey[f0 + rank] = k;
            out.tval[f0 + rank] = mode == DUP_ONE ? 1.0 : sum;
            if (cnt > 1 && out.flag && !*out.flag)
                *out.flag = 1;
        }
        if (lane == 0)
            out.deg2[r] = __popc(lm);
    }
}

__device__ __forceinline__ uint32_t table_cap_for(int64_t F, int64_t key_bound, uint32_t cap_max) {
    int64_t need = 2 * (F < key_bound ? F : key_bound);
    uint32_t cap = 32;
    while (cap < need && cap < cap_max)
        cap <<= 1;
    return cap;
}

template <class Src, bool TRACK = true>
static __global__ void __launch_bounds__(128) k_eng_reduce_warp(Src src, const int64_t *fpre, const int32_t *rows,
                                                         int64_t nrows, int64_t key_bound, int mode,
                                                         EngineOut out) {
    constexpr int CAP = 2 * ENG_WARP_F;
    __shared__ double scratch[4][32];
    __shared__ int32_t skeys[4][CAP];
    __shared__ double svals[4][CAP];
    __shared__ uint32_t scnts[4][TRACK ? CAP : 1];  // duplicate counts only when tracked
    const int wid = threadIdx.x >> 5, lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int32_t *keys = skeys[wid];
    double *vals = svals[wid];
    uint32_t *cnts = TRACK ? scnts[wid] : nullptr;
    for (int64_t i = gw; i < nrows; i += nw) {
        const int64_t r = rows[i];
        const int64_t f0 = fpre[r], f1 = fpre[r + 1];
        const uint32_t cap = table_cap_for(f1 - f0, key_bound, CAP);
        for (uint32_t s = lane; s < cap; s += 32) {
            keys[s] = EMPTY_KEY;
            vals[s] = 0.0;
            if (TRACK)
                cnts[s] = 0;
        }
        __syncwarp();
        auto cur = src.init(r, f0);
        for (int64_t f = f0; f < f1; f += 32) {
            int32_t k;
            double w;
            bool valid;
            src.load(r, f, f1, cur, k, w, valid);
            double sum;
            uint32_t cnt;
            if (warp_aggregate(k, w, valid, 0xffffffffu, scratch[wid], sum, cnt))
                table_insert(keys, vals, cnts, cap - 1, k, sum, cnt);
        }
        __syncwarp();
        int64_t base = 0;
        for (uint32_t s0 = 0; s0 < cap; s0 += 32) {
            const uint32_t s = s0 + lane;
            const bool has = keys[s] != EMPTY_KEY;
            const uint32_t bm = __ballot_sync(0xffffffffu, has);
            if (has) {
                const int64_t pos = f0 + base + __popc(bm & lanemask_lt());
                out.tkey[pos] = keys[s];
                out.tval[pos] = mode == DUP_ONE ? 1.0 : vals[s];
                if (TRACK && cnts[s] > 1 && out.flag && !*out.flag)
                    *out.flag = 1;
            }
            base += __popc(bm);
        }
        if (lane == 0)
            out.deg2[r] = base;
        __syncwarp();
    }
}

// Block tier, instantiated per table capacity: the rows of the block list
// with fmin < F <= fmax (fmax <= CAP / 2).  The small instance (rows of at
// most 1024 entries, 32 KB of tables) runs 4 blocks per SM where the 4096-row
// instance (128 KB) runs one.
template <class Src, int CAP = 2 * ENG_BLOCK_F, bool TRACK = true>
static __global__ void __launch_bounds__(512, CAP <= 2048 ? 4 : 1) k_eng_reduce_block(Src src, const int64_t *fpre, const int32_t *rows,
                                                          int64_t nrows, int64_t key_bound, int mode,
                                                          EngineOut out, int64_t fmin, int64_t fmax) {
    extern __shared__ unsigned char smem_raw[];
    double *vals = reinterpret_cast<double *>(smem_raw);
    int32_t *keys = reinterpret_cast<int32_t *>(vals + CAP);
    uint32_t *cnts = TRACK ? reinterpret_cast<uint32_t *>(keys + CAP) : nullptr;
    __shared__ double scratch[16][32];
    __shared__ int32_t counter;
    const int wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5, lane = lane_id();
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int64_t r = rows[i];
        const int64_t f0 = fpre[r], f1 = fpre[r + 1];
        if (f1 - f0 <= fmin || f1 - f0 > fmax)
            continue;
        const uint32_t cap = table_cap_for(f1 - f0, key_bound, CAP);
        for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
            keys[s] = EMPTY_KEY;
            vals[s] = 0.0;
            if (TRACK)
                cnts[s] = 0;
        }
        if (threadIdx.x == 0)
            counter = 0;
        __syncthreads();
        // each warp takes a contiguous slice of the row (cursor friendly)
        const int64_t F = f1 - f0;
        const int64_t per = ((F + nwarps - 1) / nwarps + 31) & ~int64_t(31);
        const int64_t a = f0 + wid * per;
        const int64_t b = min(f1, a + per);
        if (a < b) {
            auto cur = src.init(r, a);
            for (int64_t f = a; f < b; f += 32) {
                int32_t k;
                double w;
                bool valid;
                src.load(r, f, b, cur, k, w, valid);
                double sum;
                uint32_t cnt;
                if (warp_aggregate(k, w, valid, 0xffffffffu, scratch[wid], sum, cnt))
                    table_insert(keys, vals, cnts, cap - 1, k, sum, cnt);
            }
        }
        __syncthreads();
        for (uint32_t s0 = wid * 32; s0 < cap; s0 += blockDim.x) {
            const uint32_t s = s0 + lane;
            const bool has = s < cap && keys[s] != EMPTY_KEY;
            const int32_t pos = warp_append(&counter, has);
            if (has) {
                out.tkey[f0 + pos] = keys[s];
                out.tval[f0 + pos] = mode == DUP_ONE ? 1.0 : vals[s];
                if (TRACK && cnts[s] > 1 && out.flag && !*out.flag)
                    *out.flag = 1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0)
            out.deg2[r] = counter;
        __syncthreads();
    }
}

// global tier: grid over chunks of ENG_GLOBAL_CHUNK entries of the big rows.
// A block first combines its chunk in a small shared-memory table (a row
// with few distinct keys -- a coarse level's giant communities -- would
// otherwise hammer the same global slots with atomics from every block),
// then inserts each distinct key once into the row's global table.  Keys
// that find no smem slot within a few probes go to the global table directly.
constexpr int ENG_PRE_CAP = 2048;
constexpr int ENG_PRE_PROBES = 8;

template <class Src>
static __global__ void __launch_bounds__(256) k_eng_reduce_global_insert(Src src, const int64_t *fpre,
                                                                  const int32_t *rows, int64_t nrows,
                                                                  const int64_t *chunk_pre, const int64_t *tab_off,
                                                                  const int64_t *tab_cap, int32_t *gkeys,
                                                                  double *gvals, uint32_t *gcnts) {
    __shared__ double scratch[8][32];
    __shared__ int32_t pk[ENG_PRE_CAP];
    __shared__ double pv[ENG_PRE_CAP];
    __shared__ uint32_t pc[ENG_PRE_CAP];
    const int wid = threadIdx.x >> 5;
    const int64_t j = blockIdx.x;
    // row index: largest i with chunk_pre[i] <= j
    int64_t lo = 0, hi = nrows - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (chunk_pre[mid] <= j)
            lo = mid;
        else
            hi = mid - 1;
    }
    for (int t = threadIdx.x; t < ENG_PRE_CAP; t += blockDim.x) {
        pk[t] = EMPTY_KEY;
        pv[t] = 0.0;
        pc[t] = 0;
    }
    __syncthreads();
    const int64_t r = rows[lo];
    const int64_t f1r = fpre[r + 1];
    const int64_t cstart = fpre[r] + (j - chunk_pre[lo]) * ENG_GLOBAL_CHUNK;
    const int64_t cend = min(f1r, cstart + ENG_GLOBAL_CHUNK);
    const int64_t per = ENG_GLOBAL_CHUNK / 8;
    const int64_t a = cstart + wid * per;
    const int64_t b = min(cend, a + per);
    int32_t *keys = gkeys + tab_off[lo];
    double *vals = gvals + tab_off[lo];
    uint32_t *cnts = gcnts ? gcnts + tab_off[lo] : nullptr;
    const uint32_t cap = static_cast<uint32_t>(tab_cap[lo]);
    if (a < b) {
        auto cur = src.init(r, a);
        for (int64_t f = a; f < b; f += 32) {
            int32_t k;
            double w;
            bool valid;
            src.load(r, f, b, cur, k, w, valid);
            double sum;
            uint32_t cnt;
            if (warp_aggregate(k, w, valid, 0xffffffffu, scratch[wid], sum, cnt)) {
                uint32_t sl = hash_slot(k, ENG_PRE_CAP - 1);
                bool done = false;
                for (int p = 0; p < ENG_PRE_PROBES && !done; ++p) {
                    const int32_t old = atomicCAS(&pk[sl], EMPTY_KEY, k);
                    if (old == EMPTY_KEY || old == k) {
                        atomicAdd(&pv[sl], sum);
                        atomicAdd(&pc[sl], cnt);
                        done = true;
                    }
                    sl = (sl + 1) & (ENG_PRE_CAP - 1);
                }
                if (!done)
                    table_insert_n(keys, vals, cnts, cap, k, sum, cnt);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ENG_PRE_CAP; t += blockDim.x)
        if (pk[t] != EMPTY_KEY)
            table_insert_n(keys, vals, cnts, cap, pk[t], pv[t], pc[t]);
}

static __global__ void __launch_bounds__(512) k_eng_reduce_global_flush(const int64_t *fpre, const int32_t *rows,
                                                                 int64_t nrows, const int64_t *tab_off,
                                                                 const int64_t *tab_cap, const int32_t *gkeys,
                                                                 const double *gvals, const uint32_t *gcnts,
                                                                 int mode, EngineOut out) {
    __shared__ int32_t counter;
    const int wid = threadIdx.x >> 5, lane = lane_id();
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int64_t r = rows[i];
        const int64_t f0 = fpre[r];
        const int32_t *keys = gkeys + tab_off[i];
        const double *vals = gvals + tab_off[i];
        const uint32_t *cnts = gcnts ? gcnts + tab_off[i] : nullptr;
        const int64_t cap = tab_cap[i];
        if (threadIdx.x == 0)
            counter = 0;
        __syncthreads();
        for (int64_t s0 = wid * 32; s0 < cap; s0 += blockDim.x) {
            const int64_t s = s0 + lane;
            const bool has = s < cap && keys[s] != EMPTY_KEY;
            const int32_t pos = warp_append(&counter, has);
            if (has) {
                out.tkey[f0 + pos] = keys[s];
                out.tval[f0 + pos] = mode == DUP_ONE ? 1.0 : vals[s];
                if (out.flag && cnts && cnts[s] > 1 && !*out.flag)
                    *out.flag = 1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0)
            out.deg2[r] = counter;
        __syncthreads();
    }
    (void)lane;
}

// Chunked flush of the global tables: the tables of all big rows are one
// contiguous slot range; every block scans 8192 slots, finds each slot's row
// by binary search and appends its entries with a warp-aggregated atomic on
// the row's distinct counter (order is irrelevant: the sort phase follows).
constexpr int64_t ENG_FLUSH_CHUNK = 8192;

static __global__ void k_eng_global_zero(int64_t nb, const int32_t *rows, int64_t *deg2) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        deg2[rows[i]] = 0;
}

static __global__ void __launch_bounds__(256) k_eng_flush_chunked(const int64_t *fpre, const int32_t *rows, int64_t nb,
                                                                  const int64_t *tab_off, int64_t total,
                                                                  const int32_t *gkeys, const double *gvals,
                                                                  const uint32_t *gcnts, int mode, EngineOut out) {
    const int lane = lane_id();
    const int64_t begin = static_cast<int64_t>(blockIdx.x) * ENG_FLUSH_CHUNK;
    const int64_t end = min(total, begin + ENG_FLUSH_CHUNK);
    for (int64_t s0 = begin + (threadIdx.x & ~31); s0 < end; s0 += blockDim.x) {
        const int64_t s = s0 + lane;
        const bool has = s < end && gkeys[s] != EMPTY_KEY;
        int64_t i = -1;
        if (has) {
            int64_t lo = 0, hi = nb - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (tab_off[mid] <= s)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            i = lo;
        }
        const uint32_t hm = __ballot_sync(0xffffffffu, has);
        const uint32_t peers = __match_any_sync(0xffffffffu, i) & hm;
        int64_t base = 0;
        const int leader = __ffs(peers) - 1;
        const int64_t r = has ? rows[i] : 0;
        if (has && lane == leader)
            base = static_cast<int64_t>(atomicAdd(reinterpret_cast<unsigned long long *>(&out.deg2[r]),
                                                  static_cast<unsigned long long>(__popc(peers))));
        base = __shfl_sync(0xffffffffu, base, has ? leader : lane);
        if (has) {
            const int64_t pos = fpre[r] + base + __popc(peers & lanemask_lt());
            out.tkey[pos] = gkeys[s];
            out.tval[pos] = mode == DUP_ONE ? 1.0 : gvals[s];
            if (out.flag && gcnts && gcnts[s] > 1 && !*out.flag)
                *out.flag = 1;
        }
    }
}

// ---- sort kernels -----------------------------------------------------------

// rows of 33..512 distinct keys: one warp per row, bitonic sort in a
// per-warp smem slice (__syncwarp only)
constexpr int ENG_SORT_WARP_CAP = 512;

static __global__ void __launch_bounds__(256) k_eng_sort_warpsmem(const int64_t *fpre, const int32_t *rows,
                                                                  int64_t nrows, const int32_t *tkey,
                                                                  const double *tval, const int64_t *off2,
                                                                  int32_t *col, float *wout) {
    __shared__ int32_t sk_all[8][ENG_SORT_WARP_CAP];
    __shared__ float sv_all[8][ENG_SORT_WARP_CAP];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    int32_t *sk = sk_all[wid];
    float *sv = sv_all[wid];
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = gw; i < nrows; i += nw) {
        const int64_t r = rows[i];
        const int64_t s = fpre[r], L = off2[r + 1] - off2[r];
        int cap = 64;
        while (cap < L)
            cap <<= 1;
        for (int t = lane; t < cap; t += 32) {
            sk[t] = t < L ? tkey[s + t] : INT32_MAX;
            sv[t] = t < L ? static_cast<float>(tval[s + t]) : 0.0f;
        }
        __syncwarp();
        for (int kk = 2; kk <= cap; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int t = lane; t < cap; t += 32) {
                    const int p = t ^ j;
                    if (p > t) {
                        const bool up = (t & kk) == 0;
                        const int32_t a = sk[t], b = sk[p];
                        if ((a > b) == up) {
                            sk[t] = b;
                            sk[p] = a;
                            const float tv = sv[t];
                            sv[t] = sv[p];
                            sv[p] = tv;
                        }
                    }
                }
                __syncwarp();
            }
        }
        for (int t = lane; t < L; t += 32) {
            col[off2[r] + t] = sk[t];
            if (wout)
                wout[off2[r] + t] = sv[t];
        }
        __syncwarp();
    }
}

static __global__ void __launch_bounds__(256) k_eng_sort_warp(const int64_t *fpre, const int32_t *rows, int64_t nrows,
                                                       const int32_t *tkey, const double *tval,
                                                       const int64_t *off2, int32_t *col, float *wout) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = gw; i < nrows; i += nw) {
        const int64_t r = rows[i];
        const int64_t s = fpre[r], L = off2[r + 1] - off2[r];
        int32_t k = lane < L ? tkey[s + lane] : INT32_MAX;
        double v = lane < L ? tval[s + lane] : 0.0;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                const int32_t pk = __shfl_xor_sync(0xffffffffu, k, j);
                const double pv = __shfl_xor_sync(0xffffffffu, v, j);
                const bool up = (lane & kk) == 0;
                const bool lower = (lane & j) == 0;
                const bool take = (lower == up) ? (pk < k) : (pk > k);
                if (take) {
                    k = pk;
                    v = pv;
                }
            }
        }
        if (lane < L) {
            col[off2[r] + lane] = k;
            if (wout)
                wout[off2[r] + lane] = static_cast<float>(v);
        }
    }
}

static __global__ void __launch_bounds__(512) k_eng_sort_block(const int64_t *fpre, const int32_t *rows, int64_t nrows,
                                                        const int32_t *tkey, const double *tval,
                                                        const int64_t *off2, int32_t *col, float *wout) {
    extern __shared__ unsigned char smem_raw[];
    double *sv = reinterpret_cast<double *>(smem_raw);
    int32_t *sk = reinterpret_cast<int32_t *>(sv + ENG_SORT_BLOCK);
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int64_t r = rows[i];
        const int64_t s = fpre[r], L = off2[r + 1] - off2[r];
        int cap = 64;
        while (cap < L)
            cap <<= 1;
        for (int t = threadIdx.x; t < cap; t += blockDim.x) {
            sk[t] = t < L ? tkey[s + t] : INT32_MAX;
            sv[t] = t < L ? tval[s + t] : 0.0;
        }
        __syncthreads();
        for (int kk = 2; kk <= cap; kk <<= 1) {
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int t = threadIdx.x; t < cap; t += blockDim.x) {
                    const int p = t ^ j;
                    if (p > t) {
                        const bool up = (t & kk) == 0;
                        const int32_t a = sk[t], b = sk[p];
                        if ((a > b) == up) {
                            sk[t] = b;
                            sk[p] = a;
                            const double tv = sv[t];
                            sv[t] = sv[p];
                            sv[p] = tv;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int t = threadIdx.x; t < L; t += blockDim.x) {
            col[off2[r] + t] = sk[t];
            if (wout)
                wout[off2[r] + t] = static_cast<float>(sv[t]);
        }
        __syncthreads();
    }
}

// Block-local stable LSD radix sort (8-bit digits) of one big row per block.
// Ping-pongs between (k0, v0) at fpre[r] and (k1, v1); writes the result.
static __global__ void __launch_bounds__(1024) k_eng_sort_radix(const int64_t *fpre, const int32_t *rows, int64_t nrows,
                                                         int32_t *k0, double *v0, int32_t *k1, double *v1,
                                                         int key_bits, const int64_t *off2, int32_t *col,
                                                         float *wout) {
    __shared__ int32_t hist[256];
    __shared__ int32_t dbase[256];
    __shared__ int32_t tcount[256];
    __shared__ int32_t wcnt[32][256];
    const int tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        const int64_t r = rows[i];
        const int64_t s = fpre[r], L = off2[r + 1] - off2[r];
        int32_t *ka = k0 + s, *kb = k1 + s;
        double *va = v0 + s, *vb = v1 + s;
        for (int shift = 0; shift < key_bits; shift += 8) {
            if (tid < 256)
                hist[tid] = 0;
            __syncthreads();
            for (int64_t t = tid; t < L; t += blockDim.x)
                atomicAdd(&hist[(static_cast<uint32_t>(ka[t]) >> shift) & 255], 1);
            __syncthreads();
            if (tid == 0) {
                int32_t run = 0;
                for (int d = 0; d < 256; ++d) {
                    dbase[d] = run;
                    run += hist[d];
                }
            }
            for (int q = tid; q < 32 * 256; q += blockDim.x)
                (&wcnt[0][0])[q] = 0;
            __syncthreads();
            for (int64_t t0 = 0; t0 < L; t0 += blockDim.x) {
                const int64_t t = t0 + tid;
                const bool valid = t < L;
                const int32_t kk = valid ? ka[t] : 0;
                const double vv = valid ? va[t] : 0.0;
                const int d = valid ? static_cast<int>((static_cast<uint32_t>(kk) >> shift) & 255) : 0;
                const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
                const uint32_t peers = __match_any_sync(0xffffffffu, d) & vmask;
                const int rank = __popc(peers & lanemask_lt());
                if (valid && rank == 0)
                    wcnt[wid][d] = __popc(peers);
                __syncthreads();
                if (tid < 256) {
                    int32_t run = 0;
                    for (int w2 = 0; w2 < 32; ++w2) {
                        const int32_t c = wcnt[w2][tid];
                        wcnt[w2][tid] = run;
                        run += c;
                    }
                    tcount[tid] = run;
                }
                __syncthreads();
                if (valid) {
                    const int32_t pos = dbase[d] + wcnt[wid][d] + rank;
                    kb[pos] = kk;
                    vb[pos] = vv;
                }
                __syncthreads();
                if (tid < 256)
                    dbase[tid] += tcount[tid];
                for (int q = tid; q < 32 * 256; q += blockDim.x)
                    (&wcnt[0][0])[q] = 0;
                __syncthreads();
            }
            int32_t *tk = ka;
            ka = kb;
            kb = tk;
            double *tv = va;
            va = vb;
            vb = tv;
        }
        for (int64_t t = tid; t < L; t += blockDim.x) {
            col[off2[r] + t] = ka[t];
            if (wout)
                wout[off2[r] + t] = static_cast<float>(va[t]);
        }
        __syncthreads();
    }
}

// Unsorted output (contraction inside the detectors, where row order is
// irrelevant): the reduced rows are copied as they are.  Blocks own
// ENG_COPY_CHUNK consecutive output entries; each thread finds its row by a
// binary search over the block's row range.
constexpr int64_t ENG_COPY_CHUNK = 4096;

static __global__ void __launch_bounds__(256) k_eng_copy_rows(int64_t nrows, const int64_t *fpre, const int64_t *off2,
                                                              int64_t D2, const int32_t *tkey, const double *tval,
                                                              int32_t *col, float *wout) {
    __shared__ int64_t rng[2];
    const int64_t begin = static_cast<int64_t>(blockIdx.x) * ENG_COPY_CHUNK;
    const int64_t end = min(D2, begin + ENG_COPY_CHUNK);
    if (threadIdx.x < 2) {
        // last row with off2[row] <= (begin | end - 1)
        const int64_t target = threadIdx.x == 0 ? begin : end - 1;
        int64_t lo = 0, hi = nrows - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (off2[mid] <= target)
                lo = mid;
            else
                hi = mid - 1;
        }
        rng[threadIdx.x] = lo;
    }
    __syncthreads();
    for (int64_t i = begin + threadIdx.x; i < end; i += blockDim.x) {
        int64_t lo = rng[0], hi = rng[1];
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (off2[mid] <= i)
                lo = mid;
            else
                hi = mid - 1;
        }
        const int64_t src = fpre[lo] + (i - off2[lo]);
        col[i] = tkey[src];
        if (wout)
            wout[i] = static_cast<float>(tval[src]);
    }
}

// ---- row classification ------------------------------------------------------

// classify rows by source length (reduce) or distinct length (sort)
static __global__ void k_eng_classify(int64_t nrows, const int64_t *len_pre, const int64_t *len_direct, int64_t t0,
                               int64_t t1, int64_t t2, int32_t *l0, int32_t *l1, int32_t *l2, int32_t *l3,
                               int32_t *counts) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool in = r < nrows;
    int64_t L = 0;
    if (in)
        L = len_pre ? len_pre[r + 1] - len_pre[r] : len_direct[r];
    int cls = -1;
    if (in && L > 0)
        cls = L <= t0 ? 0 : (L <= t1 ? 1 : (L <= t2 ? 2 : 3));
    int32_t *lists[4] = {l0, l1, l2, l3};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int32_t pos = warp_append(&counts[c], cls == c);
        if (cls == c)
            lists[c][pos] = static_cast<int32_t>(r);
    }
}

static __global__ void k_eng_zero_rows(int64_t nrows, const int64_t *fpre, int64_t *deg2) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < nrows && fpre[r + 1] == fpre[r])
        deg2[r] = 0;
}

struct CapGen {
    const int32_t *rows;
    const int64_t *fpre;
    int64_t key_bound;
    __device__ int64_t operator()(int64_t i) const {
        const int64_t r = rows[i];
        const int64_t F = fpre[r + 1] - fpre[r];
        const int64_t need = 2 * (F < key_bound ? F : key_bound);
        return need < 64 ? 64 : need;  // load factor <= 1/2, no power-of-two rounding
    }
};
struct ChunkGen {
    const int32_t *rows;
    const int64_t *fpre;
    __device__ int64_t operator()(int64_t i) const {
        const int64_t r = rows[i];
        return (fpre[r + 1] - fpre[r] + ENG_GLOBAL_CHUNK - 1) / ENG_GLOBAL_CHUNK;
    }
};
struct DiffGen {
    const int64_t *a;  // a[i+1] - a[i] style not used; deg2 directly
    __device__ int64_t operator()(int64_t i) const { return a[i]; }
};
struct CapFromPre {
    const int64_t *pre;  // exclusive prefix with total at [n]
    __device__ int64_t operator()(int64_t i) const { return pre[i + 1] - pre[i]; }
};

static __global__ void k_cap_from_prefix(int64_t m, const int64_t *pre, const int64_t *total, int64_t *cap) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m)
        cap[i] = (i + 1 < m ? pre[i + 1] : *total) - pre[i];
}

// Runs the engine.  fpre: device [nrows+1] source prefix.  Produces off2
// ([nrows+1]), col ([D2]) and w ([D2], if want_w; DUP_SUM turns want_w on
// when duplicates were merged).  Returns D2.  *dup (host) = duplicates seen.
template <class Src>
int64_t run_row_engine(cd_ctx *ctx, const Src &src, int64_t nrows, const int64_t *fpre, int64_t F_total,
                       int64_t key_bound, DupMode mode, bool &want_w, DBuf<int64_t> &off2, DBuf<int32_t> &col,
                       DBuf<float> &wout, bool *dup, const char *family, bool sort_rows = true) {
    // per-phase profiler families "<family>.<phase>" (cd_ctx_kernel_stats sums them)
    const std::string fam(family);
    const std::string f_cls = fam + ".classify", f_red = fam + ".reduce", f_glob = fam + ".reduce_global",
                      f_sort = fam + ".sort", f_radix = fam + ".radix";
    off2.alloc(ctx, nrows + 1);
    if (nrows == 0) {
        off2.zero();
        col.alloc(ctx, 0);
        wout.alloc(ctx, 0);
        if (dup)
            *dup = false;
        return 0;
    }
    DBuf<int32_t> tkey(ctx, std::max<int64_t>(F_total, 1));
    DBuf<double> tval(ctx, std::max<int64_t>(F_total, 1));
    DBuf<int64_t> deg2(ctx, nrows);
    DBuf<int32_t> lists(ctx, 4 * nrows);
    DBuf<int32_t> counts(ctx, 8);
    DBuf<int64_t> flag(ctx, 1);
    flag.zero();
    counts.zero();
    const int cls_blocks = grid_for(nrows, 256, INT32_MAX);
    int32_t *L[4] = {lists.p, lists.p + nrows, lists.p + 2 * nrows, lists.p + 3 * nrows};
    CD_LAUNCH(ctx, f_cls.c_str(), k_eng_zero_rows, cls_blocks, 256, 0, nrows, fpre, deg2.p);
    CD_LAUNCH(ctx, f_cls.c_str(), k_eng_classify, cls_blocks, 256, 0, nrows, fpre, static_cast<const int64_t *>(nullptr),
              int64_t(32), int64_t(ENG_WARP_F), int64_t(ENG_BLOCK_F), L[0], L[1], L[2], L[3], counts.p);
    int32_t hc[8];
    CD_CUDA(cudaMemcpyAsync(hc, counts.p, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    // duplicates matter only for the builder (error / unweighted merge); in a
    // contraction every row is full of them
    const bool track = mode == DUP_ERROR || (mode == DUP_SUM && !want_w);
    EngineOut eo{tkey.p, tval.p, deg2.p, track ? flag.p : nullptr};
    const int sms = ctx->num_sms;
    if (hc[0])
        CD_LAUNCH(ctx, f_red.c_str(), (k_eng_reduce_direct<Src>), grid_for(hc[0], 8, sms * 8), 256, 0, src, fpre, L[0],
                  int64_t(hc[0]), int(mode), eo);
    // contraction (no duplicate tracking) drops the per-slot counts: 25 % less
    // shared memory per table, more resident warps / blocks
    if (hc[1]) {
        if (track)
            CD_LAUNCH(ctx, f_red.c_str(), (k_eng_reduce_warp<Src, true>), grid_for(hc[1], 4, sms * 8), 128, 0, src,
                      fpre, L[1], int64_t(hc[1]), key_bound, int(mode), eo);
        else
            CD_LAUNCH(ctx, f_red.c_str(), (k_eng_reduce_warp<Src, false>), grid_for(hc[1], 4, sms * 8), 128, 0, src,
                      fpre, L[1], int64_t(hc[1]), key_bound, int(mode), eo);
    }
    if (hc[2]) {
        constexpr int CAP_S = 2048, CAP_L = 2 * ENG_BLOCK_F;
        const size_t slot = sizeof(double) + sizeof(int32_t) + (track ? sizeof(uint32_t) : 0);
        const size_t smem_s = size_t(CAP_S) * slot, smem = size_t(CAP_L) * slot;
        auto launch = [&](auto ks, auto kl) {
            CD_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_s)));
            CD_CUDA(cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            CD_LAUNCH(ctx, f_red.c_str(), ks, grid_for(hc[2], 1, sms * 4), 512, smem_s, src, fpre, L[2],
                      int64_t(hc[2]), key_bound, int(mode), eo, int64_t(0), int64_t(CAP_S / 2));
            CD_LAUNCH(ctx, f_red.c_str(), kl, grid_for(hc[2], 1, sms * 2), 512, smem, src, fpre, L[2], int64_t(hc[2]),
                      key_bound, int(mode), eo, int64_t(CAP_S / 2), int64_t(ENG_BLOCK_F));
        };
        if (track)
            launch(k_eng_reduce_block<Src, CAP_S, true>, k_eng_reduce_block<Src, CAP_L, true>);
        else
            launch(k_eng_reduce_block<Src, CAP_S, false>, k_eng_reduce_block<Src, CAP_L, false>);
    }
    if (hc[3]) {
        const int64_t nb = hc[3];
        DBuf<int64_t> tab_off(ctx, nb + 1), tab_cap(ctx, nb), chunk_pre(ctx, nb + 1);
        DBuf<int64_t> totals(ctx, 2);
        exclusive_scan<int64_t>(ctx, nb, CapGen{L[3], fpre, key_bound}, tab_off.p, totals.p);
        exclusive_scan<int64_t>(ctx, nb, ChunkGen{L[3], fpre}, chunk_pre.p, totals.p + 1);
        CD_LAUNCH(ctx, f_glob.c_str(), k_cap_from_prefix, grid_for(nb, 256, INT32_MAX), 256, 0, nb,
                  static_cast<const int64_t *>(tab_off.p), static_cast<const int64_t *>(totals.p), tab_cap.p);
        int64_t ht[2];
        CD_CUDA(cudaMemcpyAsync(ht, totals.p, sizeof(ht), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        DBuf<int32_t> gk(ctx, ht[0]);
        DBuf<double> gv(ctx, ht[0]);
        DBuf<uint32_t> gc(ctx, track ? ht[0] : 0);  // duplicate counts only when tracked
        gk.fill_bytes(0xff);
        gv.zero();
        if (track)
            gc.zero();
        CD_LAUNCH(ctx, f_glob.c_str(), (k_eng_reduce_global_insert<Src>), static_cast<int>(ht[1]), 256, 0, src, fpre, L[3],
                  nb, static_cast<const int64_t *>(chunk_pre.p), static_cast<const int64_t *>(tab_off.p),
                  static_cast<const int64_t *>(tab_cap.p), gk.p, gv.p, gc.p);
        CD_LAUNCH(ctx, f_glob.c_str(), k_eng_global_zero, grid_for(nb, 256, sms * 4), 256, 0, nb,
                  static_cast<const int32_t *>(L[3]), deg2.p);
        CD_LAUNCH(ctx, f_glob.c_str(), k_eng_flush_chunked, static_cast<int>((ht[0] + ENG_FLUSH_CHUNK - 1) / ENG_FLUSH_CHUNK),
                  256, 0, fpre, static_cast<const int32_t *>(L[3]), nb, static_cast<const int64_t *>(tab_off.p), ht[0],
                  static_cast<const int32_t *>(gk.p), static_cast<const double *>(gv.p),
                  static_cast<const uint32_t *>(gc.p), int(mode), eo);
    }
    // offsets of the reduced rows
    exclusive_scan<int64_t>(ctx, nrows, ArrayGen<int64_t>{deg2.p}, off2.p, off2.p + nrows);
    int64_t D2 = 0, hflag = 0;
    CD_CUDA(cudaMemcpyAsync(&D2, off2.p + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&hflag, flag.p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (dup)
        *dup = hflag != 0;
    if (mode == DUP_ERROR && hflag)
        return D2;
    // merged duplicates of an unweighted input carry summed weights
    if (mode == DUP_SUM && hflag)
        want_w = true;
    col.alloc(ctx, std::max<int64_t>(D2, 1));
    if (want_w)
        wout.alloc(ctx, std::max<int64_t>(D2, 1));
    else
        wout.alloc(ctx, 0);
    if (!sort_rows) {
        if (D2 > 0)
            CD_LAUNCH(ctx, f_sort.c_str(), k_eng_copy_rows, static_cast<int>((D2 + ENG_COPY_CHUNK - 1) / ENG_COPY_CHUNK),
                      256, 0, nrows, fpre, static_cast<const int64_t *>(off2.p), D2,
                      static_cast<const int32_t *>(tkey.p), static_cast<const double *>(tval.p), col.p,
                      want_w ? wout.p : static_cast<float *>(nullptr));
        return D2;
    }
    // sort phase: classify by distinct length
    counts.zero();
    CD_LAUNCH(ctx, f_cls.c_str(), k_eng_classify, cls_blocks, 256, 0, nrows, static_cast<const int64_t *>(nullptr),
              static_cast<const int64_t *>(deg2.p), int64_t(32), int64_t(ENG_SORT_WARP_CAP), int64_t(ENG_SORT_BLOCK),
              L[0], L[1], L[2], L[3], counts.p);
    CD_CUDA(cudaMemcpyAsync(hc, counts.p, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    float *wp = want_w ? wout.p : nullptr;
    if (hc[0])
        CD_LAUNCH(ctx, f_sort.c_str(), k_eng_sort_warp, grid_for(hc[0], 8, sms * 8), 256, 0, fpre, L[0], int64_t(hc[0]),
                  static_cast<const int32_t *>(tkey.p), static_cast<const double *>(tval.p),
                  static_cast<const int64_t *>(off2.p), col.p, wp);
    if (hc[1])
        CD_LAUNCH(ctx, f_sort.c_str(), k_eng_sort_warpsmem, grid_for(hc[1], 8, sms * 8), 256, 0, fpre, L[1], int64_t(hc[1]),
                  static_cast<const int32_t *>(tkey.p), static_cast<const double *>(tval.p),
                  static_cast<const int64_t *>(off2.p), col.p, wp);
    if (hc[2]) {
        const size_t smem = size_t(ENG_SORT_BLOCK) * (sizeof(double) + sizeof(int32_t));
        CD_CUDA(cudaFuncSetAttribute(k_eng_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        CD_LAUNCH(ctx, f_sort.c_str(), k_eng_sort_block, grid_for(hc[2], 1, sms * 2), 512, smem, fpre, L[2], int64_t(hc[2]),
                  static_cast<const int32_t *>(tkey.p), static_cast<const double *>(tval.p),
                  static_cast<const int64_t *>(off2.p), col.p, wp);
    }
    if (hc[3]) {
        DBuf<int32_t> k1(ctx, std::max<int64_t>(F_total, 1));
        DBuf<double> v1(ctx, std::max<int64_t>(F_total, 1));
        int bits = 1;
        while ((int64_t(1) << bits) < key_bound && bits < 31)
            ++bits;
        bits = (bits + 7) / 8 * 8;
        CD_LAUNCH(ctx, f_radix.c_str(), k_eng_sort_radix, grid_for(hc[3], 1, sms), 1024, 0, fpre, L[3], int64_t(hc[3]), tkey.p,
                  tval.p, k1.p, v1.p, bits, static_cast<const int64_t *>(off2.p), col.p, wp);
    }
    return D2;
}

}  // namespace cdk
