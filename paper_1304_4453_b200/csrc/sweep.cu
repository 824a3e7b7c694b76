// sweep.cu -- degree-tiered evaluation kernels shared by PLP and PLM.
//
//   PLP (H/plp.hpp:111-126): tally neighbour labels incl. the self-loop,
//        best = argmax weight, ties -> smallest label.
//   PLM (H/louvain.hpp:95-120): tally neighbour communities excl. the
//        self-loop, delta(d) = (aff[d]-w_c)/w(E) + g(vol_c - vols[d])vol_u/(2w(E)^2),
//        best = argmax delta with ties -> smallest d, move iff delta > 0.
//
// Tiers (graph.cuh): G8/G16/G32 one pass with __match_any_sync, lanes grouped
// 8/16/32 per node; WARP per-warp smem hash; BLOCK / BLOCK2 / BLOCK3 block
// smem hash (2048 / 8192 / 16384 slots); CLUSTER one 4-CTA cluster per node
// with the hash in distributed shared memory; HUB a hash-partitioned
// multi-block tally.  Every table lists its claimed slots, so the candidate
// scan visits only distinct labels and the table cleans up after each node.
// Integer tallies are exact in uint32, general weights in fp64, so the
// decision does not depend on the summation order and equals the
// sequential reference's (tests/test_gpu_tiers.py).
//
// Selection (bucket of this sub-sweep, active flag) is inline: each warp
// loads up to 32 candidates of its tier's static list and ballots the
// selected ones; block tiers select 256 candidates cooperatively; short tier
// lists are pre-bucketed once per pass (k_prebucket_*).  Small coarse levels run
// the whole move phase in one cooperative kernel (k_small_move).
#include "sweep.cuh"

#include <atomic>

#include <cooperative_groups.h>

#include <cmath>
#include <chrono>
#include <cstdio>
#include <map>
#include <mutex>

#include "comm.cuh"
#include "scan.cuh"

namespace cdk {

struct SweepParams {
    const int64_t *off;
    const int32_t *col;
    const float *w;
    const double *vol;
    const int32_t *z;
    uint8_t *active;
    int2 *chg;  // margin mode (PLP, count tallies): (changes, margin) per node; see evaluate_again
    const double *vols;
    const int32_t *csize;
    double gamma, inv_total, inv_sq2;
    int guard;
    const unsigned long long *keyp;  // bucket key of the current pass (device)
    int bucket, buckets;
    const int32_t *tlist;
    // this rank's slice [tbeg[t], tend[t]) of each tier list (whole lists on
    // one device); nodes outside [own_lo, own_hi) are never evaluated
    int64_t tbeg[NUM_TIERS], tend[NUM_TIERS];
    int32_t own_lo, own_hi;
    // pre-bucketed tiers (bit t of pre_mask): once per pass k_prebucket_*
    // partitions the tier's segment by bucket into blist (same offsets as
    // tlist), bucket b at [boff[9t + b], boff[9t + b + 1]) of the segment
    uint32_t pre_mask;
    int32_t pre_tiers[NUM_TIERS], n_pre;
    int32_t *blist;
    int32_t *boff;
    int32_t *pb_cnt, *pb_cur;  // k_prebucket_*: per (tier, bucket) counts and cursors
    int32_t *mv_count;  // moves of this bucket
    int2 *mv;           // (node, label) of this bucket's moves
    int32_t *dense_best;
    double *dense_gain;
    unsigned long long *stats;
    long long *gain_fx;  // PLM: sum of the movers' Δ in units of 2^-44 (fixed point: order-free)
    // hub tier (hash-partitioned tally, graph.cuh)
    const int32_t *hubs;
    const int32_t *chunk_hub;
    const int32_t *chunk_part;
    const int32_t *hub_pbits;
    const int64_t *hub_pbase;
    const int32_t *part_hub;
    int32_t *hp_cnt, *hp_cur;
    const int64_t *hp_start;
    int32_t *hp_key;
    double *hp_val;
    double *hp_best_val;
    double *hp_second;
    int32_t *hp_best_key;
    int32_t *hp_flag;
    double *hub_aux;
    int64_t *hp_scan;  // host-side scan scratch of hp_cnt (never read by kernels)
    int32_t *st_key;   // count pass -> scatter: staged pairs (chunk-major) and their counts
    double *st_val;
    int32_t *chunk_np;
    int64_t n_hubs, n_parts;
};

template <int VC>
using TallyT = typename std::conditional<VC == VC_REAL, double, unsigned int>::type;

// Row entries are streamed once per sub-sweep: load them evict-first so the
// gathered arrays (labels, volumes, per-node state: ~200 MB at C3, most of
// the 126 MB L2) stay cached across the sweep
__device__ __forceinline__ int32_t col_at(const SweepParams &P, int64_t f) { return __ldcs(P.col + f); }


constexpr int SW_ILP = 4;  // independent loads per lane per round

__device__ __forceinline__ double plm_delta(double aff_d, double w_c, double vol_c, double vols_d, double vol_u,
                                            const SweepParams &P) {
    // (aff[d] - w_c) * inv_total + gamma * (vol_c - vols[d]) * vol_u * inv_sq2
    // evaluated exactly as the reference's left-to-right double expression
    // (no FMA contraction): H/louvain.hpp:111-112.
    const double t1 = __dmul_rn(__dsub_rn(aff_d, w_c), P.inv_total);
    const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(P.gamma, __dsub_rn(vol_c, vols_d)), vol_u), P.inv_sq2);
    return __dadd_rn(t1, t2);
}

__device__ __forceinline__ bool better(double a, int32_t ka, double b, int32_t kb) {
    return a > b || (a == b && ka < kb);
}

// Own-label bypass: entries labelled like the evaluated node itself never go
// into the tally table.  PLM sums them into w(u, C) (the own community is no
// candidate, H/louvain.hpp:105-113); PLP with integer tallies counts them in a
// register and offers the own label as one more candidate after the scan
// (exact: integer sums are order-free; fp64 PLP tallies keep the lane-order
// combine).  Converged neighbourhoods are mostly own-labelled, so most
// shared-memory atomics of the later passes disappear.
template <int MODE, int VC>
__host__ __device__ constexpr bool own_bypass() {
    return MODE == MODE_PLM || VC != VC_REAL;
}

// Group argmax (ties to the smaller key) over WIDTH-lane groups: the value
// as an order-preserving 64-bit key, reduced by redux.sync on its halves, then
// the smallest key among the lanes holding the maximum -- three instructions
// in place of log2(WIDTH) rounds of two fp64 and one int shuffles
__device__ __forceinline__ unsigned long long f64_order_key(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v == 0.0 ? 0.0 : v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double f64_from_order_key(unsigned long long key) {
    return __longlong_as_double(static_cast<long long>((key >> 63) ? (key & 0x7fffffffffffffffull) : ~key));
}

template <int WIDTH>
__device__ __forceinline__ void argmax_redux(double &v, int32_t &k) {
    const uint32_t mask =
        WIDTH == 32 ? 0xffffffffu : (((1u << WIDTH) - 1u) << ((threadIdx.x & 31) & ~(WIDTH - 1)));
    const unsigned long long key = f64_order_key(v);
    const uint32_t hi = static_cast<uint32_t>(key >> 32), lo = static_cast<uint32_t>(key);
    const uint32_t mh = __reduce_max_sync(mask, hi);
    const uint32_t ml = __reduce_max_sync(mask, hi == mh ? lo : 0u);
    k = static_cast<int32_t>(__reduce_min_sync(mask, (hi == mh && lo == ml) ? k : INT32_MAX));
    v = f64_from_order_key((static_cast<unsigned long long>(mh) << 32) | ml);
}

template <int WIDTH>
__device__ __forceinline__ void argmax_xor(double &v, int32_t &k) {
#pragma unroll
    for (int o = WIDTH / 2; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int32_t ok = __shfl_xor_sync(0xffffffffu, k, o);
        if (better(ov, ok, v, k)) {
            v = ov;
            k = ok;
        }
    }
}

// PLM: the redux form (C3 PLM -1.5 %, C2 -1.8 %); PLP keeps the shuffles (its
// kernels grew registers with the redux form: C3 PLP +13 %)
template <int MODE, int WIDTH>
__device__ __forceinline__ void argmax_m(double &v, int32_t &k) {
    if (MODE == MODE_PLM)
        argmax_redux<WIDTH>(v, k);
    else
        argmax_xor<WIDTH>(v, k);
}

// argmax that also keeps the runner-up's value s (over all other keys)
template <int WIDTH>
__device__ __forceinline__ void argmax2_xor(double &v, int32_t &k, double &s) {
#pragma unroll
    for (int o = WIDTH / 2; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int32_t ok = __shfl_xor_sync(0xffffffffu, k, o);
        const double os = __shfl_xor_sync(0xffffffffu, s, o);
        if (better(ov, ok, v, k)) {
            s = fmax(os, v);
            v = ov;
            k = ok;
        } else {
            s = fmax(s, ov);
        }
    }
}

__device__ __forceinline__ void keep2(double val, int32_t key, double &v, int32_t &k, double &s) {
    if (better(val, key, v, k)) {
        s = fmax(s, v);
        v = val;
        k = key;
    } else {
        s = fmax(s, val);
    }
}

template <int WIDTH>
__device__ __forceinline__ double sum_xor(double v) {
#pragma unroll
    for (int o = WIDTH / 2; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Group aggregation: returns leader flag and the group's count / weight sum
// (weights summed in lane order by the leader).
template <int VC>
__device__ __forceinline__ bool aggregate(int32_t key, double w, bool valid, uint32_t gmask, double *scratch,
                                          double &val) {
    const int lane = lane_id();
    const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
    const uint32_t peers = __match_any_sync(0xffffffffu, key) & vmask & gmask;
    const bool leader = valid && ((__ffs(peers) - 1) == lane);
    if (VC != VC_COUNT) {
        scratch[lane] = w;
        __syncwarp();
        double s = 0.0;
        if (leader)
            for (uint32_t m = peers; m; m &= m - 1)
                s += scratch[__ffs(m) - 1];
        __syncwarp();
        val = s;
    } else {
        val = static_cast<double>(__popc(peers));
    }
    return leader;
}

// insert; true if this call claimed a new slot for `key` (*slot = its index)
template <class V>
__device__ __forceinline__ bool tinsert_claim(int32_t *keys, V *vals, uint32_t mask, int32_t key, V w,
                                              uint32_t *slot) {
    uint32_t s = hash_slot(key, mask);
    while (true) {
        const int32_t old = atomicCAS(&keys[s], EMPTY_KEY, key);
        if (old == EMPTY_KEY || old == key) {
            atomicAdd(&vals[s], w);
            *slot = s;
            return old == EMPTY_KEY;
        }
        s = (s + 1) & mask;
    }
}

// Count tallies (unweighted graphs): an empty slot already holds 1, so the
// entry that claims a slot needs no add -- one shared-memory atomic per
// distinct label instead of two (a shared atomic costs one L1 wavefront per
// lane; tools/microbench/tally_bench.cu).  Other tallies start at 0.
template <int VC>
__device__ __forceinline__ TallyT<VC> tally_empty() {
    return VC == VC_COUNT ? TallyT<VC>(1) : TallyT<VC>(0);
}

// insert one entry of weight w (1 for count tallies); true if it claimed the
// key's slot (*slot = its index)
template <int VC>
__device__ __forceinline__ bool tinsert_entry(int32_t *keys, TallyT<VC> *vals, uint32_t mask, int32_t key,
                                              TallyT<VC> w, uint32_t *slot) {
    if (VC != VC_COUNT)
        return tinsert_claim<TallyT<VC>>(keys, vals, mask, key, w, slot);
    uint32_t s = hash_slot(key, mask);
    while (true) {
        const int32_t old = atomicCAS(&keys[s], EMPTY_KEY, key);
        if (old == EMPTY_KEY) {
            *slot = s;
            return true;
        }
        if (old == key) {
            atomicAdd(&vals[s], TallyT<VC>(1));
            *slot = s;
            return false;
        }
        s = (s + 1) & mask;
    }
}

// insert `cnt` equal entries (a match_any group) into a count table
__device__ __forceinline__ bool tinsert_count_n(int32_t *keys, unsigned int *vals, uint32_t mask, int32_t key,
                                                unsigned int cnt, uint32_t *slot) {
    uint32_t s = hash_slot(key, mask);
    while (true) {
        const int32_t old = atomicCAS(&keys[s], EMPTY_KEY, key);
        if (old == EMPTY_KEY || old == key) {
            const unsigned int add = old == EMPTY_KEY ? cnt - 1u : cnt;  // an empty slot holds 1
            if (add)
                atomicAdd(&vals[s], add);
            *slot = s;
            return old == EMPTY_KEY;
        }
        s = (s + 1) & mask;
    }
}

template <int VC>
__device__ __forceinline__ double load_w(const SweepParams &P, int64_t f, bool valid) {
    return (VC != VC_COUNT && valid) ? static_cast<double>(P.w[f]) : 1.0;
}

// Margin-pruned active set (PLP, count tallies).  At its last evaluation u's
// best label b led every other label by margin = T(b) - max_{l != b} T(l)
// (T = neighbour label counts incl. the self-loop, H/plp.hpp:112-124); since
// then chg[u] entries of its row changed label.  Each change moves one count
// from one label to another, so b still wins -- and u, already labelled b,
// would not move -- while 2 * chg < margin: evaluating it is skipped
// (chg == 0 is the reference's inactive node, H/plp.hpp:131-132).  Labels,
// update counts and iterations are exactly those of the flag rule.
constexpr int32_t CHG_ALL = 0x20202020;  // "changed beyond counting": evaluate (a byte fill)

__device__ __forceinline__ bool evaluate_again(const SweepParams &P, int32_t u) {
    const int2 cm = P.chg[u];  // one 8-byte load
    return cm.x > 0 && 2 * cm.x >= cm.y;
}

__device__ __forceinline__ bool is_active(const SweepParams &P, int32_t u) {
    if (P.chg)
        return evaluate_again(P, u);
    return !P.active || P.active[u];
}

__device__ __forceinline__ bool selected(const SweepParams &P, unsigned long long key, int32_t u) {
    if (u < P.own_lo || u >= P.own_hi)
        return false;
    if (P.buckets > 1 && bucket_of(key, u, P.buckets) != P.bucket)
        return false;
    return is_active(P, u);
}

__device__ __forceinline__ unsigned long long load_key(const SweepParams &P) {
    return P.buckets > 1 ? *P.keyp : 0ULL;
}

// candidates of tier t in this sub-sweep: a pre-bucketed tier lists exactly
// the bucket's nodes (only the active flag is left to test)
__device__ __forceinline__ bool tier_range(const SweepParams &P, int t, const int32_t *&list, int64_t &count) {
    if ((P.pre_mask >> t) & 1u) {
        const int32_t *bo = P.boff + 9 * t;
        list = P.blist + P.tbeg[t] + bo[P.bucket];
        count = bo[P.bucket + 1] - bo[P.bucket];
        return true;
    }
    list = P.tlist + P.tbeg[t];
    count = P.tend[t] - P.tbeg[t];
    return false;
}

__device__ __forceinline__ bool selected_in(const SweepParams &P, unsigned long long key, int32_t u, bool pre) {
    return pre ? is_active(P, u) : selected(P, key, u);
}

// Once per pass: each pre-bucketed tier segment partitioned by bucket, on
// every SM (count, offsets, scatter).  Order within a bucket is irrelevant
// (a sub-sweep's decisions read frozen labels).  One block per tier took
// 79 us per pass at C3, serial at every pass's start.
constexpr int PB_BLOCKS = 16;

__global__ void __launch_bounds__(256) k_prebucket_count(SweepParams P) {
    const int t = P.pre_tiers[blockIdx.y];
    const int32_t *list = P.tlist + P.tbeg[t];
    const int64_t count = P.tend[t] - P.tbeg[t];
    const unsigned long long key = *P.keyp;
    __shared__ int c[8];
    if (threadIdx.x < 8)
        c[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(&c[bucket_of(key, list[i], P.buckets)], 1);
    __syncthreads();
    if (threadIdx.x < P.buckets && c[threadIdx.x])
        atomicAdd(&P.pb_cnt[9 * t + threadIdx.x], c[threadIdx.x]);
}

__global__ void k_prebucket_offsets(SweepParams P) {
    if (static_cast<int>(threadIdx.x) >= P.n_pre)
        return;
    const int t = P.pre_tiers[threadIdx.x];
    int run = 0;
    for (int b = 0; b < P.buckets; ++b) {
        P.boff[9 * t + b] = run;
        P.pb_cur[9 * t + b] = run;
        run += P.pb_cnt[9 * t + b];
        P.pb_cnt[9 * t + b] = 0;  // ready for the next pass
    }
    P.boff[9 * t + P.buckets] = run;
}

__global__ void __launch_bounds__(256) k_prebucket_scatter(SweepParams P) {
    const int t = P.pre_tiers[blockIdx.y];
    const int32_t *list = P.tlist + P.tbeg[t];
    int32_t *out = P.blist + P.tbeg[t];
    const int64_t count = P.tend[t] - P.tbeg[t];
    const unsigned long long key = *P.keyp;
    for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31); i0 < count;
         i0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = i0 + lane_id();
        const bool in = i < count;
        const int32_t u = in ? list[i] : 0;
        const int b = in ? bucket_of(key, u, P.buckets) : -1;
        const uint32_t peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (in && lane_id() == leader)
            base = atomicAdd(&P.pb_cur[9 * t + b], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (in)
            out[base + __popc(peers & lanemask_lt())] = u;
    }
}

// Per-warp register queue of moves: lane i holds entry i; one global atomic
// per 32 moves instead of one per warp-round (the bucket's move counter is a
// single hot address).
constexpr double GAIN_FX_SCALE = 17592186044416.0;  // 2^44

struct MoveQueue {
    int32_t u = 0, l = 0;
    int n = 0;           // warp-uniform fill
    long long gain = 0;  // this lane's movers' Δ (fixed point)

    // at kernel end, by all lanes of the warp
    __device__ __forceinline__ void flush_gain(const SweepParams &P) {
        const long long g = warp_sum(gain);
        if (lane_id() == 0 && g && P.gain_fx)
            atomicAdd(reinterpret_cast<unsigned long long *>(P.gain_fx), static_cast<unsigned long long>(g));
        gain = 0;
    }

    __device__ __forceinline__ void flush(const SweepParams &P) {
        if (n == 0)
            return;
        int32_t base = 0;
        if (lane_id() == 0)
            base = atomicAdd(P.mv_count, n);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (lane_id() < n)
            P.mv[base + lane_id()] = make_int2(u, l);
        n = 0;
    }
    // all lanes: lanes with `moved` enqueue (node, label)
    __device__ __forceinline__ void push(const SweepParams &P, bool moved, int32_t node, int32_t label) {
        const uint32_t mask = __ballot_sync(0xffffffffu, moved);
        const int cnt = __popc(mask);
        if (cnt == 0)
            return;
        if (n + cnt > 32)
            flush(P);
        const int lane = lane_id();
        const int k = lane - n;  // this lane receives the k-th mover
        const bool recv = k >= 0 && k < cnt;
        const int src = recv ? static_cast<int>(__fns(mask, 0, k + 1)) : lane;
        const int32_t nu = __shfl_sync(0xffffffffu, node, src);
        const int32_t nl = __shfl_sync(0xffffffffu, label, src);
        if (recv) {
            u = nu;
            l = nl;
        }
        n += cnt;
    }
};

// Applies one decision.  Must be reached by all lanes of the warp (moves are
// queued warp-collectively); only lanes with `act` carry a decision.
// `margin`: PLP count tallies, best count minus the runner-up's (0 where a
// tier does not track the runner-up: the node is re-evaluated on any change)
template <int MODE>
__device__ __forceinline__ void decide(const SweepParams &P, MoveQueue &q, bool act, int32_t u, int32_t cur,
                                       int32_t best, double val, double margin = 0.0) {
    bool moved = false;
    if (act) {
        if (MODE == MODE_PLP) {
            moved = best != cur;
        } else {
            moved = best != INT32_MAX && best != cur && val > 0.0;
            if (moved && P.guard && P.csize && P.csize[cur] == 1 && P.csize[best] == 1 && best > cur)
                moved = false;
        }
    }
    if (P.dense_best) {
        if (act) {
            P.dense_best[u] = moved ? best : cur;
            if (P.dense_gain)
                P.dense_gain[u] = (moved && MODE == MODE_PLM) ? val : 0.0;
        }
        return;
    }
    q.push(P, moved, u, best);
    if (MODE == MODE_PLM && moved)
        q.gain += llrint(val * GAIN_FX_SCALE);
    // PLP active set (H/plp.hpp:127-133); PLM pruning: a non-mover sleeps
    // until a neighbour moves
    if (act && !moved && P.active)
        P.active[u] = 0;
    if (MODE == MODE_PLP && act && P.chg) {
        P.chg[u] = make_int2(0, static_cast<int32_t>(margin));
    }
}

// stats layout per mode: [0] nodes, [1] entries unweighted, [2] entries weighted
__device__ __forceinline__ void flush_stats(const SweepParams &P, int slot, unsigned long long nodes,
                                            unsigned long long entries) {
    nodes = warp_sum(nodes);
    entries = warp_sum(entries);
    if (lane_id() == 0 && (nodes | entries)) {
        atomicAdd(&P.stats[3 * slot], nodes);
        atomicAdd(&P.stats[3 * slot + (P.w ? 2 : 1)], entries);
    }
}

// ---------------------------------------------------------------------------
// tiers G8 / G16 / G32: one entry per lane, G lanes per node
// ---------------------------------------------------------------------------
// One warp's share of a direct tier in one sub-sweep (warps gw of nw).
template <int G, int MODE, int VC, bool REDUX = true>
__device__ __forceinline__ void direct_tier(const SweepParams &P, int tier, int chunk, unsigned long long bkey,
                                            int64_t gw, int64_t nw, double *scratch_w, MoveQueue &q,
                                            unsigned long long &st_n, unsigned long long &st_e) {
    constexpr int NPW = 32 / G;
    const int lane = lane_id();
    const int sub = lane / G, k = lane % G;
    const uint32_t gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (sub * G));
    const int32_t *list = P.tlist + P.tbeg[tier];
    const int64_t count = P.tend[tier] - P.tbeg[tier];
    // each warp owns `chunk` (<= 32) candidates per iteration: short warps,
    // many of them, so the tail of a sub-sweep stays occupied
    for (int64_t base = gw * chunk; base < count; base += nw * chunk) {
        const bool in = lane < chunk && base + lane < count;
        const int32_t cand = in ? list[base + lane] : 0;
        uint32_t selmask = __ballot_sync(0xffffffffu, in && selected(P, bkey, cand));
        while (selmask) {
            const uint32_t pos = __fns(selmask, 0, sub + 1);
            const bool has = pos < 32;
            const int32_t u = __shfl_sync(0xffffffffu, cand, has ? pos : 0);
#pragma unroll
            for (int j = 0; j < NPW; ++j)
                selmask &= selmask - 1;
            int64_t s = 0, d = 0;
            if (has) {
                s = P.off[u];
                d = P.off[u + 1] - s;
            }
            bool valid = has && k < d;
            const int32_t v = valid ? col_at(P, s + k) : 0;
            const double wt = load_w<VC>(P, s + k, valid);
            if (MODE == MODE_PLM)
                valid = valid && v != u;
            const int32_t key = valid ? P.z[v] : 0;
            double agg;
            const bool leader = aggregate<VC>(key, wt, valid, gmask, scratch_w, agg);
            const int32_t cur = has ? P.z[u] : 0;
            double cv;
            int32_t ck;
            if (MODE == MODE_PLP) {
                cv = leader ? agg : -1.0;
                ck = leader ? key : INT32_MAX;
            } else {
                const double wc = sum_xor<G>((valid && key == cur) ? wt : 0.0);
                if (leader && key != cur) {
                    const double vol_u = P.vol[u];
                    const double vol_c = __dsub_rn(P.vols[cur], vol_u);
                    cv = plm_delta(agg, wc, vol_c, P.vols[key], vol_u, P);
                    ck = key;
                } else {
                    cv = -INFINITY;
                    ck = INT32_MAX;
                }
            }
            double margin = 0.0;
            if (REDUX && MODE == MODE_PLP && VC != VC_REAL) {
                // integer tallies: each distinct label sits in one leader lane, so the
                // group's winner (ties to the smaller label) and runner-up are three
                // redux.sync over (count, label) instead of log2(G) shuffle rounds
                const uint32_t bv = leader ? static_cast<uint32_t>(agg) : 0u;
                const int32_t bk = leader ? key : INT32_MAX;
                const uint32_t mv = __reduce_max_sync(gmask, bv);
                const int32_t ml = __reduce_min_sync(gmask, bv == mv ? bk : INT32_MAX);
                const uint32_t sv = __reduce_max_sync(gmask, (bv == mv && bk == ml) ? 0u : bv);
                cv = static_cast<double>(mv);
                ck = ml;
                margin = P.chg ? static_cast<double>(mv - sv) : 0.0;
            } else if (MODE == MODE_PLP && P.chg) {
                double cs = -1.0;
                argmax2_xor<G>(cv, ck, cs);
                margin = cv - fmax(cs, 0.0);
            } else {
                argmax_m<MODE, G>(cv, ck);
            }
            const bool act = has && k == 0;
            decide<MODE>(P, q, act, u, cur, ck, cv, margin);
            if (act) {
                ++st_n;
                st_e += static_cast<unsigned long long>(d);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// tiers G8 / G16 (deg <= DM): a thread per node.  The row's <= DM labels are tallied in
// registers (each label's first entry sums the equal ones after it, in entry
// order -- the lane order of the group aggregate), so a warp evaluates 32
// nodes at once with no shuffles, no __match_any_sync and no cross-lane
// argmax; 8 lanes per node spent most of the round on those collectives.
// ---------------------------------------------------------------------------
template <int DM, int MODE, int VC>
__global__ void __launch_bounds__(256, VC == VC_COUNT ? 4 : 1) k_sweep_thread(SweepParams P, int tier) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int32_t *list;
    int64_t count;
    const bool pre = tier_range(P, tier, list, count);
    const unsigned long long bkey = load_key(P);
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    // evaluates node u on this lane (act) and decides; warp-collective
    auto eval = [&](int32_t u, bool act) {
        int32_t best = INT32_MAX, cur = 0;
        double bv = (MODE == MODE_PLP) ? -1.0 : -INFINITY, sv = -1.0;
        if (act) {
            const int64_t s = P.off[u];
            const int d = static_cast<int>(P.off[u + 1] - s);
            cur = P.z[u];
            int32_t kk[DM];
            double ww[DM];
#pragma unroll
            for (int c = 0; c < DM; ++c) {
                const bool valid = c < d;
                const int32_t v = valid ? col_at(P, s + c) : -1;
                ww[c] = (VC != VC_COUNT && valid) ? static_cast<double>(P.w[s + c]) : 1.0;
                kk[c] = (valid && !(MODE == MODE_PLM && v == u)) ? v : -1;
            }
#pragma unroll
            for (int c = 0; c < DM; ++c)
                kk[c] = kk[c] >= 0 ? P.z[kk[c]] : EMPTY_KEY;
            double wc = 0.0, vol_u = 0.0, vol_c = 0.0;
            if (MODE == MODE_PLM) {
#pragma unroll
                for (int c = 0; c < DM; ++c)
                    if (kk[c] != EMPTY_KEY && kk[c] == cur)
                        wc += ww[c];
                vol_u = P.vol[u];
                vol_c = __dsub_rn(P.vols[cur], vol_u);
            }
            // candidates: each label's first entry; their volumes gathered together
            bool head[DM];
            double vd[DM];
#pragma unroll
            for (int c = 0; c < DM; ++c) {
                head[c] = kk[c] != EMPTY_KEY && !(MODE == MODE_PLM && kk[c] == cur);
#pragma unroll
                for (int j = 0; j < c; ++j)
                    head[c] = head[c] && kk[j] != kk[c];
                vd[c] = (MODE == MODE_PLM && head[c]) ? P.vols[kk[c]] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < DM; ++c) {
                if (!head[c])
                    continue;
                double agg = 0.0;
#pragma unroll
                for (int j = c; j < DM; ++j)
                    if (kk[j] == kk[c])
                        agg += ww[j];
                const double val = (MODE == MODE_PLP) ? agg : plm_delta(agg, wc, vol_c, vd[c], vol_u, P);
                keep2(val, kk[c], bv, best, sv);
            }
            ++st_n;
            st_e += static_cast<unsigned long long>(d);
        }
        const double margin = (MODE == MODE_PLP && P.chg) ? bv - fmax(sv, 0.0) : 0.0;
        decide<MODE>(P, q, act, u, cur, best, bv, margin);
    };
    // A bucket selects 1/K of the candidates (fewer with margins), so a warp
    // collects the selected nodes of successive 32-candidate rounds in its
    // lanes and evaluates 32 at a time: without it 1/K of the lanes worked
    int32_t pu = 0;
    int np = 0;  // pending selected nodes, lanes [0, np) (warp-uniform)
    // the next round's candidates load while this round's selection (bucket,
    // then the changes / active flag) runs: a sparse sub-sweep is all scan
    int32_t cand_next = gw * 32 + lane < count ? list[gw * 32 + lane] : 0;
    for (int64_t base = gw * 32; base < count; base += nw * 32) {
        const int64_t i = base + lane;
        const int32_t cand = cand_next;
        const int64_t inext = i + nw * 32;
        cand_next = inext < count ? list[inext] : 0;
        const bool act = i < count && selected_in(P, bkey, cand, pre);
        const uint32_t m = __ballot_sync(0xffffffffu, act);
        const int c = __popc(m);
        if (c == 0)
            continue;
        const int take = min(c, 32 - np);
        {
            const int k = lane - np;
            const bool recv = k >= 0 && k < take;
            const int32_t v = __shfl_sync(0xffffffffu, cand, recv ? static_cast<int>(__fns(m, 0, k + 1)) : lane);
            if (recv)
                pu = v;
        }
        np += take;
        if (np == 32) {
            eval(pu, true);
            np = c - take;  // the round's remaining selected nodes start the next batch
            const bool recv = lane < np;
            const int32_t v =
                __shfl_sync(0xffffffffu, cand, recv ? static_cast<int>(__fns(m, 0, take + lane + 1)) : lane);
            if (recv)
                pu = v;
        }
    }
    if (np)
        eval(pu, lane < np);
    q.flush(P);
    q.flush_gain(P);
    flush_stats(P, tier, st_n, st_e);
}

template <int G, int MODE, int VC>
// count tallies: 32 registers (8-16 B of spill), 8 blocks per SM instead of 6
// (C2 level 0 -6 %)
__global__ void __launch_bounds__(256, VC == VC_COUNT ? 8 : 1) k_sweep_direct(SweepParams P, int tier, int chunk) {
    __shared__ double scratch[8][32];
    const int wid = threadIdx.x >> 5;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    direct_tier<G, MODE, VC>(P, tier, chunk, load_key(P), gw, nw, scratch[wid], q, st_n, st_e);
    q.flush(P);
    q.flush_gain(P);
    flush_stats(P, tier, st_n, st_e);
}

// ---------------------------------------------------------------------------
// tier WARP: one warp per node (deg <= 256), per-warp smem hash (cap <= 512).
// All of a row's neighbour ids, then all labels, are loaded up front (8 per
// lane) so a node costs two rounds of memory latency, not deg/32.  (Parking
// vols[label] in the table at insert time was measured slower: the extra
// 4 KB of shared memory per warp costs more occupancy than the scan's
// gather rounds.)
// ---------------------------------------------------------------------------
#ifdef CD_PHASE_TIMING
// debug build only: clock64 phase sums of the warp tier (lane 0 of each warp)
__device__ unsigned long long g_phase[16];
#define CD_PT_START(t) long long t = clock64()
#define CD_PT(t, i)                                                                                  \
    do {                                                                                             \
        __syncwarp();                                                                                \
        if (lane == 0) {                                                                             \
            const long long now_ = clock64();                                                        \
            atomicAdd(&g_phase[i], static_cast<unsigned long long>(now_ - t));                       \
            t = now_;                                                                                \
        }                                                                                            \
    } while (0)
#else
#define CD_PT_START(t)
#define CD_PT(t, i)
#endif

constexpr int SW_WARP_CAP = WARP_TABLE_CAP;
constexpr int SW_WARP_ITEMS = 8;  // 256 / 32

// One warp's share of the WARP tier in one sub-sweep; the warp's table
// (keys / vals / dist) is empty on entry and left empty.
template <int MODE, int VC>
__device__ __forceinline__ void warp_tier(const SweepParams &P, int chunk, unsigned long long bkey, int64_t gw,
                                          int64_t nw, int32_t *keys, TallyT<VC> *vals, uint16_t *dist,
                                          double *scratch_w, MoveQueue &q, unsigned long long &st_n,
                                          unsigned long long &st_e) {
    using V = TallyT<VC>;
    const int lane = lane_id();
    const int32_t *list;
    int64_t count;
    const bool pre = tier_range(P, TIER_WARP, list, count);
    // each warp owns `chunk` (<= 32) candidates per iteration: short warps,
    // many of them, so the tail of a sub-sweep stays occupied
    for (int64_t base = gw * chunk; base < count; base += nw * chunk) {
        const bool in = lane < chunk && base + lane < count;
        const int32_t cand = in ? list[base + lane] : 0;
        uint32_t selmask = __ballot_sync(0xffffffffu, in && selected_in(P, bkey, cand, pre));
        while (selmask) {
            const int32_t u = __shfl_sync(0xffffffffu, cand, __ffs(selmask) - 1);
            selmask &= selmask - 1;
            CD_PT_START(pt);
            const int64_t s = P.off[u], e = P.off[u + 1];
            uint32_t cap = 64;
            while (cap < 2 * (e - s))
                cap <<= 1;
            CD_PT(pt, 0);
            const int32_t cur = P.z[u];
            int32_t vv[SW_WARP_ITEMS], kk[SW_WARP_ITEMS];
            float ww[SW_WARP_ITEMS];
#pragma unroll
            for (int c = 0; c < SW_WARP_ITEMS; ++c) {
                const int64_t f = s + c * 32 + lane;
                vv[c] = f < e ? col_at(P, f) : -1;
                ww[c] = (VC != VC_COUNT && f < e) ? P.w[f] : 1.0f;
            }
            // the mover's own volume terms, off the critical path
            const double vol_u = (MODE == MODE_PLM) ? P.vol[u] : 0.0;
            const double vols_cur = (MODE == MODE_PLM) ? P.vols[cur] : 0.0;
            CD_PT(pt, 1);
#pragma unroll
            for (int c = 0; c < SW_WARP_ITEMS; ++c)
                kk[c] = vv[c] >= 0 ? P.z[vv[c]] : 0;
            __syncwarp();
            CD_PT(pt, 2);
            double wc = 0.0;
            int nd = 0;  // distinct labels so far (warp-uniform)
#pragma unroll
            for (int c = 0; c < SW_WARP_ITEMS; ++c) {
                if (s + c * 32 >= e)
                    break;
                bool valid = vv[c] >= 0;
                if (MODE == MODE_PLM)
                    valid = valid && vv[c] != u;
                const double wt = static_cast<double>(ww[c]);
                if (own_bypass<MODE, VC>() && valid && kk[c] == cur) {
                    wc += wt;
                    valid = false;
                }
                if (!__any_sync(0xffffffffu, valid))
                    continue;  // an all-own round: nothing to tally
                bool claimed = false;
                uint32_t slot = 0;
                if (VC == VC_REAL) {
                    // fp64 tallies: combine equal labels in lane order first,
                    // so every slot sees one add per round (deterministic)
                    double agg;
                    if (aggregate<VC>(kk[c], wt, valid, 0xffffffffu, scratch_w, agg))
                        claimed = tinsert_claim<V>(keys, vals, cap - 1, kk[c], static_cast<V>(agg), &slot);
                } else if (valid) {
                    // integer tallies are order-free: insert directly
                    claimed = tinsert_entry<VC>(keys, vals, cap - 1, kk[c], static_cast<V>(ww[c]), &slot);
                }
                const uint32_t cm = __ballot_sync(0xffffffffu, claimed);
                if (claimed)
                    dist[nd + __popc(cm & lanemask_lt())] = static_cast<uint16_t>(slot);
                nd += __popc(cm);
            }
            __syncwarp();
            CD_PT(pt, 3);
            if (own_bypass<MODE, VC>())
                wc = warp_sum(wc);
            double cv = (MODE == MODE_PLP) ? -1.0 : -INFINITY;
            double cs = -1.0;  // PLP margin mode: the runner-up's count
            int32_t ck = INT32_MAX;
            const double vol_c = (MODE == MODE_PLM) ? __dsub_rn(vols_cur, vol_u) : 0.0;
            // the distinct labels in rounds of SW_ILP per lane: the vols[key]
            // gathers of a round are independent and in flight together
            for (int j0 = lane; j0 < nd; j0 += 32 * SW_ILP) {
                int32_t key[SW_ILP];
                double aff[SW_ILP], vd[SW_ILP];
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c) {
                    const int j = j0 + 32 * c;
                    const uint32_t t = j < nd ? dist[j] : 0;
                    key[c] = j < nd ? keys[t] : EMPTY_KEY;
                    aff[c] = j < nd ? static_cast<double>(vals[t]) : 0.0;
                }
                if (MODE == MODE_PLM) {
#pragma unroll
                    for (int c = 0; c < SW_ILP; ++c)
                        vd[c] = (key[c] != EMPTY_KEY && key[c] != cur) ? P.vols[key[c]] : 0.0;
                }
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c) {
                    if (key[c] == EMPTY_KEY || (MODE == MODE_PLM && key[c] == cur))
                        continue;
                    const double val = (MODE == MODE_PLP) ? aff[c] : plm_delta(aff[c], wc, vol_c, vd[c], vol_u, P);
                    if (MODE == MODE_PLP && P.chg) {
                        keep2(val, key[c], cv, ck, cs);
                    } else if (better(val, key[c], cv, ck)) {
                        cv = val;
                        ck = key[c];
                    }
                }
            }
            CD_PT(pt, 4);
            if (MODE == MODE_PLP && own_bypass<MODE, VC>() && lane == 0 && wc > 0.0) {
                if (P.chg)
                    keep2(wc, cur, cv, ck, cs);
                else if (better(wc, cur, cv, ck)) {
                    cv = wc;
                    ck = cur;
                }
            }
            double margin = 0.0;
            if (MODE == MODE_PLP && P.chg) {
                argmax2_xor<32>(cv, ck, cs);
                margin = cv - fmax(cs, 0.0);
            } else {
                argmax_m<MODE, 32>(cv, ck);
            }
            decide<MODE>(P, q, lane == 0, u, cur, ck, cv, margin);
            if (lane == 0) {
                ++st_n;
                st_e += static_cast<unsigned long long>(e - s);
            }
            // leave the table empty for the next node: only the claimed slots
            for (int j = lane; j < nd; j += 32) {
                const uint32_t t = dist[j];
                keys[t] = EMPTY_KEY;
                vals[t] = tally_empty<VC>();
            }
            __syncwarp();
            CD_PT(pt, 5);
#ifdef CD_PHASE_TIMING
            if (lane == 0) {
                atomicAdd(&g_phase[8], 1ULL);
                atomicAdd(&g_phase[9], static_cast<unsigned long long>(e - s));
            }
#endif
        }
    }
}

// next power of two >= 2*deg, at least 64 (the table size of a node)
__device__ __forceinline__ uint32_t table_cap(int64_t deg) {
    const uint32_t want = static_cast<uint32_t>(2 * deg);
    return want <= 64 ? 64u : (1u << (32 - __clz(want - 1)));
}

// The selected candidates of one warp's chunks, in list order (warp-uniform).
struct NodeStream {
    const int32_t *list;
    int64_t count, base, step;
    unsigned long long bkey;
    int chunk;
    bool pre;
    int32_t cand = 0;
    uint32_t sel = 0;

    // next selected node, or -1 once the warp's chunks are exhausted
    __device__ __forceinline__ int32_t next(const SweepParams &P) {
        const int lane = lane_id();
        while (sel == 0) {
            if (base >= count)
                return -1;
            const bool in = lane < chunk && base + lane < count;
            cand = in ? list[base + lane] : 0;
            sel = __ballot_sync(0xffffffffu, in && selected_in(P, bkey, cand, pre));
            base += step;
        }
        const int32_t u = __shfl_sync(0xffffffffu, cand, __ffs(sel) - 1);
        sel &= sel - 1;
        return u;
    }
};

// PLP, integer tallies: each lane's best (count, label) and runner-up count
// over its distinct labels -> the warp's winner (ties to the smaller label) and
// the runner-up's count, by three redux.sync instead of five shuffle rounds
// of (fp64 value, label, fp64 runner-up).  Every distinct label lives in one
// lane, so the winner's runner-up is the max of the other lanes' bests and
// the winning lane's own runner-up -- argmax2_xor's result.
__device__ __forceinline__ void keep2_u(uint32_t val, int32_t key, uint32_t &v, int32_t &k, uint32_t &s) {
    if (val > v || (val == v && key < k)) {
        s = max(s, v);
        v = val;
        k = key;
    } else {
        s = max(s, val);
    }
}

__device__ __forceinline__ void warp_best_u(uint32_t &v, int32_t &k, uint32_t &s) {
    const uint32_t m = __reduce_max_sync(0xffffffffu, v);
    const int32_t l = __reduce_min_sync(0xffffffffu, v == m ? k : INT32_MAX);
    s = __reduce_max_sync(0xffffffffu, (v == m && k == l) ? s : v);
    v = m;
    k = l;
}

// argmax2_xor<32> for integer tallies held as doubles (-1: none): warp_best_u
template <int VC>
__device__ __forceinline__ void argmax2_w(double &v, int32_t &k, double &s) {
    if (VC == VC_REAL) {
        argmax2_xor<32>(v, k, s);
        return;
    }
    uint32_t bv = v > 0.0 ? static_cast<uint32_t>(v) : 0u, sv = s > 0.0 ? static_cast<uint32_t>(s) : 0u;
    warp_best_u(bv, k, sv);
    v = bv ? static_cast<double>(bv) : -1.0;
    s = sv ? static_cast<double>(sv) : -1.0;
}

// Tier WARP for integer tallies, software-pipelined over the warp's nodes:
// while node i is tallied, node i+1's label gathers, node i+2's row loads and
// node i+3's offsets are in flight (a node's off -> col -> z chain is three
// dependent memory round trips; one node at a time left the SM waiting on
// them: long-scoreboard stalls, profiles/r02_ncu_c3_plp_k_sweep_warp.txt).
// Same tally, candidate scan and decision as warp_tier.
template <int MODE, int VC>
__device__ __forceinline__ void warp_tier_pipe(const SweepParams &P, int chunk, unsigned long long bkey, int64_t gw,
                                               int64_t nw, int32_t *keys, TallyT<VC> *vals, uint16_t *dist,
                                               MoveQueue &q, unsigned long long &st_n, unsigned long long &st_e) {
    static_assert(VC != VC_REAL, "fp64 tallies keep warp_tier (lane-order combine)");
    using V = TallyT<VC>;
    constexpr bool W = VC != VC_COUNT;
    const int lane = lane_id();
    NodeStream ns;
    ns.pre = tier_range(P, TIER_WARP, ns.list, ns.count);
    ns.base = gw * chunk;
    ns.step = nw * chunk;
    ns.bkey = bkey;
    ns.chunk = chunk;
    // stage A: offsets; stage B: row ids (+ weights); stage C: labels
    int32_t uA, uB, uC;
    int64_t sA = 0, eA = 0, sB = 0, eB = 0;
    int dC = 0;
    int32_t vB[SW_WARP_ITEMS], kC[SW_WARP_ITEMS];
    float wB[SW_WARP_ITEMS], wC[SW_WARP_ITEMS];
    int32_t curC = 0;
    double volC = 0.0;
    auto load_off = [&](int32_t u, int64_t &s, int64_t &e) {
        if (u >= 0) {
            s = P.off[u];
            e = P.off[u + 1];
        }
    };
    auto load_row = [&](int32_t u, int64_t s, int64_t e, int32_t *v, float *w) {
#pragma unroll
        for (int c = 0; c < SW_WARP_ITEMS; ++c) {
            const int64_t f = s + c * 32 + lane;
            const bool in = u >= 0 && f < e;
            v[c] = in ? col_at(P, f) : -1;
            if (MODE == MODE_PLM && v[c] == u)
                v[c] = -1;  // the self-loop is no candidate (H/louvain.hpp:98)
            if (W)
                w[c] = in ? __ldcs(P.w + f) : 0.0f;
        }
    };
    auto gather = [&](int32_t u, const int32_t *v, int32_t *k, int32_t &cur, double &vol) {
#pragma unroll
        for (int c = 0; c < SW_WARP_ITEMS; ++c)
            k[c] = v[c] >= 0 ? P.z[v[c]] : EMPTY_KEY;
        if (u >= 0) {
            cur = P.z[u];
            if (MODE == MODE_PLM)
                vol = P.vol[u];
        }
    };
    // prime the pipeline
    uC = ns.next(P);
    load_off(uC, sA, eA);
    load_row(uC, sA, eA, vB, wB);
    dC = static_cast<int>(eA - sA);
    gather(uC, vB, kC, curC, volC);
#pragma unroll
    for (int c = 0; c < SW_WARP_ITEMS; ++c)
        wC[c] = wB[c];
    uB = uC >= 0 ? ns.next(P) : -1;
    load_off(uB, sB, eB);
    load_row(uB, sB, eB, vB, wB);
    uA = uB >= 0 ? ns.next(P) : -1;
    load_off(uA, sA, eA);
    while (uC >= 0) {
        // ---- issue the next nodes' loads (consumed one and two iterations later)
        int32_t kN[SW_WARP_ITEMS];
        float wN[SW_WARP_ITEMS];
        int32_t curN = 0;
        double volN = 0.0;
        gather(uB, vB, kN, curN, volN);
        const int dN = static_cast<int>(eB - sB);
#pragma unroll
        for (int c = 0; c < SW_WARP_ITEMS; ++c)
            wN[c] = wB[c];
        load_row(uA, sA, eA, vB, wB);
        const int32_t uN2 = uA;
        const int64_t sN2 = sA, eN2 = eA;
        uA = uA >= 0 ? ns.next(P) : -1;
        load_off(uA, sA, eA);
        // ---- node C: tally its labels
        const int32_t u = uC, cur = curC;
        const uint32_t cap = table_cap(dC);
        const double vols_cur = (MODE == MODE_PLM) ? P.vols[cur] : 0.0;
        double wc = 0.0;
        uint32_t own = 0;  // PLP: the own label's tally
        int nd = 0;  // distinct labels so far (warp-uniform)
#pragma unroll
        for (int c = 0; c < SW_WARP_ITEMS; ++c) {
            if (c * 32 >= dC)
                break;
            bool valid = kC[c] != EMPTY_KEY;
            const V wt = W ? static_cast<V>(wC[c]) : V(1);
            if (valid && kC[c] == cur) {  // own-label bypass
                if (MODE == MODE_PLM)
                    wc += static_cast<double>(wt);
                else
                    own += static_cast<uint32_t>(wt);
                valid = false;
            }
            if (!__any_sync(0xffffffffu, valid))
                continue;  // an all-own round: nothing to tally
            uint32_t slot = 0;
            const bool claimed = valid && tinsert_entry<VC>(keys, vals, cap - 1, kC[c], wt, &slot);
            const uint32_t cm = __ballot_sync(0xffffffffu, claimed);
            if (claimed)
                dist[nd + __popc(cm & lanemask_lt())] = static_cast<uint16_t>(slot);
            nd += __popc(cm);
        }
        __syncwarp();
        // ---- candidate scan over the distinct labels, decision
        if (MODE == MODE_PLP) {
            uint32_t bv = 0, sv = 0;
            int32_t bk = INT32_MAX;
            for (int j = lane; j < nd; j += 32) {
                const uint32_t t = dist[j];
                keep2_u(static_cast<uint32_t>(vals[t]), keys[t], bv, bk, sv);
            }
            own = __reduce_add_sync(0xffffffffu, own);
            if (lane == 0 && own > 0)
                keep2_u(own, cur, bv, bk, sv);
            warp_best_u(bv, bk, sv);
            const double margin = P.chg ? static_cast<double>(bv - sv) : 0.0;
            decide<MODE>(P, q, lane == 0, u, cur, bk, static_cast<double>(bv), margin);
        } else {
            wc = warp_sum(wc);
            const double vol_c = __dsub_rn(vols_cur, volC);
            double cv = -INFINITY;
            int32_t ck = INT32_MAX;
            for (int j0 = lane; j0 < nd; j0 += 32 * SW_ILP) {
                int32_t key[SW_ILP];
                double aff[SW_ILP], vd[SW_ILP];
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c) {
                    const int j = j0 + 32 * c;
                    const uint32_t t = j < nd ? dist[j] : 0;
                    key[c] = j < nd ? keys[t] : EMPTY_KEY;
                    aff[c] = j < nd ? static_cast<double>(vals[t]) : 0.0;
                }
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c)
                    vd[c] = (key[c] != EMPTY_KEY && key[c] != cur) ? P.vols[key[c]] : 0.0;
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c) {
                    if (key[c] == EMPTY_KEY || key[c] == cur)
                        continue;
                    const double val = plm_delta(aff[c], wc, vol_c, vd[c], volC, P);
                    if (better(val, key[c], cv, ck)) {
                        cv = val;
                        ck = key[c];
                    }
                }
            }
            argmax_m<MODE, 32>(cv, ck);
            decide<MODE>(P, q, lane == 0, u, cur, ck, cv);
        }
        if (lane == 0) {
            ++st_n;
            st_e += static_cast<unsigned long long>(dC);
        }
        // leave the table empty for the next node: only the claimed slots
        for (int j = lane; j < nd; j += 32) {
            const uint32_t t = dist[j];
            keys[t] = EMPTY_KEY;
            vals[t] = tally_empty<VC>();
        }
        __syncwarp();
        // ---- rotate: B -> C, A -> B
        uC = uB;
        dC = dN;
        curC = curN;
        volC = volN;
#pragma unroll
        for (int c = 0; c < SW_WARP_ITEMS; ++c) {
            kC[c] = kN[c];
            wC[c] = wN[c];
        }
        uB = uN2;
        sB = sN2;
        eB = eN2;
    }
}

template <int MODE, int VC, int MINB>
__global__ void __launch_bounds__(128, MINB) k_sweep_warp_pipe(SweepParams P, int chunk) {
    using V = TallyT<VC>;
    __shared__ int32_t skeys[4][SW_WARP_CAP];
    __shared__ V svals[4][SW_WARP_CAP];
    __shared__ uint16_t sdist[4][SW_WARP_CAP / 2];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    for (int t = lane; t < SW_WARP_CAP; t += 32) {
        skeys[wid][t] = EMPTY_KEY;
        svals[wid][t] = tally_empty<VC>();
    }
    __syncwarp();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    warp_tier_pipe<MODE, VC>(P, chunk, load_key(P), gw, nw, skeys[wid], svals[wid], sdist[wid], q, st_n, st_e);
    q.flush(P);
    q.flush_gain(P);
    flush_stats(P, TIER_WARP, st_n, st_e);
}

template <int MODE, int VC>
// count tallies fit 64 registers without spills: 8 blocks (32 warps) per SM
// instead of 7 (C2 level 0 -3 %); the weighted instances would spill
__global__ void __launch_bounds__(128, VC == VC_COUNT ? 8 : 1) k_sweep_warp(SweepParams P, int chunk) {
    using V = TallyT<VC>;
    __shared__ double scratch[4][32];
    __shared__ int32_t skeys[4][SW_WARP_CAP];
    __shared__ V svals[4][SW_WARP_CAP];
    __shared__ uint16_t sdist[4][SW_WARP_CAP / 2];  // claimed slots = the distinct labels
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    for (int t = lane; t < SW_WARP_CAP; t += 32) {  // empty once; each node cleans up after itself
        skeys[wid][t] = EMPTY_KEY;
        svals[wid][t] = tally_empty<VC>();
    }
    __syncwarp();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    warp_tier<MODE, VC>(P, chunk, load_key(P), gw, nw, skeys[wid], svals[wid], sdist[wid], scratch[wid], q, st_n,
                        st_e);
    q.flush(P);
    q.flush_gain(P);
    flush_stats(P, TIER_WARP, st_n, st_e);
}

#ifdef CD_PHASE_TIMING
extern "C" __attribute__((visibility("default"))) int cd_debug_phase(unsigned long long *out) {
    cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase));
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    return 0;
}
#endif

// ---------------------------------------------------------------------------
// tiers BLOCK / BLOCK2: one block per node, block smem hash of CAP slots.
// Entry and slot loops are unrolled 4-wide so each thread keeps 4
// independent global loads in flight.
// ---------------------------------------------------------------------------
constexpr int SW_BLOCK_THREADS = 256;
constexpr int64_t SW_PREBUCKET_MAX = 1 << 16;  // tiers up to this size are pre-bucketed


// Block-cooperative selection: the block's next SW_BLOCK_THREADS candidates
// (indices blockIdx.x + k * gridDim.x) are tested in parallel and the
// selected ones compacted into sel[] (ascending k).  Returns their number.
template <int NT = SW_BLOCK_THREADS>
__device__ __forceinline__ int block_select(const SweepParams &P, unsigned long long bkey, const int32_t *list,
                                            int64_t count, int64_t k0, int32_t *sel, int *wcount, bool pre) {
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const int64_t i = static_cast<int64_t>(blockIdx.x) + (k0 + threadIdx.x) * gridDim.x;
    const int32_t u = i < count ? list[i] : 0;
    const bool take = i < count && selected_in(P, bkey, u, pre);
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (lane == 0)
        wcount[wid] = __popc(m);
    __syncthreads();
    int base = 0, total = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        base += w < wid ? wcount[w] : 0;
        total += wcount[w];
    }
    if (take)
        sel[base + __popc(m & lanemask_lt())] = u;
    __syncthreads();
    return total;
}

// Shared state of the block evaluator (one node per block at a time).
template <int NW = SW_BLOCK_THREADS / 32>
struct BlockShared {
    double scratch[NW][32];
    double red_v[NW];
    int32_t red_k[NW];
    double red_s[NW];  // PLP margin mode: each warp's runner-up
    double red_wc[NW];
    int ndist;
};

// Evaluates node u with the whole block (256 threads): smem hash tally of
// its neighbours' labels (table of table_cap(deg) slots, claimed slots listed
// in dlist), Δ / affinity of every distinct label, block argmax, decision.
// Called by all threads of the block; ends with a block barrier.
// Where a node's row entries come from (the CSR in global memory).
struct GlobalRow {
    const SweepParams *P;
    int64_t s;
    __device__ __forceinline__ int32_t col(int64_t f) const { return col_at(*P, s + f); }
    __device__ __forceinline__ float w(int64_t f) const { return P->w[s + f]; }
};
template <int MODE, int VC, int NT, class Row>
__device__ __forceinline__ void block_eval_row(const SweepParams &P, int32_t u, int64_t d, const Row &row,
                                               TallyT<VC> *vals, int32_t *keys, uint16_t *dlist,
                                               BlockShared<NT / 32> &sh, MoveQueue &q, unsigned long long &st_n,
                                               unsigned long long &st_e) {
    using V = TallyT<VC>;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const int32_t cur = P.z[u];
    const double vol_u = (MODE == MODE_PLM) ? P.vol[u] : 0.0;
    const double volsc = (MODE == MODE_PLM) ? P.vols[cur] : 0.0;
    const uint32_t cap = table_cap(d);  // the table is empty on entry (block_table_init)
    double wc = 0.0;
    // round c of a warp covers entries c * NT + wid * 32 + lane: a row spreads
    // over every warp of the block (the barrier after the tally waits for the
    // warp with the most entries)
    for (int64_t f0 = wid * 32; f0 < d; f0 += NT * SW_ILP) {
        int32_t vv[SW_ILP], kk[SW_ILP];
        float ww[SW_ILP];
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            const int64_t f = f0 + c * NT + lane;
            vv[c] = f < d ? row.col(f) : -1;
            ww[c] = (VC != VC_COUNT && f < d) ? row.w(f) : 1.0f;
        }
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c)
            kk[c] = vv[c] >= 0 ? P.z[vv[c]] : 0;
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            bool valid = vv[c] >= 0;
            if (MODE == MODE_PLM)
                valid = valid && vv[c] != u;
            const double wt = static_cast<double>(ww[c]);
            if (own_bypass<MODE, VC>() && valid && kk[c] == cur) {
                wc += wt;
                valid = false;
            }
            if (!__any_sync(0xffffffffu, valid))
                continue;  // an all-own round (converged rows): nothing to tally
            bool claimed = false;
            uint32_t slot = 0;
            // integer tallies insert each entry directly (match_any costs about an
            // atomic per lane when the labels differ), unless the round is flooded
            // -- half its entries share the first one's label, whose slot every
            // warp of the block would hit: then equal labels are combined first
            bool combine = false;
            if (VC != VC_REAL) {
                const uint32_t vm = __ballot_sync(0xffffffffu, valid);
                if (__popc(vm) >= 16) {  // (a flood needs 16 equal labels)
                    const int32_t k0 = __shfl_sync(0xffffffffu, kk[c], __ffs(vm) - 1);
                    combine = __popc(__ballot_sync(0xffffffffu, valid && kk[c] == k0)) >= 16;
                }
            }
            if (VC == VC_REAL) {
                // fp64: equal labels combined in lane order first (one add per slot per round)
                double agg;
                if (aggregate<VC>(kk[c], wt, valid, 0xffffffffu, sh.scratch[wid], agg))
                    claimed = tinsert_claim<V>(keys, vals, cap - 1, kk[c], static_cast<V>(agg), &slot);
            } else if (combine) {
                double agg;
                if (aggregate<VC>(kk[c], wt, valid, 0xffffffffu, sh.scratch[wid], agg)) {
                    if (VC == VC_COUNT)
                        claimed = tinsert_count_n(keys, reinterpret_cast<unsigned int *>(vals), cap - 1, kk[c],
                                                  static_cast<unsigned int>(agg), &slot);
                    else
                        claimed = tinsert_claim<V>(keys, vals, cap - 1, kk[c], static_cast<V>(agg), &slot);
                }
            } else if (valid) {
                // integer tallies are order-free: insert directly (tools/microbench/tally_bench.cu)
                claimed = tinsert_entry<VC>(keys, vals, cap - 1, kk[c], static_cast<V>(ww[c]), &slot);
            }
            // the claimers of new slots list them (one counter add per warp)
            const uint32_t cm = __ballot_sync(0xffffffffu, claimed);
            int base = 0;
            if (lane == 0 && cm)
                base = atomicAdd(&sh.ndist, __popc(cm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (claimed)
                dlist[base + __popc(cm & lanemask_lt())] = static_cast<uint16_t>(slot);
        }
    }
    if (own_bypass<MODE, VC>()) {
        wc = warp_sum(wc);
        if (lane == 0)
            sh.red_wc[wid] = wc;
    }
    __syncthreads();
    if (own_bypass<MODE, VC>()) {
        wc = 0.0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w)
            wc += sh.red_wc[w];
    }
    const int nd = sh.ndist;
    double cv = (MODE == MODE_PLP) ? -1.0 : -INFINITY;
    double cs = -1.0;
    int32_t ck = INT32_MAX;
    const double vol_c = (MODE == MODE_PLM) ? __dsub_rn(volsc, vol_u) : 0.0;
    // candidates = the distinct labels only (not the whole table)
    for (int j0 = threadIdx.x; j0 < nd; j0 += NT * SW_ILP) {
        int32_t key[SW_ILP];
        double aff[SW_ILP], vd[SW_ILP];
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            const int jj = j0 + c * NT;
            const uint32_t t = jj < nd ? dlist[jj] : 0;
            key[c] = jj < nd ? keys[t] : EMPTY_KEY;
            aff[c] = jj < nd ? static_cast<double>(vals[t]) : 0.0;
        }
        if (MODE == MODE_PLM) {
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c)
                vd[c] = (key[c] != EMPTY_KEY && key[c] != cur) ? P.vols[key[c]] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            if (key[c] == EMPTY_KEY || (MODE == MODE_PLM && key[c] == cur))
                continue;
            const double val = (MODE == MODE_PLP) ? aff[c] : plm_delta(aff[c], wc, vol_c, vd[c], vol_u, P);
            if (MODE == MODE_PLP && P.chg) {
                keep2(val, key[c], cv, ck, cs);
            } else if (better(val, key[c], cv, ck)) {
                cv = val;
                ck = key[c];
            }
        }
    }
    const bool two = MODE == MODE_PLP && P.chg != nullptr;
    if (MODE == MODE_PLP && own_bypass<MODE, VC>() && threadIdx.x == 0 && wc > 0.0) {
        if (two)
            keep2(wc, cur, cv, ck, cs);
        else if (better(wc, cur, cv, ck)) {
            cv = wc;
            ck = cur;
        }
    }
    if (two)
        argmax2_w<VC>(cv, ck, cs);
    else
        argmax_m<MODE, 32>(cv, ck);
    if (lane == 0) {
        sh.red_v[wid] = cv;
        sh.red_k[wid] = ck;
        sh.red_s[wid] = cs;
    }
    __syncthreads();
    if (wid == 0) {
        cv = lane < NT / 32 ? sh.red_v[lane] : -INFINITY;
        ck = lane < NT / 32 ? sh.red_k[lane] : INT32_MAX;
        cs = lane < NT / 32 ? sh.red_s[lane] : -1.0;
        double margin = 0.0;
        if (two) {
            argmax2_w<VC>(cv, ck, cs);
            margin = cv - fmax(cs, 0.0);
        } else {
            argmax_m<MODE, 32>(cv, ck);
        }
        decide<MODE>(P, q, lane == 0, u, cur, ck, cv, margin);
        if (lane == 0) {
            ++st_n;
            st_e += static_cast<unsigned long long>(d);
        }
    }
    // leave the table empty for the next node: only the claimed slots
    for (int j = threadIdx.x; j < nd; j += NT) {
        const uint32_t t = dlist[j];
        keys[t] = EMPTY_KEY;
        vals[t] = tally_empty<VC>();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        sh.ndist = 0;
    __syncthreads();
}

template <int MODE, int VC, int NT = SW_BLOCK_THREADS>
__device__ __forceinline__ void block_eval_node(const SweepParams &P, int32_t u, TallyT<VC> *vals, int32_t *keys,
                                                uint16_t *dlist, BlockShared<NT / 32> &sh, MoveQueue &q,
                                                unsigned long long &st_n, unsigned long long &st_e) {
    const int64_t s = P.off[u], e = P.off[u + 1];
    block_eval_row<MODE, VC, NT>(P, u, e - s, GlobalRow{&P, s}, vals, keys, dlist, sh, q, st_n, st_e);
}

// Empties a block evaluator's table once per kernel (nodes then clean up
// after themselves); ends with a block barrier.
template <int VC, class SH>
__device__ __forceinline__ void block_table_init(TallyT<VC> *vals, int32_t *keys, uint32_t cap, SH &sh) {
    for (uint32_t t = threadIdx.x; t < cap; t += blockDim.x) {
        keys[t] = EMPTY_KEY;
        vals[t] = tally_empty<VC>();
    }
    if (threadIdx.x == 0)
        sh.ndist = 0;
    __syncthreads();
}

template <int MODE, int VC, int CAP, int TIER, int NT = SW_BLOCK_THREADS>
__global__ void __launch_bounds__(NT) k_sweep_block(SweepParams P) {
    using V = TallyT<VC>;
    extern __shared__ unsigned char smem_raw[];
    V *vals = reinterpret_cast<V *>(smem_raw);
    int32_t *keys = reinterpret_cast<int32_t *>(vals + CAP);
    uint16_t *dlist = reinterpret_cast<uint16_t *>(keys + CAP);  // claimed slots (distinct <= deg <= CAP/2)
    static_assert(CAP <= 65536, "slot ids are 16-bit");
    __shared__ BlockShared<NT / 32> sh;
    __shared__ int32_t sel[NT];
    __shared__ int wcount[NT / 32];
    const int wid = threadIdx.x >> 5;
    const int32_t *list;
    int64_t count;
    const bool pre = tier_range(P, TIER, list, count);
    const unsigned long long bkey = load_key(P);
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    block_table_init<VC>(vals, keys, CAP, sh);
    const int64_t per_block = (count - blockIdx.x + gridDim.x - 1) / gridDim.x;  // candidates of this block
    for (int64_t k0 = 0; k0 < per_block; k0 += NT) {
        const int nsel = block_select<NT>(P, bkey, list, count, k0, sel, wcount, pre);
        for (int j = 0; j < nsel; ++j)
            block_eval_node<MODE, VC, NT>(P, sel[j], vals, keys, dlist, sh, q, st_n, st_e);
    }
    if (wid == 0) {
        q.flush(P);
        q.flush_gain(P);
    }
    flush_stats(P, TIER, st_n, st_e);
}

// ---------------------------------------------------------------------------
// tier CLUSTER (8192 < deg <= 32768, integer tallies): one 4-CTA cluster per node.
// The node's label tally is one hash table spread over the CTAs' shared
// memory (distributed shared memory): label k lives in CTA owner(k), every
// CTA streams a slice of the row and inserts into the owners' tables with
// remote shared-memory atomics; each CTA then scans its own distinct labels,
// and CTA 0 reduces the CTAs' best candidates.  One pass over the row, no
// global scratch -- the partitioned HUB path needs three.
// ---------------------------------------------------------------------------
constexpr int CL_THREADS = 1024;
constexpr int CL_CAP = 16384;  // slots per CTA

template <int CL>
__device__ __forceinline__ int cluster_owner(int32_t key) {
    return static_cast<int>((static_cast<uint32_t>(key) * 0x9E3779B1u) >> 27) % CL;
}

template <int MODE, int VC, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CL_THREADS) k_sweep_cluster(SweepParams P) {
    namespace cg = cooperative_groups;
    using V = TallyT<VC>;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ unsigned char smem_raw[];
    V *vals = reinterpret_cast<V *>(smem_raw);
    int32_t *keys = reinterpret_cast<int32_t *>(vals + CL_CAP);
    uint16_t *dlist = reinterpret_cast<uint16_t *>(keys + CL_CAP);
    __shared__ double scratch[CL_THREADS / 32][32];
    __shared__ double red_v[CL_THREADS / 32], red_s[CL_THREADS / 32];
    __shared__ int32_t red_k[CL_THREADS / 32];
    __shared__ double red_wc[CL_THREADS / 32];
    __shared__ int ndist, overflow;
    __shared__ double part_wc, best_v, best_s;
    __shared__ int32_t best_k;
    const bool two = MODE == MODE_PLP && P.chg != nullptr;  // PLP margins: the runner-up too
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    constexpr int NW = CL_THREADS / 32;
    const int rank = static_cast<int>(cluster.block_rank());
    const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const int32_t *list;
    int64_t count;
    const bool pre = tier_range(P, TIER_CLUSTER, list, count);
    const unsigned long long bkey = load_key(P);
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    for (int t = threadIdx.x; t < CL_CAP; t += CL_THREADS) {
        keys[t] = EMPTY_KEY;
        vals[t] = V(0);
    }
    if (threadIdx.x == 0) {
        ndist = 0;
        overflow = 0;
    }
    cluster.sync();
    // 32 of the cluster's candidates per round, the bucket / activity test once per
    // lane: one candidate per iteration cost a dependent load chain (list, flags) for
    // every node of the other K - 1 buckets.  Every warp of the cluster computes the
    // same mask (a node's flags change only when the node itself is decided)
    for (int64_t r0 = 0; cid + r0 * ncl < count; r0 += 32) {
      const int64_t ci = cid + (r0 + lane) * ncl;
      const int32_t cand = ci < count ? list[ci] : 0;
      uint32_t selm = __ballot_sync(0xffffffffu, ci < count && selected_in(P, bkey, cand, pre));
      while (selm) {
        const int32_t u = __shfl_sync(0xffffffffu, cand, __ffs(selm) - 1);
        selm &= selm - 1;
        const int64_t s = P.off[u], e = P.off[u + 1];
        const int32_t cur = P.z[u];
        double wc = 0.0;
        for (int64_t f0 = s + (static_cast<int64_t>(rank) * NW + wid) * 32 * SW_ILP; f0 < e;
             f0 += static_cast<int64_t>(CL) * CL_THREADS * SW_ILP) {
            int32_t vv[SW_ILP], kk[SW_ILP];
            float ww[SW_ILP];
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                const int64_t f = f0 + c * 32 + lane;
                vv[c] = f < e ? col_at(P, f) : -1;
                ww[c] = (VC != VC_COUNT && f < e) ? P.w[f] : 1.0f;
            }
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c)
                kk[c] = vv[c] >= 0 ? P.z[vv[c]] : 0;
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                bool valid = vv[c] >= 0;
                if (MODE == MODE_PLM)
                    valid = valid && vv[c] != u;
                const double wt = static_cast<double>(ww[c]);
                if (own_bypass<MODE, VC>() && valid && kk[c] == cur) {
                    wc += wt;
                    valid = false;
                }
                if (!__any_sync(0xffffffffu, valid))
                    continue;  // an all-own round: nothing to tally
                double agg;
                if (aggregate<VC>(kk[c], wt, valid, 0xffffffffu, scratch[wid], agg)) {
                    const int owner = cluster_owner<CL>(kk[c]);
                    int32_t *rk = cluster.map_shared_rank(keys, owner);
                    V *rv = cluster.map_shared_rank(vals, owner);
                    uint32_t sl = hash_slot(kk[c], CL_CAP - 1);
                    bool done = false;
                    for (int probe = 0; probe < CL_CAP; ++probe) {
                        const int32_t old = atomicCAS(&rk[sl], EMPTY_KEY, kk[c]);
                        if (old == EMPTY_KEY || old == kk[c]) {
                            atomicAdd(&rv[sl], static_cast<V>(agg));
                            if (old == EMPTY_KEY) {
                                const int pos = atomicAdd(cluster.map_shared_rank(&ndist, owner), 1);
                                cluster.map_shared_rank(dlist, owner)[pos] = static_cast<uint16_t>(sl);
                            }
                            done = true;
                            break;
                        }
                        sl = (sl + 1) & (CL_CAP - 1);
                    }
                    if (!done)
                        atomicExch(cluster.map_shared_rank(&overflow, owner), 1);
                }
            }
        }
        if (own_bypass<MODE, VC>()) {
            wc = warp_sum(wc);
            if (lane == 0)
                red_wc[wid] = wc;
        }
        __syncthreads();
        if (own_bypass<MODE, VC>() && threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < NW; ++w)
                t += red_wc[w];
            part_wc = t;
        }
        cluster.sync();  // tallies and partial w(u, C) complete everywhere
        if (overflow && threadIdx.x == 0 && P.hp_flag)
            *P.hp_flag = 1;
        double wc_all = 0.0;
        if (own_bypass<MODE, VC>())
            for (int r = 0; r < CL; ++r)  // rank order: the same sum on every CTA
                wc_all += *cluster.map_shared_rank(&part_wc, r);
        const double vol_u = (MODE == MODE_PLM) ? P.vol[u] : 0.0;
        const double vol_c = (MODE == MODE_PLM) ? __dsub_rn(P.vols[cur], vol_u) : 0.0;
        const int nd = ndist;
        double cv = (MODE == MODE_PLP) ? -1.0 : -INFINITY, cs = -1.0;
        int32_t ck = INT32_MAX;
        for (int j0 = threadIdx.x; j0 < nd; j0 += CL_THREADS * SW_ILP) {
            int32_t key[SW_ILP];
            double aff[SW_ILP], vd[SW_ILP];
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                const int jj = j0 + c * CL_THREADS;
                const uint32_t t = jj < nd ? dlist[jj] : 0;
                key[c] = jj < nd ? keys[t] : EMPTY_KEY;
                aff[c] = jj < nd ? static_cast<double>(vals[t]) : 0.0;
            }
            if (MODE == MODE_PLM) {
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c)
                    vd[c] = (key[c] != EMPTY_KEY && key[c] != cur) ? P.vols[key[c]] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                if (key[c] == EMPTY_KEY || (MODE == MODE_PLM && key[c] == cur))
                    continue;
                const double val = (MODE == MODE_PLP) ? aff[c] : plm_delta(aff[c], wc_all, vol_c, vd[c], vol_u, P);
                if (two) {
                    keep2(val, key[c], cv, ck, cs);
                } else if (better(val, key[c], cv, ck)) {
                    cv = val;
                    ck = key[c];
                }
            }
        }
        // the own label (in no CTA's table): one more candidate, on CTA 0
        if (MODE == MODE_PLP && own_bypass<MODE, VC>() && rank == 0 && threadIdx.x == 0 && wc_all > 0.0) {
            if (two)
                keep2(wc_all, cur, cv, ck, cs);
            else if (better(wc_all, cur, cv, ck)) {
                cv = wc_all;
                ck = cur;
            }
        }
        if (two)
            argmax2_w<VC>(cv, ck, cs);
        else
            argmax_m<MODE, 32>(cv, ck);
        if (lane == 0) {
            red_v[wid] = cv;
            red_k[wid] = ck;
            red_s[wid] = cs;
        }
        __syncthreads();
        if (wid == 0) {
            cv = lane < NW ? red_v[lane] : -INFINITY;
            ck = lane < NW ? red_k[lane] : INT32_MAX;
            cs = lane < NW ? red_s[lane] : -1.0;
            if (two)
                argmax2_w<VC>(cv, ck, cs);
            else
                argmax_m<MODE, 32>(cv, ck);
            if (lane == 0) {
                best_v = cv;
                best_k = ck;
                best_s = cs;
            }
        }
        cluster.sync();  // every CTA's best is visible
        if (rank == 0 && wid == 0) {
            cv = lane < CL ? *cluster.map_shared_rank(&best_v, lane < CL ? lane : 0) : -INFINITY;
            ck = lane < CL ? *cluster.map_shared_rank(&best_k, lane < CL ? lane : 0) : INT32_MAX;
            cs = lane < CL ? *cluster.map_shared_rank(&best_s, lane < CL ? lane : 0) : -1.0;
            double margin = 0.0;
            if (two) {
                argmax2_w<VC>(cv, ck, cs);
                margin = cv - fmax(cs, 0.0);
            } else {
                argmax_m<MODE, 32>(cv, ck);
            }
            decide<MODE>(P, q, lane == 0, u, cur, ck, cv, margin);
            if (lane == 0) {
                ++st_n;
                st_e += static_cast<unsigned long long>(e - s);
            }
        }
        // clear this CTA's claimed slots for the next node
        for (int j = threadIdx.x; j < nd; j += CL_THREADS) {
            const uint32_t t = dlist[j];
            keys[t] = EMPTY_KEY;
            vals[t] = V(0);
        }
        __syncthreads();
        if (threadIdx.x == 0)
            ndist = 0;
        cluster.sync();  // nobody inserts before every table is clean
      }
    }
    if (rank == 0 && wid == 0) {
        q.flush(P);
        q.flush_gain(P);
    }
    flush_stats(P, TIER_CLUSTER, st_n, st_e);
}

// ---------------------------------------------------------------------------
// Fused phase: a whole PLP run or PLM move phase on a graph whose degrees
// stay within the warp-granular tiers (G8 / G16 / G32 / WARP, deg <= 256) in
// one cooperative kernel.  Every warp takes its share of every tier, grid
// barriers replace the kernel boundaries between evaluation, apply and the
// next sub-sweep, and the stop rules run on the device -- no launch gaps, no
// graph replays, no host round trip per pass.  Same decisions, order and
// stop rules as the Sweeper path (tests/test_gpu_parity.py, bit-exact).
// ---------------------------------------------------------------------------
struct FusedPhase {
    int K;
    unsigned long long seed, salt;
    int max_passes;
    long long theta;      // PLP: iterate while updated > theta; PLM: stop at <= theta
    double stall, qtol;   // PLM rules
    int chunk[4];         // G8, G16, G32, WARP
    int32_t *ctr;         // [0,8) moves of bucket b
    long long *gain;      // [1] this pass's gain (PLM, fixed point)
    long long *result;    // passes, moves, changed
    long long *trace;     // [trace_cap] moves per pass
    unsigned long long *stamp;  // [trace_cap] globaltimer at each pass end
    int trace_cap;
    int print;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int FUSED_THREADS = 128;

template <int MODE, int VC>
__global__ void __launch_bounds__(FUSED_THREADS, 8) k_fused_phase(SweepParams P, FusedPhase F) {
    namespace cg = cooperative_groups;
    using V = TallyT<VC>;
    cg::grid_group grid = cg::this_grid();
    __shared__ double scratch[4][32];
    __shared__ int32_t skeys[4][SW_WARP_CAP];
    __shared__ V svals[4][SW_WARP_CAP];
    __shared__ uint16_t sdist[4][SW_WARP_CAP / 2];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    for (int t = lane; t < SW_WARP_CAP; t += 32) {
        skeys[wid][t] = EMPTY_KEY;
        svals[wid][t] = tally_empty<VC>();
    }
    __syncwarp();
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gsize = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t gw = gtid >> 5, nw = gsize >> 5;
    const int64_t n = P.own_hi;  // whole graph (single device)
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    long long hist0 = -1, hist1 = -1, moves_total = 0, cum_fx = 0;
    int passes = 0;
    bool changed = false;
    // pass counters (per-bucket moves, summed gain) are double-buffered by
    // pass parity: the buffer of pass p+1 is reset after pass p's first grid
    // barrier (every thread has read pass p-1's values by then), so the end
    // of a pass needs no extra barriers
    const bool has_gain = P.gain_fx != nullptr;
    for (int pass = 0; pass < F.max_passes; ++pass) {
        const unsigned long long key = bucket_key(F.seed, F.salt + static_cast<unsigned long long>(pass));
        int32_t *ctr = F.ctr + 8 * (pass & 1);
        long long *gain = F.gain + (pass & 1);
        if (has_gain)
            P.gain_fx = gain;
        long long pass_moves = 0;
        for (int b = 0; b < F.K; ++b) {
            P.bucket = b;
            P.mv_count = ctr + b;
            // (the shuffle argmax: the redux form cost the fused kernel registers, C1 PLP +2 %)
            direct_tier<8, MODE, VC, false>(P, TIER_G8, F.chunk[0], key, gw, nw, scratch[wid], q, st_n, st_e);
            direct_tier<16, MODE, VC, false>(P, TIER_G16, F.chunk[1], key, gw, nw, scratch[wid], q, st_n, st_e);
            direct_tier<32, MODE, VC, false>(P, TIER_G32, F.chunk[2], key, gw, nw, scratch[wid], q, st_n, st_e);
            warp_tier<MODE, VC>(P, F.chunk[3], key, gw, nw, skeys[wid], svals[wid], sdist[wid], scratch[wid], q,
                                st_n, st_e);
            q.flush(P);
            q.flush_gain(P);
            grid.sync();
            if (b == 0) {  // the next pass's counters (read by everyone before this barrier)
                if (gtid < 8)
                    F.ctr[8 * ((pass + 1) & 1) + gtid] = 0;
                if (gtid == 0)
                    F.gain[(pass + 1) & 1] = 0;
            }
            const int64_t mc = ctr[b];
            if (MODE == MODE_PLM) {  // H/louvain.hpp:121-125
                for (int64_t i = gtid; i < mc; i += gsize) {
                    const int2 m = P.mv[i];
                    const int32_t c = P.z[m.x];
                    const_cast<int32_t *>(P.z)[m.x] = m.y;
                    const double vu = P.vol[m.x];
                    atomicAdd(const_cast<double *>(&P.vols[m.y]), vu);
                    atomicAdd(const_cast<double *>(&P.vols[c]), -vu);
                    atomicAdd(const_cast<int32_t *>(&P.csize[m.y]), 1);
                    atomicSub(const_cast<int32_t *>(&P.csize[c]), 1);
                }
            } else {
                for (int64_t i = gtid; i < mc; i += gsize) {
                    const int2 m = P.mv[i];
                    const_cast<int32_t *>(P.z)[m.x] = m.y;
                }
            }
            if (P.active) {  // H/plp.hpp:127-133 / pruning: the movers' neighbours wake up
                if (mc > n / 16) {
                    for (int64_t i = gtid; i < n; i += gsize)
                        P.active[i] = 1;
                } else {
                    for (int64_t i = gw; i < mc; i += nw) {
                        const int32_t u = P.mv[i].x;
                        for (int64_t e = P.off[u] + lane; e < P.off[u + 1]; e += 32)
                            P.active[P.col[e]] = 1;
                    }
                }
            }
            pass_moves += mc;
            grid.sync();
        }
        if (pass < F.trace_cap && gtid == 0) {
            F.trace[pass] = pass_moves;
            F.stamp[pass] = global_ns();
        }
        ++passes;
        moves_total += pass_moves;
        if (F.print && gtid == 0)
            printf("[cd] %s(fused) n=%lld pass=%d moved=%lld\n", MODE == MODE_PLP ? "plp" : "move",
                   static_cast<long long>(n), pass, pass_moves);
        bool stop = false;
        if (MODE == MODE_PLP) {
            stop = pass_moves <= F.theta;  // H/plp.hpp:98
        } else if (pass_moves == 0) {
            stop = true;
        } else {
            changed = true;
            if (pass_moves <= F.theta)
                stop = true;
            else if (F.stall > 0.0 && pass >= 8 && static_cast<double>(pass_moves) > F.stall * static_cast<double>(hist0))
                stop = true;
            if (!stop) {
                const long long pass_fx = *gain;
                cum_fx += pass_fx;
                if (F.qtol > 0.0 && static_cast<double>(pass_fx) <= F.qtol * static_cast<double>(cum_fx))
                    stop = true;
            }
            hist0 = hist1;
            hist1 = pass_moves;
        }
        if (stop)
            break;
    }
    flush_stats(P, STAT_SLOT_FUSED, st_n, st_e);
    if (gtid == 0) {
        F.result[0] = passes;
        F.result[1] = moves_total;
        F.result[2] = changed ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// Small graphs (coarse levels): the whole move phase in one cooperative
// launch.  Every pass partitions the nodes by bucket (grid-wide atomics into
// per-bucket lists, heaviest nodes first), every sub-sweep hands nodes to
// blocks through a work counter (block_eval_node, the BLOCK-tier evaluator),
// grid barriers separate evaluation, apply and the next sub-sweep, and the
// stop rules of move_phase_dev run on the device.  No launches, graph
// replays or host round trips between sub-sweeps: on a level of a few
// thousand nodes those, not the work, set the time.
// ---------------------------------------------------------------------------
struct SmallPhase {
    const int32_t *order;  // nodes with deg > 0, heavy tiers first
    int32_t nn;
    int32_t *bsel;         // [nn] bucket of order[i] (scratch)
    int32_t *blist;        // [nn] bucket-partitioned nodes
    int32_t *ctr;          // [0,8) counts [8,16) cursors [16,24) work [24,32) moves
    unsigned long long seed, salt;
    int K;
    int max_passes;
    long long theta;
    double stall, qtol;
    long long *gain;       // [1] this pass's movers' gain (fixed point)
    uint32_t cap_max;
    long long *result;     // passes, moves, changed
    int trace;
};

constexpr int SMALL_THREADS = 256;  // one node per block (512 measured slower: C2 level 1 2.06 -> 2.50 ms)

template <int VC>
__global__ void __launch_bounds__(SMALL_THREADS) k_small_move(SweepParams P, SmallPhase S) {
    namespace cg = cooperative_groups;
    using V = TallyT<VC>;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ unsigned char smem_raw[];
    V *vals = reinterpret_cast<V *>(smem_raw);
    int32_t *keys = reinterpret_cast<int32_t *>(vals + S.cap_max);
    uint16_t *dlist = reinterpret_cast<uint16_t *>(keys + S.cap_max);
    __shared__ BlockShared<SMALL_THREADS / 32> sh;
    __shared__ int s_idx;
    const int wid = threadIdx.x >> 5;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gsize = static_cast<int64_t>(gridDim.x) * blockDim.x;
    unsigned long long st_n = 0, st_e = 0;
    MoveQueue q;
    block_table_init<VC>(vals, keys, S.cap_max, sh);
    long long hist0 = -1, hist1 = -1, moves_total = 0, cum_fx = 0;
    int passes = 0;
    bool changed = false;
    // the 32 pass counters and the gain are double-buffered by pass parity:
    // pass p+1's buffer is reset after pass p's first grid barrier (everyone
    // has read pass p-1's values by then), so a pass ends without barriers
    for (int pass = 0; pass < S.max_passes; ++pass) {
        const unsigned long long key = bucket_key(S.seed, S.salt + static_cast<unsigned long long>(pass));
        int32_t *ctr = S.ctr + 32 * (pass & 1);
        long long *gain = S.gain + (pass & 1);
        P.gain_fx = gain;
        for (int64_t i = gtid; i < S.nn; i += gsize) {
            const int b = S.K > 1 ? bucket_of(key, S.order[i], S.K) : 0;
            S.bsel[i] = b;
            atomicAdd(&ctr[b], 1);
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x < 32)
            S.ctr[32 * ((pass + 1) & 1) + threadIdx.x] = 0;
        if (gtid == 0)
            S.gain[(pass + 1) & 1] = 0;
        for (int64_t i = gtid; i < S.nn; i += gsize) {
            const int b = S.bsel[i];
            int off = 0;
            for (int c = 0; c < b; ++c)
                off += ctr[c];
            S.blist[off + atomicAdd(&ctr[8 + b], 1)] = S.order[i];
        }
        grid.sync();
        long long pass_moves = 0;
        int base = 0;
        for (int b = 0; b < S.K; ++b) {
            const int cnt = ctr[b];
            P.bucket = b;
            P.mv_count = ctr + 24 + b;
            while (true) {
                if (threadIdx.x == 0)
                    s_idx = atomicAdd(&ctr[16 + b], 1);
                __syncthreads();
                const int idx = s_idx;
                __syncthreads();
                if (idx >= cnt)
                    break;
                block_eval_node<MODE_PLM, VC, SMALL_THREADS>(P, S.blist[base + idx], vals, keys, dlist, sh, q, st_n,
                                                             st_e);
            }
            if (wid == 0) {
                q.flush(P);
                q.flush_gain(P);
            }
            grid.sync();
            const int mc = ctr[24 + b];
            for (int64_t i = gtid; i < mc; i += gsize) {  // H/louvain.hpp:121-125
                const int2 m = P.mv[i];
                const int32_t c = P.z[m.x];
                const_cast<int32_t *>(P.z)[m.x] = m.y;
                const double vu = P.vol[m.x];
                atomicAdd(const_cast<double *>(&P.vols[m.y]), vu);
                atomicAdd(const_cast<double *>(&P.vols[c]), -vu);
                atomicAdd(const_cast<int32_t *>(&P.csize[m.y]), 1);
                atomicSub(const_cast<int32_t *>(&P.csize[c]), 1);
            }
            pass_moves += mc;
            base += cnt;
            grid.sync();
        }
        ++passes;
        moves_total += pass_moves;
        if (S.trace && gtid == 0)
            printf("[cd] move(small) nodes=%d pass=%d moved=%lld\n", S.nn, pass, pass_moves);
        bool stop = false;  // the rules of move_phase_dev, identical on every thread
        if (pass_moves == 0) {
            stop = true;
        } else {
            changed = true;
            if (pass_moves <= S.theta)
                stop = true;
            else if (S.stall > 0.0 && pass >= 8 && static_cast<double>(pass_moves) > S.stall * static_cast<double>(hist0))
                stop = true;
            if (!stop) {
                const long long pass_fx = *gain;
                cum_fx += pass_fx;
                if (S.qtol > 0.0 && static_cast<double>(pass_fx) <= S.qtol * static_cast<double>(cum_fx))
                    stop = true;
            }
            hist0 = hist1;
            hist1 = pass_moves;
        }
        if (stop)
            break;
    }
    flush_stats(P, STAT_SLOT_SMALL, st_n, st_e);
    if (gtid == 0) {
        S.result[0] = passes;
        S.result[1] = moves_total;
        S.result[2] = changed ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// tier HUB (largest degrees): hash-partitioned tally.
//   count   chunk blocks (HUB_CHUNK entries) pre-aggregate with match_any,
//           count pairs per partition p = top pbits of (label * phi) and
//           stage the pairs chunk-major
//   scan    partition offsets
//   scatter the staged pairs, written contiguously per partition
//   part    one block per partition aggregates its pairs in a smem hash and
//           keeps the partition's best candidate
//   decide  one block per hub reduces its partitions' candidates
// A pass streams the hub's entries once; there are no global hash tables.
// ---------------------------------------------------------------------------
struct CountGen {
    const int32_t *c;
    __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

__device__ __forceinline__ int32_t hub_part(int32_t key, int pbits) {
    return pbits ? static_cast<int32_t>((static_cast<uint32_t>(key) * 0x9E3779B1u) >> (32 - pbits)) : 0;
}

// Count pass: chunk blocks pre-aggregate their slice of the hub's row per
// warp (match_any), count pairs per partition and stage the pairs
// (chunk-major) for k_hub_scatter_staged; PLM also sums w(u, C) into hub_aux.
template <int MODE, int VC>
__global__ void __launch_bounds__(256) k_hub_pairs(SweepParams P) {
    extern __shared__ unsigned char hub_smem[];
    int32_t *hist = reinterpret_cast<int32_t *>(hub_smem);  // [np]
    __shared__ double scratch[8][32];
    __shared__ double red_wc[8];
    __shared__ int32_t npairs;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const int32_t h = P.chunk_hub[blockIdx.x];
    const int32_t u = P.hubs[h];
    if (!selected(P, load_key(P), u))
        return;
    const int pbits = P.hub_pbits[h];
    const int np = 1 << pbits;
    const int64_t pbase = P.hub_pbase[h];
    const int64_t s0 = P.off[u], e0 = P.off[u + 1];
    const int64_t s = s0 + static_cast<int64_t>(P.chunk_part[blockIdx.x]) * HUB_CHUNK;
    const int64_t e = min(e0, s + HUB_CHUNK);
    const int32_t cur = P.z[u];
    for (int q = threadIdx.x; q < np; q += blockDim.x)
        hist[q] = 0;
    if (threadIdx.x == 0)
        npairs = 0;
    __syncthreads();
    double wc = 0.0;
    for (int64_t f0 = s + wid * 32 * SW_ILP; f0 < e; f0 += 256 * SW_ILP) {
        int32_t vv[SW_ILP], kk[SW_ILP];
        float ww[SW_ILP];
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            const int64_t f = f0 + c * 32 + lane;
            vv[c] = f < e ? col_at(P, f) : -1;
            ww[c] = (VC != VC_COUNT && f < e) ? P.w[f] : 1.0f;
        }
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c)
            kk[c] = vv[c] >= 0 ? P.z[vv[c]] : 0;
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            bool valid = vv[c] >= 0;
            if (MODE == MODE_PLM)
                valid = valid && vv[c] != u;
            const double wt = static_cast<double>(ww[c]);
            // the own label gets no pairs (it was the hottest key of every hub
            // partition table): PLM sums it into w_c, PLP's integer tallies into
            // the own label's count (both in hub_aux; k_hub_decide)
            if (own_bypass<MODE, VC>() && valid && kk[c] == cur) {
                wc += wt;
                valid = false;
            }
            if (!__any_sync(0xffffffffu, valid))
                continue;
            double agg;
            if (aggregate<VC>(kk[c], wt, valid, 0xffffffffu, scratch[wid], agg)) {
                atomicAdd(&hist[hub_part(kk[c], pbits)], 1);
                const int64_t at = static_cast<int64_t>(blockIdx.x) * HUB_CHUNK + atomicAdd(&npairs, 1);
                P.st_key[at] = kk[c];
                P.st_val[at] = agg;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0)
        P.chunk_np[blockIdx.x] = npairs;
    for (int q = threadIdx.x; q < np; q += blockDim.x)
        if (hist[q])
            atomicAdd(&P.hp_cnt[pbase + q], hist[q]);
    if (own_bypass<MODE, VC>()) {
        wc = warp_sum(wc);
        if (lane == 0)
            red_wc[wid] = wc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q)
                t += red_wc[q];
            if (t != 0.0)
                atomicAdd(&P.hub_aux[h], t);
        }
    }
    if (threadIdx.x == 0)
        atomicAdd(&P.stats[3 * TIER_HUB + (P.w ? 2 : 1)], static_cast<unsigned long long>(e - s));
}

// The scatter pass from the count pass's staged pairs: one block per chunk
// reads its pairs back (coalesced, recently written), reserves each
// partition's range once and writes -- instead of re-reading the row and
// re-gathering its labels.
__global__ void __launch_bounds__(256) k_hub_scatter_staged(SweepParams P) {
    extern __shared__ unsigned char hub_smem[];
    int32_t *hist = reinterpret_cast<int32_t *>(hub_smem);
    const int32_t h = P.chunk_hub[blockIdx.x];
    const int32_t u = P.hubs[h];
    if (!selected(P, load_key(P), u))
        return;
    const int pbits = P.hub_pbits[h];
    const int np = 1 << pbits;
    int32_t *hbase = hist + np;
    const int64_t pbase = P.hub_pbase[h];
    const int32_t n = P.chunk_np[blockIdx.x];
    const int64_t cbase = static_cast<int64_t>(blockIdx.x) * HUB_CHUNK;
    for (int q = threadIdx.x; q < np; q += blockDim.x)
        hist[q] = 0;
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x)
        atomicAdd(&hist[hub_part(P.st_key[cbase + i], pbits)], 1);
    __syncthreads();
    for (int q = threadIdx.x; q < np; q += blockDim.x) {
        hbase[q] = hist[q] ? atomicAdd(&P.hp_cur[pbase + q], hist[q]) : 0;
        hist[q] = 0;
    }
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int32_t key = P.st_key[cbase + i];
        const int32_t p = hub_part(key, pbits);
        const int64_t pos = P.hp_start[pbase + p] + hbase[p] + atomicAdd(&hist[p], 1);
        P.hp_key[pos] = key;
        P.hp_val[pos] = P.st_val[cbase + i];
    }
}

template <int MODE, int VC>
__global__ void __launch_bounds__(256, VC == VC_COUNT ? 8 : 1) k_hub_part(SweepParams P) {
    using V = TallyT<VC>;
    extern __shared__ unsigned char hub_smem[];
    V *vals = reinterpret_cast<V *>(hub_smem);
    int32_t *keys = reinterpret_cast<int32_t *>(vals + HUB_PART_CAP);
    __shared__ double red_v[8], red_s[8];
    __shared__ int32_t red_k[8];
    __shared__ double scratch[8][32];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    for (int64_t q = blockIdx.x; q < P.n_parts; q += gridDim.x) {
        const int32_t nq = P.hp_cnt[q];
        if (nq == 0) {
            if (threadIdx.x == 0) {
                P.hp_best_val[q] = -INFINITY;
                P.hp_best_key[q] = INT32_MAX;
                P.hp_second[q] = -1.0;
            }
            continue;
        }
        const int32_t h = P.part_hub[q];
        const int32_t u = P.hubs[h];
        const int32_t cur = P.z[u];
        uint32_t cap = 64;
        while (cap < 2u * static_cast<uint32_t>(nq) && cap < HUB_PART_CAP)
            cap <<= 1;
        for (uint32_t t = threadIdx.x; t < cap; t += blockDim.x) {
            keys[t] = EMPTY_KEY;
            vals[t] = V(0);
        }
        __syncthreads();
        const int64_t st = P.hp_start[q];
        // a warp's 32 consecutive pairs combine equal labels first (a hub's
        // pairs repeat its popular labels once per chunk warp)
        for (int32_t i0 = wid * 32; i0 < nq; i0 += blockDim.x) {
            const int32_t i = i0 + lane;
            const bool valid = i < nq;
            const int32_t key = valid ? P.hp_key[st + i] : 0;
            const double pv = valid ? P.hp_val[st + i] : 0.0;
            double agg;
            if (!aggregate<VC_REAL>(key, pv, valid, 0xffffffffu, scratch[wid], agg))
                continue;
            const V w = static_cast<V>(agg);
            uint32_t sl = hash_slot(key, cap - 1);
            bool done = false;
            for (uint32_t probe = 0; probe < cap; ++probe) {
                const int32_t old = atomicCAS(&keys[sl], EMPTY_KEY, key);
                if (old == EMPTY_KEY || old == key) {
                    atomicAdd(&vals[sl], w);
                    done = true;
                    break;
                }
                sl = (sl + 1) & (cap - 1);
            }
            if (!done)
                *P.hp_flag = 1;  // more distinct labels than slots: reported by the host
        }
        __syncthreads();
        const double wc = (MODE == MODE_PLM) ? P.hub_aux[h] : 0.0;
        const double vol_u = (MODE == MODE_PLM) ? P.vol[u] : 0.0;
        const double vol_c = (MODE == MODE_PLM) ? __dsub_rn(P.vols[cur], vol_u) : 0.0;
        double cv = -INFINITY, cs = -1.0;
        int32_t ck = INT32_MAX;
        const bool two = MODE == MODE_PLP && P.chg != nullptr;  // PLP margins: the runner-up too
        for (uint32_t t0 = threadIdx.x; t0 < cap; t0 += blockDim.x * SW_ILP) {
            int32_t key[SW_ILP];
            double aff[SW_ILP], vd[SW_ILP];
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                const uint32_t t = t0 + blockDim.x * c;
                key[c] = t < cap ? keys[t] : EMPTY_KEY;
                aff[c] = t < cap ? static_cast<double>(vals[t]) : 0.0;
            }
            if (MODE == MODE_PLM) {
#pragma unroll
                for (int c = 0; c < SW_ILP; ++c)
                    vd[c] = (key[c] != EMPTY_KEY && key[c] != cur) ? P.vols[key[c]] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < SW_ILP; ++c) {
                if (key[c] == EMPTY_KEY || (MODE == MODE_PLM && key[c] == cur))
                    continue;
                const double val = (MODE == MODE_PLP) ? aff[c] : plm_delta(aff[c], wc, vol_c, vd[c], vol_u, P);
                if (two) {
                    keep2(val, key[c], cv, ck, cs);
                } else if (better(val, key[c], cv, ck)) {
                    cv = val;
                    ck = key[c];
                }
            }
        }
        if (two)
            argmax2_w<VC>(cv, ck, cs);
        else
            argmax_m<MODE, 32>(cv, ck);
        if (lane == 0) {
            red_v[wid] = cv;
            red_k[wid] = ck;
            red_s[wid] = cs;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            cv = red_v[0];
            ck = red_k[0];
            cs = red_s[0];
            for (int w2 = 1; w2 < 8; ++w2) {
                if (better(red_v[w2], red_k[w2], cv, ck)) {
                    cs = fmax(red_s[w2], cv);
                    cv = red_v[w2];
                    ck = red_k[w2];
                } else {
                    cs = fmax(cs, red_v[w2]);
                }
            }
            P.hp_best_val[q] = cv;
            P.hp_best_key[q] = ck;
            P.hp_second[q] = cs;
        }
        __syncthreads();
    }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_hub_decide(SweepParams P) {
    __shared__ double red_v[8], red_s[8];
    __shared__ int32_t red_k[8];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const unsigned long long bkey = load_key(P);
    const bool two = MODE == MODE_PLP && P.chg != nullptr;  // PLP margins
    MoveQueue mq;
    for (int64_t h = blockIdx.x; h < P.n_hubs; h += gridDim.x) {
        const int32_t u = P.hubs[h];
        if (!selected(P, bkey, u))
            continue;
        double cv = -INFINITY, cs = -1.0;
        int32_t ck = INT32_MAX;
        for (int64_t q = P.hub_pbase[h] + threadIdx.x; q < P.hub_pbase[h + 1]; q += blockDim.x) {
            const double v = P.hp_best_val[q];
            const int32_t k = P.hp_best_key[q];
            if (two) {  // a partition's (best, runner-up) against the running pair
                const double s = P.hp_second[q];
                if (better(v, k, cv, ck)) {
                    cs = fmax(s, cv);
                    cv = v;
                    ck = k;
                } else {
                    cs = fmax(cs, v);
                }
            } else if (better(v, k, cv, ck)) {
                cv = v;
                ck = k;
            }
        }
        const int32_t cur = P.z[u];
        if (MODE == MODE_PLP && threadIdx.x == 0) {
            // PLP integer tallies: the own label's count (no pairs, k_hub_pairs)
            const double own = P.hub_aux[h];
            if (own > 0.0) {
                if (two)
                    keep2(own, cur, cv, ck, cs);
                else if (better(own, cur, cv, ck)) {
                    cv = own;
                    ck = cur;
                }
            }
        }
        if (two)
            argmax2_xor<32>(cv, ck, cs);
        else
            argmax_m<MODE, 32>(cv, ck);
        if (lane == 0) {
            red_v[wid] = cv;
            red_k[wid] = ck;
            red_s[wid] = cs;
        }
        __syncthreads();
        if (wid == 0) {
            cv = lane < 8 ? red_v[lane] : -INFINITY;
            ck = lane < 8 ? red_k[lane] : INT32_MAX;
            cs = lane < 8 ? red_s[lane] : -1.0;
            double margin = 0.0;
            if (two) {
                argmax2_xor<32>(cv, ck, cs);
                margin = cv - fmax(cs, 0.0);
            } else {
                argmax_m<MODE, 32>(cv, ck);
            }
            decide<MODE>(P, mq, lane == 0, u, cur, ck, cv, margin);
            if (lane == 0) {
                P.hub_aux[h] = 0.0;
                atomicAdd(&P.stats[3 * TIER_HUB], 1ULL);
            }
        }
        __syncthreads();
    }
    if (wid == 0) {
        mq.flush(P);
        mq.flush_gain(P);
    }
}

// ---------------------------------------------------------------------------
// PLP's first sub-sweep from z = node ids (run_plp without `initial`,
// H/plp.hpp:75) on count tallies.  Every label in a row is distinct (rows are
// strictly ascending: no duplicate entries; a self-loop is u's own label
// once), so each tallies 1 and the tie rule (H/plp.hpp:118-124) picks the
// smallest: the row's first entry.  Same decision, margin and move as the
// tally kernels; 8 bytes per node instead of the row and its label gathers.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_plp_identity(SweepParams P) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const unsigned long long key = load_key(P);
    MoveQueue q;
    for (int64_t base = P.own_lo + gw * 32; base < P.own_hi; base += nw * 32) {
        const int64_t u = base + lane;
        bool act = u < P.own_hi && selected(P, key, static_cast<int32_t>(u));
        int64_t s = 0, d = 0;
        if (act) {
            s = P.off[u];
            d = P.off[u + 1] - s;
            act = d > 0;  // isolated nodes are never evaluated (H/plp.hpp:109)
        }
        const int32_t best = act ? P.col[s] : 0;
        // a single label leads the (empty) runner-up by 1; two or more tie
        decide<MODE_PLP>(P, q, act, static_cast<int32_t>(u), static_cast<int32_t>(u), best, 1.0,
                         d == 1 ? 1.0 : 0.0);
    }
    q.flush(P);
}

// ---------------------------------------------------------------------------
// PLM's first sub-sweep of a move phase from singletons (every level of the
// recursion, H/louvain.hpp:242).  Each neighbour v != u is its own
// community, so its tally is exactly w(u, v); u's own community holds u
// alone (w_c = 0, vol_c = vols[u] - vol_u); the candidates are the row's
// entries and each gets the same plm_delta the tally kernels compute.  No
// table: a gather of vols[v] per entry.  Nodes up to BLOCK3 degree: a warp
// each; CLUSTER / HUB degrees: a block each.  (Not counted in the sweep
// families' work counters or times: no tally runs.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void plm_identity_scan(const SweepParams &P, int32_t u, int64_t s, int64_t e,
                                                  double vol_u, double vol_c, int stride, int first, double &cv,
                                                  int32_t &ck) {
    for (int64_t f0 = s + first; f0 < e; f0 += int64_t(stride) * SW_ILP) {
        int32_t vv[SW_ILP];
        double ww[SW_ILP], vd[SW_ILP];
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            const int64_t f = f0 + int64_t(c) * stride;
            vv[c] = f < e ? col_at(P, f) : -1;
            ww[c] = (P.w && f < e) ? static_cast<double>(P.w[f]) : 1.0;
        }
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            if (vv[c] == u)
                vv[c] = -1;  // the self-loop is no candidate (H/louvain.hpp:96-97)
            vd[c] = vv[c] >= 0 ? P.vols[vv[c]] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < SW_ILP; ++c) {
            if (vv[c] < 0)
                continue;
            const double val = plm_delta(ww[c], 0.0, vol_c, vd[c], vol_u, P);
            if (better(val, vv[c], cv, ck)) {
                cv = val;
                ck = vv[c];
            }
        }
    }
}

// SCAN32: the short-row tiers (G8 .. WARP); the block tiers' rows (up to 8192 entries)
// keep a candidate per warp iteration, which spreads the long rows over the warps
template <bool SCAN32>
__global__ void __launch_bounds__(256) k_plm_identity_warp(SweepParams P) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const unsigned long long key = load_key(P);
    const int32_t *list = P.tlist + (SCAN32 ? P.tbeg[TIER_G8] : P.tbeg[TIER_BLOCK]);
    const int64_t count = SCAN32 ? P.tend[TIER_WARP] - P.tbeg[TIER_G8] : P.tend[TIER_BLOCK3] - P.tbeg[TIER_BLOCK];
    MoveQueue q;
    if (!SCAN32) {
        for (int64_t i = gw; i < count; i += nw) {
            const int32_t u = list[i];
            if (!selected(P, key, u))
                continue;
            const int64_t s = P.off[u], e = P.off[u + 1];
            const double vol_u = P.vol[u];
            const double vol_c = __dsub_rn(P.vols[u], vol_u);
            double cv = -INFINITY;
            int32_t ck = INT32_MAX;
            plm_identity_scan(P, u, s, e, vol_u, vol_c, 32, lane, cv, ck);
            argmax_m<MODE_PLM, 32>(cv, ck);
            decide<MODE_PLM>(P, q, lane == 0, u, u, ck, cv);
        }
        q.flush(P);
        q.flush_gain(P);
        return;
    }
    // 32 candidates per round, the bucket test once per lane (a candidate per warp
    // iteration spent most iterations on the K - 1 other buckets' nodes); each
    // selected node's row bounds and volumes are loaded by its lane before the
    // warp evaluates the selected nodes one after the other
    for (int64_t base = gw * 32; base < count; base += nw * 32) {
        const int64_t i = base + lane;
        const int32_t cand = i < count ? list[i] : 0;
        const bool sel = i < count && selected(P, key, cand);
        int64_t ls = 0, le = 0;
        double lvol = 0.0, lvols = 0.0;
        if (sel) {
            ls = P.off[cand];
            le = P.off[cand + 1];
            lvol = P.vol[cand];
            lvols = P.vols[cand];
        }
        uint32_t m = __ballot_sync(0xffffffffu, sel);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const int32_t u = __shfl_sync(0xffffffffu, cand, src);
            const int64_t s = __shfl_sync(0xffffffffu, ls, src), e = __shfl_sync(0xffffffffu, le, src);
            const double vol_u = __shfl_sync(0xffffffffu, lvol, src);
            const double vol_c = __dsub_rn(__shfl_sync(0xffffffffu, lvols, src), vol_u);
            double cv = -INFINITY;
            int32_t ck = INT32_MAX;
            plm_identity_scan(P, u, s, e, vol_u, vol_c, 32, lane, cv, ck);
            argmax_m<MODE_PLM, 32>(cv, ck);
            decide<MODE_PLM>(P, q, lane == 0, u, u, ck, cv);
        }
    }
    q.flush(P);
    q.flush_gain(P);
}

__global__ void __launch_bounds__(256) k_plm_identity_block(SweepParams P) {
    __shared__ double red_v[8];
    __shared__ int32_t red_k[8];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const unsigned long long key = load_key(P);
    const int32_t *list = P.tlist + P.tbeg[TIER_CLUSTER];
    const int64_t count = P.tend[TIER_HUB] - P.tbeg[TIER_CLUSTER];
    MoveQueue q;
    for (int64_t i = blockIdx.x; i < count; i += gridDim.x) {
        const int32_t u = list[i];
        if (!selected(P, key, u))  // uniform across the block
            continue;
        const int64_t s = P.off[u], e = P.off[u + 1];
        const double vol_u = P.vol[u];
        const double vol_c = __dsub_rn(P.vols[u], vol_u);
        double cv = -INFINITY;
        int32_t ck = INT32_MAX;
        plm_identity_scan(P, u, s, e, vol_u, vol_c, 256, threadIdx.x, cv, ck);
        argmax_m<MODE_PLM, 32>(cv, ck);
        if (lane == 0) {
            red_v[wid] = cv;
            red_k[wid] = ck;
        }
        __syncthreads();
        if (wid == 0) {
            cv = lane < 8 ? red_v[lane] : -INFINITY;
            ck = lane < 8 ? red_k[lane] : INT32_MAX;
            argmax_m<MODE_PLM, 32>(cv, ck);
            decide<MODE_PLM>(P, q, lane == 0, u, u, ck, cv);
        }
        __syncthreads();
    }
    if (wid == 0) {
        q.flush(P);
        q.flush_gain(P);
    }
}

// ---------------------------------------------------------------------------
// apply: the bucket's moves become visible to the next sub-sweep
// ---------------------------------------------------------------------------
// A changed node activates its neighbours (H/plp.hpp:127-130).  When a
// bucket moved more than n/16 nodes, every node is activated instead (n bytes
// instead of sum-of-degrees scattered bytes): a node whose neighbourhood did
// not change re-derives the label it already has, so the result is identical.
//
// The move list is `nseg` segments of `stride` entries, segment s holding
// counts[s] moves (one segment on one device; one per rank, rank order, after
// the sharded exchange).  Activation walks (toff, tcol): the graph itself, or
// on a row shard its transposed block -- the owned neighbours of every node.
__device__ __forceinline__ int64_t seg_total(const int32_t *counts, int nseg) {
    int64_t t = 0;
    for (int s = 0; s < nseg; ++s)
        t += counts[s];
    return t;
}

// One mover's row walked by a warp, APPLY_UNROLL loads in flight per lane before
// their updates: with one load per iteration every update waited for its own
// load (ncu: 95 % long-scoreboard stalls, and C3 PLM's first apply -- 1M movers,
// hubs among them -- took 3.3 ms of the phase's 14 ms).
constexpr int APPLY_UNROLL = 8;
template <class F>
__device__ __forceinline__ void for_row_entries(const int32_t *tcol, int64_t s, int64_t t, int lane, F &&f) {
    for (int64_t e0 = s + lane; e0 < t; e0 += 32 * APPLY_UNROLL) {
        int32_t v[APPLY_UNROLL];
#pragma unroll
        for (int c = 0; c < APPLY_UNROLL; ++c)
            v[c] = e0 + 32 * c < t ? __ldcs(tcol + e0 + 32 * c) : -1;
#pragma unroll
        for (int c = 0; c < APPLY_UNROLL; ++c)
            if (v[c] >= 0)
                f(v[c]);
    }
}

// A warp's movers i = gw, gw + nw, ... of one segment: the next mover and its
// row bounds load while the current row is walked (move -> offsets -> entries
// were three dependent loads per mover; C3 PLM's first pass applies ~770 k
// sparse movers per sub-sweep, ~160 in sequence per warp).  f(move, s, t).
template <class F>
__device__ __forceinline__ void for_movers(const int2 *m, int64_t cnt, int64_t gw, int64_t nw, const int64_t *toff,
                                           F &&f) {
    if (gw >= cnt)
        return;
    int2 cur = m[gw];
    int64_t s = toff[cur.x], t = toff[cur.x + 1];
    for (int64_t i = gw; i < cnt; i += nw) {
        const int64_t in = i + nw;
        int2 nxt = cur;
        int64_t sn = 0, tn = 0;
        if (in < cnt) {
            nxt = m[in];
            sn = toff[nxt.x];
            tn = toff[nxt.x + 1];
        }
        f(cur, s, t);
        cur = nxt;
        s = sn;
        t = tn;
    }
}

__global__ void __launch_bounds__(256) k_apply_plp(const int2 *mv, const int32_t *counts, int nseg, int64_t stride,
                                                   int32_t *z, uint8_t *active, int2 *chg, const int64_t *toff,
                                                   const int32_t *tcol, long long *total, int64_t n,
                                                   int64_t dense_at) {
    const int64_t count = seg_total(counts, nseg);
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(reinterpret_cast<unsigned long long *>(total), static_cast<unsigned long long>(count));
    // margin mode: neighbours count the changes in their rows (each entry
    // whose label changed); beyond n/16 movers every node is re-evaluated
    const bool dense = (active || chg) && count > dense_at;
    if (dense && chg)  // (the margins are recomputed at the next evaluation)
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n + 1) / 2;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            if (2 * i + 2 <= n)
                reinterpret_cast<int4 *>(chg)[i] = make_int4(CHG_ALL, 0, CHG_ALL, 0);
            else
                chg[2 * i] = make_int2(CHG_ALL, 0);
        }
    else if (dense)
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n + 15) / 16;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            if (16 * i + 16 <= n)
                reinterpret_cast<uint4 *>(active)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
            else
                for (int64_t j = 16 * i; j < n; ++j)
                    active[j] = 1;
        }
    if ((!active && !chg) || dense) {
        // labels only: a thread per move (coalesced move-list reads; a warp per
        // move left 31 lanes idle -- C3 PLP iteration 1 moves 2.2M nodes per bucket)
        for (int sg = 0; sg < nseg; ++sg) {
            const int2 *m = mv + sg * stride;
            const int64_t cnt = counts[sg];
            for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
                 i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
                const int2 e2 = m[i];
                z[e2.x] = e2.y;
            }
        }
        return;
    }
    for (int sg = 0; sg < nseg; ++sg) {
        const int2 *m = mv + sg * stride;
        const int64_t cnt = counts[sg];
        for_movers(m, cnt, gw, nw, toff, [&](int2 e2, int64_t rs, int64_t rt) {
            if (lane == 0)
                z[e2.x] = e2.y;
            if (chg)
                for_row_entries(tcol, rs, rt, lane, [&](int32_t v) { atomicAdd(&chg[v].x, 1); });
            else
                for_row_entries(tcol, rs, rt, lane, [&](int32_t v) { active[v] = 1; });
        });
    }
}

__device__ __forceinline__ void activate_moved(const int2 *mv, const int32_t *counts, int nseg, int64_t stride,
                                               int64_t count, uint8_t *active, const int64_t *toff,
                                               const int32_t *tcol, int64_t n, int64_t dense_at) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    if (count > dense_at) {
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n + 15) / 16;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            if (16 * i + 16 <= n)
                reinterpret_cast<uint4 *>(active)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
            else
                for (int64_t j = 16 * i; j < n; ++j)
                    active[j] = 1;
        }
        return;
    }
    for (int sg = 0; sg < nseg; ++sg) {
        const int2 *m = mv + sg * stride;
        const int64_t cnt = counts[sg];
        for_movers(m, cnt, gw, nw, toff, [&](int2, int64_t rs, int64_t rt) {
            for_row_entries(tcol, rs, rt, lane, [&](int32_t v) { active[v] = 1; });
        });
    }
}

__global__ void __launch_bounds__(256) k_apply_plm(const int2 *mv, const int32_t *counts, int nseg, int64_t stride,
                                                   int32_t *z, double *vols, int32_t *csize, const double *vol,
                                                   uint8_t *active, const int64_t *toff, const int32_t *tcol,
                                                   int64_t n, long long *total, int64_t dense_at) {
    __shared__ double scratch[8][32];
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    const int64_t count_all = seg_total(counts, nseg);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(reinterpret_cast<unsigned long long *>(total), static_cast<unsigned long long>(count_all));
    // pruning: the movers' neighbours wake up (same rule as PLP's active set)
    if (active)
        activate_moved(mv, counts, nseg, stride, count_all, active, toff, tcol, n, dense_at);
    for (int sg = 0; sg < nseg; ++sg) {
        const int2 *m = mv + sg * stride;
        const int64_t count = counts[sg];
        for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < count;
             base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t i = base + threadIdx.x;
            const bool valid = i < count;
            const int2 e2 = valid ? m[i] : make_int2(0, -1);
            const int32_t u = e2.x, d = e2.y;
            const int32_t c = valid ? z[u] : -1;
            if (valid)
                z[u] = d;
            const double vu = valid ? vol[u] : 0.0;  // H/louvain.hpp:121-125
            // moves into / out of the same community combine per warp first
            double s;
            if (warp_aggregate_sum(d, vu, valid, scratch[wid], s))
                atomicAdd(&vols[d], s);
            if (warp_aggregate_sum(c, vu, valid, scratch[wid], s))
                atomicAdd(&vols[c], -s);
            if (csize) {
                const uint32_t vm = __ballot_sync(0xffffffffu, valid);
                const uint32_t pd = __match_any_sync(0xffffffffu, d) & vm;
                if (valid && (__ffs(pd) - 1) == lane)
                    atomicAdd(&csize[d], __popc(pd));
                const uint32_t pc = __match_any_sync(0xffffffffu, c) & vm;
                if (valid && (__ffs(pc) - 1) == lane)
                    atomicSub(&csize[c], __popc(pc));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static void ensure_side_streams(cd_ctx *ctx) {
    if (ctx->fork_ev)
        return;
    for (int i = 0; i < cd_ctx::NSIDE; ++i) {
        CD_CUDA(cudaStreamCreateWithFlags(&ctx->side[i], cudaStreamNonBlocking));
        CD_CUDA(cudaEventCreateWithFlags(&ctx->join_ev[i], cudaEventDisableTiming));
    }
    CD_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
}

// first index of each tier list segment holding ids >= lo / >= hi (tier
// lists are ascending within a tier)
__global__ void k_tier_narrow(const int32_t *tlist, const int64_t *tstart, int64_t lo, int64_t hi, int64_t *out) {
    const int t = threadIdx.x >> 1;
    if (t >= NUM_TIERS)
        return;
    const int64_t bound = (threadIdx.x & 1) ? hi : lo;
    int64_t a = tstart[t], b = tstart[t + 1];
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (tlist[mid] < bound)
            a = mid + 1;
        else
            b = mid;
    }
    out[threadIdx.x] = a;
}

Sweeper::Sweeper(cd_ctx *ctx, cd_graph *g, const SweepCall &c) : ctx_(ctx), g_(g), c_(c) {
    // PLP needs count tallies (an unweighted graph); PLM's identity sub-sweep takes any weights
    identity_pending_ = c.identity_first && !c.dense_best && (c.mode == MODE_PLM || !g->weighted);
    graph_ensure_bins(ctx, g);
    cnt_.alloc(ctx, 8);
    mv_.alloc(ctx, std::max<int64_t>(g->n, 1));
    total_.alloc(ctx, 1);
    total_.zero();
    gain_.alloc(ctx, 1);
    gain_.zero();
    key_.alloc(ctx, 1);
    key_.zero();
    if (c_.buckets < 1)
        c_.buckets = 1;
    if (c_.buckets > 8)
        fail(CD_EINVAL, "at most 8 buckets per pass");
    if (c_.own_hi < 0) {
        c_.own_lo = 0;
        c_.own_hi = g->n;
    }
    // any attached communicator takes the exchange path (also at size 1)
    exchange_ = !c_.dense_best && ctx->comm != nullptr;
    world_ = exchange_ ? ctx->comm->size : 1;
    for (int t = 0; t < NUM_TIERS; ++t) {
        tbeg_[t] = g->tier_start[t];
        tend_[t] = g->tier_start[t + 1];
    }
    if (c_.own_lo > 0 || c_.own_hi < g->n) {
        DBuf<int64_t> ts(ctx, NUM_TIERS + 1), nb(ctx, 2 * NUM_TIERS);
        CD_CUDA(cudaMemcpyAsync(ts.p, g->tier_start, (NUM_TIERS + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        CD_LAUNCH(ctx, "shard", k_tier_narrow, 1, 32, 0, static_cast<const int32_t *>(g->tlist.p),
                  static_cast<const int64_t *>(ts.p), c_.own_lo, c_.own_hi, nb.p);
        int64_t h[2 * NUM_TIERS];
        CD_CUDA(cudaMemcpyAsync(h, nb.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int t = 0; t < NUM_TIERS; ++t) {
            tbeg_[t] = h[2 * t];
            tend_[t] = h[2 * t + 1];
        }
    }
    if (exchange_)
        rcnt_.alloc(ctx, world_);
    if (c_.buckets > 1 && !c_.dense_best) {
        for (int t : {int(TIER_WARP), int(TIER_BLOCK), int(TIER_BLOCK2), int(TIER_BLOCK3), int(TIER_CLUSTER)}) {
            const int64_t cnt = tend_[t] - tbeg_[t];
            if (cnt > 0 && cnt <= SW_PREBUCKET_MAX) {
                pre_mask_ |= 1u << t;
                pre_tiers_[n_pre_++] = t;
            }
        }
        if (n_pre_) {
            blist_.alloc(ctx, std::max<int64_t>(g->tier_start[NUM_TIERS], 1));
            boff_.alloc(ctx, NUM_TIERS * 9);
            pb_cnt_.alloc(ctx, NUM_TIERS * 9);
            pb_cur_.alloc(ctx, NUM_TIERS * 9);
            pb_cnt_.zero();
        }
    }
}

Sweeper::~Sweeper() {
    if (exec_)
        cudaGraphExecDestroy(exec_);
    if (graph_)
        cudaGraphDestroy(graph_);
}

template <class K>
static void set_smem(K kernel, size_t bytes) {
    CD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
}

// resident blocks per SM of a kernel (occupancy API, cached per kernel)
template <class K>
static int resident_blocks(K kernel, int threads, size_t smem) {
    static std::map<const void *, int> cache;
    static std::mutex mu;  // loopback ranks are host threads
    std::lock_guard<std::mutex> lk(mu);
    const void *key = reinterpret_cast<const void *>(kernel);
    auto it = cache.find(key);
    if (it != cache.end())
        return it->second;
    int b = 0;
    CD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
    b = b > 0 ? b : 1;
    cache[key] = b;
    return b;
}

// nodes a tier kernel gets per sub-sweep (a pre-bucketed tier: about 1/K of
// its list, with 1/8 headroom for uneven buckets; the kernels grid-stride)
static int64_t pre_count(const SweepParams &P, int t, int64_t cnt) {
    if (!((P.pre_mask >> t) & 1u))
        return cnt;
    const int64_t per = (cnt + P.buckets - 1) / P.buckets;
    return std::min(cnt, per + per / 8 + 1);
}

template <int MODE, int VC>
static void launch_tiers(cd_ctx *ctx, cd_graph *g, const SweepParams &P, bool capture, int &branch) {
    using V = TallyT<VC>;
    const int sms = ctx->num_sms;
    // per-tier profiler families; cd_ctx_kernel_stats aggregates "plp_sweep.*"
    // and "plm_move.*" into the family the roofline reports
    static const char *names[2][NUM_TIERS] = {
        {"plp_sweep.g8", "plp_sweep.g16", "plp_sweep.g32", "plp_sweep.warp", "plp_sweep.block", "plp_sweep.block2",
         "plp_sweep.block3", "plp_sweep.cluster", "plp_sweep.hub"},
        {"plm_move.g8", "plm_move.g16", "plm_move.g32", "plm_move.warp", "plm_move.block", "plm_move.block2",
         "plm_move.block3", "plm_move.cluster", "plm_move.hub"}};
    const char *fam = names[MODE][0];
    auto go = [&](auto launch) {
        if (capture) {
            cudaStream_t s = ctx->side[branch];
            CD_CUDA(cudaStreamWaitEvent(s, ctx->fork_ev, 0));
            launch(s);
            CD_CUDA(cudaEventRecord(ctx->join_ev[branch], s));
            ++branch;
        } else {
            launch(static_cast<cudaStream_t>(nullptr));
        }
    };
    // candidates per warp: about two rounds of work per warp (a round serves
    // 32/G nodes; a bucket selects 1/buckets of the candidates)
    // (short tier lists: about one selected node per warp, so the few nodes
    // of a coarse level run on many warps instead of a few serial ones)
    auto chunk_for = [&](int npw, int64_t nodes, int64_t wave_warps) {
        const int64_t hi = std::min<int64_t>(32, 2LL * npw * P.buckets);
        const int64_t lo = std::min<int64_t>(hi, static_cast<int64_t>(npw) * P.buckets);
        const int64_t fit = (nodes + wave_warps - 1) / std::max<int64_t>(wave_warps, 1);
        return static_cast<int>(std::max(lo, std::min(hi, fit)));
    };
    // grid: one resident wave (grid-stride over the chunks), fewer blocks if
    // the tier list is short
    auto wave = [&](auto kernel, int threads, size_t smem) { return sms * resident_blocks(kernel, threads, smem); };
    auto warps_grid_k = [&](auto kernel, int64_t nodes, int threads, int chunk) {
        const int64_t warps = (nodes + chunk - 1) / chunk;
        return grid_for(warps, threads / 32, wave(kernel, threads, 0));
    };
#define CD_TIER_LAUNCH(KERNEL, GRID, BLOCK, SMEM, ...)                                               \
    go([&](cudaStream_t s) {                                                                         \
        if (s)                                                                                       \
            CD_LAUNCH_S(ctx, s, fam, KERNEL, GRID, BLOCK, SMEM, __VA_ARGS__);                        \
        else                                                                                         \
            CD_LAUNCH(ctx, fam, KERNEL, GRID, BLOCK, SMEM, __VA_ARGS__);                             \
    })
    if ((P.tend[TIER_G8] - P.tbeg[TIER_G8])) {
        fam = names[MODE][TIER_G8];
        auto kfn = k_sweep_thread<8, MODE, VC>;  // a thread per node
        const int64_t nodes = pre_count(P, TIER_G8, P.tend[TIER_G8] - P.tbeg[TIER_G8]);
        const int grid = grid_for((nodes + 31) / 32, 8, wave(kfn, 256, 0));
        CD_TIER_LAUNCH(kfn, grid, 256, 0, P, int(TIER_G8));
    }
    if ((P.tend[TIER_G16] - P.tbeg[TIER_G16])) {
        fam = names[MODE][TIER_G16];
        // a thread per node for PLP count tallies (PLM's 16 volume gathers, or 16
        // fp64 weights, per thread cost too many registers: 100-128)
        if (MODE == MODE_PLP && VC == VC_COUNT) {
            auto kfn = k_sweep_thread<16, MODE, VC>;
            const int64_t nodes = pre_count(P, TIER_G16, P.tend[TIER_G16] - P.tbeg[TIER_G16]);
            const int grid = grid_for((nodes + 31) / 32, 8, wave(kfn, 256, 0));
            CD_TIER_LAUNCH(kfn, grid, 256, 0, P, int(TIER_G16));
        } else {
            auto kfn = k_sweep_direct<16, MODE, VC>;
            const int ch = chunk_for(2, P.tend[TIER_G16] - P.tbeg[TIER_G16], int64_t(wave(kfn, 256, 0)) * (256 / 32));
            const int grid = warps_grid_k(kfn, (P.tend[TIER_G16] - P.tbeg[TIER_G16]), 256, ch);
            CD_TIER_LAUNCH(kfn, grid, 256, 0, P, int(TIER_G16), ch);
        }
    }
    if ((P.tend[TIER_G32] - P.tbeg[TIER_G32])) {
        fam = names[MODE][TIER_G32];
        auto kfn = k_sweep_direct<32, MODE, VC>;
        const int ch = chunk_for(1, P.tend[TIER_G32] - P.tbeg[TIER_G32], int64_t(wave(kfn, 256, 0)) * (256 / 32));
        const int grid = warps_grid_k(kfn, (P.tend[TIER_G32] - P.tbeg[TIER_G32]), 256, ch);
        CD_TIER_LAUNCH(kfn, grid, 256, 0, P, int(TIER_G32), ch);
    }
    if ((P.tend[TIER_WARP] - P.tbeg[TIER_WARP])) {
        fam = names[MODE][TIER_WARP];
        // integer tallies: the software-pipelined evaluator (CD_WARP_PIPE=0: the plain one)
        // (value = minimum resident blocks per SM the registers are bounded for)
        // PLP only by default: PLM's pipelined instance needs 96 registers (5 blocks
        // per SM) and was measured slower (C3 PLM warp tier 29.3 -> 32.4 ms; C3 PLP
        // 3.19 -> 2.73 ms)
        static const int pipe = static_cast<int>(env_i64("CD_WARP_PIPE", MODE == MODE_PLP ? 1 : 0));
        constexpr int PVC = VC == VC_REAL ? VC_COUNT : VC;
        auto kfn = VC == VC_REAL || pipe == 0 ? k_sweep_warp<MODE, VC>
                   : pipe == 8                ? k_sweep_warp_pipe<MODE, PVC, 8>
                   : pipe == 6                ? k_sweep_warp_pipe<MODE, PVC, 6>
                                              : k_sweep_warp_pipe<MODE, PVC, 1>;
        const int64_t wave_warps = int64_t(wave(kfn, 128, 0)) * (128 / 32);
        const int64_t cnt = P.tend[TIER_WARP] - P.tbeg[TIER_WARP];
        // pre-bucketed: every listed node is a candidate of this sub-sweep
        const int64_t per = pre_count(P, TIER_WARP, cnt);
        const int ch = (P.pre_mask >> TIER_WARP) & 1u
                           ? static_cast<int>(std::min<int64_t>(32, std::max<int64_t>(1, (per + wave_warps - 1) / wave_warps)))
                           : chunk_for(1, cnt, wave_warps);
        const int grid = warps_grid_k(kfn, per, 128, ch);
        CD_TIER_LAUNCH(kfn, grid, 128, 0, P, ch);
    }
    // block tiers: one block per node; the block size trades threads per
    // node against nodes in flight per SM (env CD_BLOCK_NT / CD_BLOCK2_NT)
    // (the once-per-kernel attribute flags are atomics: concurrent EPP bases
    // launch from several host threads)
    auto block_tier = [&](auto kfn, int tier, int nt, uint32_t cap, std::atomic<bool> &attr) {
        fam = names[MODE][tier];
        const size_t smem = size_t(cap) * (sizeof(V) + sizeof(int32_t)) + size_t(cap / 2) * sizeof(uint16_t);
        if (!attr.load(std::memory_order_acquire)) {
            set_smem(kfn, smem);
            attr.store(true, std::memory_order_release);
        }
        const int nb = grid_for(pre_count(P, tier, P.tend[tier] - P.tbeg[tier]), 1, wave(kfn, nt, smem));
        CD_TIER_LAUNCH(kfn, nb, nt, smem, P);
    };
    static const int block_nt = static_cast<int>(env_i64("CD_BLOCK_NT", 256));
    static const int block2_nt = static_cast<int>(env_i64("CD_BLOCK2_NT", 512));
    if ((P.tend[TIER_BLOCK] - P.tbeg[TIER_BLOCK])) {
        static std::atomic<bool> a128{false}, a256{false};
        if (block_nt == 128)
            block_tier(k_sweep_block<MODE, VC, BLOCK_TABLE_CAP, TIER_BLOCK, 128>, TIER_BLOCK, 128, BLOCK_TABLE_CAP,
                       a128);
        else
            block_tier(k_sweep_block<MODE, VC, BLOCK_TABLE_CAP, TIER_BLOCK, 256>, TIER_BLOCK, 256, BLOCK_TABLE_CAP,
                       a256);
    }
    if ((P.tend[TIER_BLOCK2] - P.tbeg[TIER_BLOCK2])) {
        static std::atomic<bool> a256{false}, a512{false};
        if (block2_nt == 512)
            block_tier(k_sweep_block<MODE, VC, BLOCK2_TABLE_CAP, TIER_BLOCK2, 512>, TIER_BLOCK2, 512,
                       BLOCK2_TABLE_CAP, a512);
        else
            block_tier(k_sweep_block<MODE, VC, BLOCK2_TABLE_CAP, TIER_BLOCK2, 256>, TIER_BLOCK2, 256,
                       BLOCK2_TABLE_CAP, a256);
    }
    if ((P.tend[TIER_BLOCK3] - P.tbeg[TIER_BLOCK3])) {
        constexpr int NT3 = 1024;
        static std::atomic<bool> a3{false};
        block_tier(k_sweep_block<MODE, VC, BLOCK3_TABLE_CAP, TIER_BLOCK3, NT3>, TIER_BLOCK3, NT3, BLOCK3_TABLE_CAP, a3);
    }
    if ((P.tend[TIER_CLUSTER] - P.tbeg[TIER_CLUSTER])) {
        fam = names[MODE][TIER_CLUSTER];
        constexpr int CLN = CLUSTER_CTAS;  // CLN x 16384 slots: <= 50 % load at CLUSTER_MAX_DEG
        auto kfn = k_sweep_cluster<MODE, VC, CLN>;
        const size_t smem = size_t(CL_CAP) * (sizeof(V) + sizeof(int32_t)) + size_t(CL_CAP / 2) * sizeof(uint16_t);
        static std::atomic<int> max_clusters_once{0};
        int max_clusters = max_clusters_once.load(std::memory_order_acquire);
        if (!max_clusters) {
            set_smem(kfn, smem);
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(CLN * ctx->num_sms);
            lc.blockDim = dim3(CL_THREADS);
            lc.dynamicSmemBytes = smem;
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = CLN;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            lc.attrs = &at;
            lc.numAttrs = 1;
            CD_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, reinterpret_cast<const void *>(kfn), &lc));
            max_clusters = std::max(1, max_clusters);
            max_clusters_once.store(max_clusters, std::memory_order_release);
        }
        const int64_t nodes = pre_count(P, TIER_CLUSTER, P.tend[TIER_CLUSTER] - P.tbeg[TIER_CLUSTER]);
        const int ncl = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_clusters, nodes)));
        CD_TIER_LAUNCH(kfn, ncl * CLN, CL_THREADS, smem, P);
    }
    if (P.tend[TIER_HUB] > P.tbeg[TIER_HUB]) {
        fam = names[MODE][TIER_HUB];
        // histograms sized for this graph's largest hub (the attribute once
        // for the largest possible): the scatter kernel's occupancy is set
        // by its shared memory
        const int max_np = 1 << HUB_MAX_PBITS;
        const int np = 1 << hub_pbits_of(g->max_degree);
        const size_t smem_count = size_t(np) * sizeof(int32_t);
        const size_t smem_scatter = 2 * size_t(np) * sizeof(int32_t);  // staged: histogram + bases
        const size_t smem_part = size_t(HUB_PART_CAP) * (sizeof(V) + sizeof(int32_t));
        static std::atomic<bool> attr{false};
        if (!attr.load(std::memory_order_acquire)) {
            set_smem(k_hub_pairs<MODE, VC>, size_t(max_np) * sizeof(int32_t));
            set_smem(k_hub_scatter_staged, 2 * size_t(max_np) * sizeof(int32_t));
            set_smem(k_hub_part<MODE, VC>, smem_part);
            attr.store(true, std::memory_order_release);
        }
        const int nchunks = static_cast<int>(g->n_hub_chunks);
        const int npart = static_cast<int>(std::min<int64_t>(
            g->n_hub_parts, int64_t(sms) * resident_blocks(k_hub_part<MODE, VC>, 256, smem_part)));
        const int ndec = static_cast<int>(std::min<int64_t>(g->n_hubs, sms * 8));
        go([&](cudaStream_t s) {
            cudaStream_t st = s ? s : ctx->stream;
            CD_CUDA(cudaMemsetAsync(P.hp_cnt, 0, g->n_hub_parts * sizeof(int32_t), st));
            CD_CUDA(cudaMemsetAsync(P.hp_cur, 0, g->n_hub_parts * sizeof(int32_t), st));
            const int64_t tiles = scan_scratch_elems(g->n_hub_parts);  // per scratch half
            // per-step profiler families: <mode>.hub_count / _scatter / _part / _decide
            static const std::string sub[2][5] = {
                {"plp_sweep.hub_count", "plp_sweep.hub_scan", "plp_sweep.hub_scatter", "plp_sweep.hub_part",
                 "plp_sweep.hub_decide"},
                {"plm_move.hub_count", "plm_move.hub_scan", "plm_move.hub_scatter", "plm_move.hub_part",
                 "plm_move.hub_decide"}};
            const std::string *nm = sub[MODE];
            auto run = [&](auto launch_one) {
                launch_one((k_hub_pairs<MODE, VC>), nchunks, smem_count, nm[0].c_str());
                exclusive_scan_on<int64_t>(ctx, st, g->n_hub_parts, CountGen{P.hp_cnt},
                                           const_cast<int64_t *>(P.hp_start),
                                           const_cast<int64_t *>(P.hp_start) + g->n_hub_parts, P.hp_scan,
                                           P.hp_scan + tiles,
                                           nm[1].c_str());
                launch_one(k_hub_scatter_staged, nchunks, smem_scatter, nm[2].c_str());
                launch_one((k_hub_part<MODE, VC>), npart, smem_part, nm[3].c_str());
                launch_one((k_hub_decide<MODE>), ndec, size_t(0), nm[4].c_str());
            };
            if (s)
                run([&](auto kernel, int grid, size_t smem, const char *f) {
                    CD_LAUNCH_S(ctx, s, f, kernel, grid, 256, smem, P);
                });
            else
                run([&](auto kernel, int grid, size_t smem, const char *f) {
                    CD_LAUNCH(ctx, f, kernel, grid, 256, smem, P);
                });
        });
    }
#undef CD_TIER_LAUNCH
}

template <int MODE>
static void launch_tiers_vc(cd_ctx *ctx, cd_graph *g, const SweepParams &P, bool capture, int &branch) {
    if (!g->weighted)
        launch_tiers<MODE, VC_COUNT>(ctx, g, P, capture, branch);
    else if (g->int_weights)
        launch_tiers<MODE, VC_INT>(ctx, g, P, capture, branch);
    else
        launch_tiers<MODE, VC_REAL>(ctx, g, P, capture, branch);
}

void Sweeper::enqueue(bool capture, bool recording) {
    cd_ctx *ctx = ctx_;
    cd_graph *g = g_;
    SweepParams P;
    P.off = g->off.p;
    P.col = g->col.p;
    P.w = g->weighted ? g->w.p : nullptr;
    P.vol = g->vol.p;
    P.z = c_.z;
    P.active = c_.active;
    P.chg = c_.chg;
    P.vols = c_.vols;
    P.csize = c_.csize;
    P.gamma = c_.gamma;
    P.inv_total = g->total > 0 ? 1.0 / g->total : 0.0;
    P.inv_sq2 = g->total > 0 ? 1.0 / (2.0 * g->total * g->total) : 0.0;
    P.guard = c_.guard;
    P.keyp = key_.p;
    P.buckets = c_.buckets;
    P.tlist = g->tlist.p;
    for (int t = 0; t < NUM_TIERS; ++t) {
        P.tbeg[t] = tbeg_[t];
        P.tend[t] = tend_[t];
    }
    P.own_lo = static_cast<int32_t>(c_.own_lo);
    P.own_hi = static_cast<int32_t>(c_.own_hi);
    P.pre_mask = pre_mask_;
    P.n_pre = n_pre_;
    for (int i = 0; i < NUM_TIERS; ++i)
        P.pre_tiers[i] = pre_tiers_[i];
    P.blist = blist_.p;
    P.boff = boff_.p;
    P.pb_cnt = pb_cnt_.p;
    P.pb_cur = pb_cur_.p;
    P.mv = mv_.p;
    P.gain_fx = c_.mode == MODE_PLM ? gain_.p : nullptr;
    P.dense_best = c_.dense_best;
    P.dense_gain = c_.dense_gain;
    P.stats = ctx->dstats + (c_.mode == MODE_PLP ? 0 : STAT_MODE_STRIDE);
    P.hubs = g->hubs;
    P.chunk_hub = g->chunk_hub.p;
    P.chunk_part = g->chunk_part.p;
    P.hub_pbits = g->hub_pbits.p;
    P.hub_pbase = g->hub_pbase.p;
    P.part_hub = g->part_hub.p;
    HubScratch *hs = hub_scratch_for(ctx, g);  // private in a concurrent child context
    P.hp_cnt = hs ? hs->hp_cnt.p : g->hp_cnt.p;
    P.hp_cur = hs ? hs->hp_cur.p : g->hp_cur.p;
    P.hp_start = hs ? hs->hp_start.p : g->hp_start.p;
    P.hp_key = hs ? hs->hp_key.p : g->hp_key.p;
    P.hp_val = hs ? hs->hp_val.p : g->hp_val.p;
    P.hp_best_val = hs ? hs->hp_best_val.p : g->hp_best_val.p;
    P.hp_second = hs ? hs->hp_second.p : g->hp_second.p;
    P.hp_best_key = hs ? hs->hp_best_key.p : g->hp_best_key.p;
    P.hp_flag = hs ? hs->hp_flag.p : g->hp_flag.p;
    P.hub_aux = hs ? hs->hub_aux.p : g->hub_aux.p;
    P.hp_scan = hs ? hs->hp_scan.p : g->hp_scan.p;
    P.st_key = hs ? hs->st_key.p : g->st_key.p;
    P.st_val = hs ? hs->st_val.p : g->st_val.p;
    P.chunk_np = hs ? hs->chunk_np.p : g->chunk_np.p;
    P.n_hubs = g->n_hubs;
    P.n_parts = g->n_hub_parts;
    const bool plp = c_.mode == MODE_PLP;
    if (!c_.dense_best)
        CD_CUDA(cudaMemsetAsync(cnt_.p, 0, 8 * sizeof(int32_t), ctx->stream));
    if (n_pre_) {
        CD_LAUNCH(ctx, "prebucket", k_prebucket_count, dim3(PB_BLOCKS, n_pre_), 256, 0, P);
        CD_LAUNCH(ctx, "prebucket", k_prebucket_offsets, 1, 32, 0, P);
        CD_LAUNCH(ctx, "prebucket", k_prebucket_scatter, dim3(PB_BLOCKS, n_pre_), 256, 0, P);
    }
    const bool identity = identity_pending_ && !recording;
    if (!recording)
        identity_pending_ = false;
    for (int b = 0; b < c_.buckets; ++b) {
        P.bucket = b;
        P.mv_count = cnt_.p + b;
        if (b == 0 && identity) {
            if (plp) {
                // labels are still the node ids: the tally is 1 for every neighbour,
                // so the decision is the row's first (smallest) entry
                const int64_t span = P.own_hi - P.own_lo;
                CD_LAUNCH(ctx, "plp_first", k_plp_identity, grid_for((span + 31) / 32, 8, ctx->num_sms * 16), 256,
                          0, P);
            } else {
                // singletons: every neighbour is its own community
                const int64_t nw = P.tend[TIER_WARP] - P.tbeg[TIER_G8];
                const int64_t nw2 = P.tend[TIER_BLOCK3] - P.tbeg[TIER_BLOCK];
                const int64_t nb = P.tend[TIER_HUB] - P.tbeg[TIER_CLUSTER];
                if (nw > 0)
                    CD_LAUNCH(ctx, "plm_first", k_plm_identity_warp<true>, grid_for((nw + 31) / 32, 8, ctx->num_sms * 16),
                              256, 0, P);
                if (nw2 > 0)
                    CD_LAUNCH(ctx, "plm_first", k_plm_identity_warp<false>, grid_for(nw2, 8, ctx->num_sms * 16), 256, 0,
                              P);
                if (nb > 0)
                    CD_LAUNCH(ctx, "plm_first", k_plm_identity_block, grid_for(nb, 1, ctx->num_sms * 8), 256, 0, P);
            }
            if (exchange_)
                exchange_and_apply(b);
            else
                apply(mv_.p, cnt_.p + b, 1, 0);
            continue;
        }
        int branch = 0;
        // profiling mode 2: the sub-sweep's concurrent tier group is the unit
        // timed (non-overlapping: its kernels run as in the timed run)
        cudaEvent_t ga = nullptr;
        if (capture && ctx->profiling == 2) {
            ga = ctx_event(ctx);
            CD_CUDA(cudaEventRecord(ga, ctx->stream));
        }
        if (capture)
            CD_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
        if (plp)
            launch_tiers_vc<MODE_PLP>(ctx, g, P, capture, branch);
        else
            launch_tiers_vc<MODE_PLM>(ctx, g, P, capture, branch);
        for (int i = 0; i < branch; ++i)
            CD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev[i], 0));
        if (ga) {
            cudaEvent_t gb = ctx_event(ctx);
            CD_CUDA(cudaEventRecord(gb, ctx->stream));
            ctx->pending.push_back({plp ? "plp_sweep.group" : "plm_move.group", ga, gb});
        }
        if (c_.dense_best)
            continue;
        if (exchange_)
            exchange_and_apply(b);
        else
            apply(mv_.p, cnt_.p + b, 1, 0);
    }
}

// movers in one PLP sub-sweep beyond which every node is re-evaluated instead
// of counting per neighbour (CD_PLP_DENSE_DIV: n / div, default 16)
static int64_t plp_dense_at(int64_t n) {
    static const int64_t div = std::max<int64_t>(1, env_i64("CD_PLP_DENSE_DIV", 16));
    return n / div;
}

// PLM pruning: movers in one sub-sweep beyond which every node wakes up
// (CD_PLM_DENSE_DIV: n / div, default 16; ported as cdo_activate's rule)
static int64_t plm_dense_at(int64_t n) {
    static const int64_t div = std::max<int64_t>(1, env_i64("CD_PLM_DENSE_DIV", 16));
    return n / div;
}

void Sweeper::apply(const int2 *mv, const int32_t *counts, int nseg, int64_t stride) {
    cd_ctx *ctx = ctx_;
    cd_graph *g = g_;
    // 8 blocks of 256 per SM (30 registers): every resident warp walks movers' rows
    // (C3 PLM apply 10.4 -> 9.5 ms, C3 PLP apply 1.71 -> 1.42 ms against 4 per SM)
    static const int64_t per_sm = std::max<int64_t>(1, env_i64("CD_APPLY_BLOCKS_PER_SM", 8));
    const int64_t napply = std::max<int64_t>(1, std::min<int64_t>((g->n + 255) / 256, ctx->num_sms * per_sm));
    if (c_.mode == MODE_PLP)
        CD_LAUNCH(ctx, "plp_apply", k_apply_plp, static_cast<int>(napply), 256, 0, mv, counts, nseg, stride, c_.z,
                  c_.active, c_.chg, c_.toff ? c_.toff : static_cast<const int64_t *>(g->off.p),
                  c_.tcol ? c_.tcol : static_cast<const int32_t *>(g->col.p), total_.p, g->n, plp_dense_at(g->n));
    else
        CD_LAUNCH(ctx, "plm_apply", k_apply_plm, static_cast<int>(napply), 256, 0, mv, counts, nseg, stride, c_.z,
                  c_.vols, c_.csize, static_cast<const double *>(g->vol.p), c_.active,
                  c_.toff ? c_.toff : static_cast<const int64_t *>(g->off.p),
                  c_.tcol ? c_.tcol : static_cast<const int32_t *>(g->col.p), g->n, total_.p, plm_dense_at(g->n));
}

// Sharded sub-sweep exchange: allgather the per-rank move counts, then the
// move lists padded to the largest count; every rank applies all segments in
// rank order.  One host synchronisation per sub-sweep (the padded size).
void Sweeper::exchange_and_apply(int b) {
    cd_ctx *ctx = ctx_;
    Comm *comm = ctx->comm;
    comm->allgather(ctx, cnt_.p + b, rcnt_.p, sizeof(int32_t));
    std::vector<int32_t> hc(world_);
    CD_CUDA(cudaMemcpyAsync(hc.data(), rcnt_.p, world_ * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t maxc = 0;
    for (int r = 0; r < world_; ++r)
        maxc = std::max<int64_t>(maxc, hc[r]);
    if (maxc == 0)
        return;
    if (rmv_.n < static_cast<size_t>(world_ * maxc))
        rmv_.alloc(ctx, static_cast<size_t>(world_) * std::max<int64_t>(maxc, g_->n / world_ + 1));
    comm->allgather(ctx, mv_.p, rmv_.p, maxc * sizeof(int2));
    apply(rmv_.p, rcnt_.p, world_, maxc);
}

void Sweeper::pass(uint64_t key) {
    unsigned long long k = key;
    CD_CUDA(cudaMemcpyAsync(key_.p, &k, sizeof(k), cudaMemcpyHostToDevice, ctx_->stream));
    if (ctx_->profiling == 2 && !exchange_) {
        ensure_side_streams(ctx_);
        enqueue(true);  // concurrent tier branches, eagerly, group-timed
        return;
    }
    if (ctx_->profiling || !ctx_->use_graphs || exchange_) {
        enqueue(false);
        return;
    }
    if (!exec_) {
        // the first pass runs eagerly (tier kernels on parallel side streams
        // as in the graph); the host records and instantiates the graph for
        // the remaining passes while the device executes it
        ensure_side_streams(ctx_);
        enqueue(true);
        const int64_t l0 = ctx_->launches;
        CD_CUDA(cudaStreamBeginCapture(ctx_->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue(true, true);
        } catch (...) {
            cudaGraph_t gtmp = nullptr;
            cudaStreamEndCapture(ctx_->stream, &gtmp);
            if (gtmp)
                cudaGraphDestroy(gtmp);
            throw;
        }
        CD_CUDA(cudaStreamEndCapture(ctx_->stream, &graph_));
        CD_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
        kernels_per_pass_ = ctx_->launches - l0;
        ctx_->launches = l0;
        return;
    }
    CD_CUDA(cudaGraphLaunch(exec_, ctx_->stream));
    ctx_->launches += kernels_per_pass_;
}

// Eligible: one device (no exchange), every degree within the warp tiers,
// and few enough entries (CD_FUSED_MAX_D, default 2^23) that per-sub-sweep
// launch and join latency, not the work, dominates: on C2's level 0 (18 M
// entries) the separate, concurrently running tier kernels are faster.
bool fused_eligible(const cd_ctx *ctx, const cd_graph *g, const SweepCall &c) {
    static const int64_t max_d = [] {
        const char *e = std::getenv("CD_FUSED_MAX_D");
        return e ? std::atoll(e) : (int64_t(1) << 23);
    }();
    return ctx->comm == nullptr && !c.dense_best && g->n > 0 && g->D <= max_d && g->max_degree <= 256 &&
           c.buckets >= 1 && c.buckets <= 8;
}

template <int MODE, int VC>
static void launch_fused(cd_ctx *ctx, SweepParams &P, FusedPhase &F) {
    auto kfn = k_fused_phase<MODE, VC>;
    int per_sm = 0;
    CD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, FUSED_THREADS, 0));
    if (per_sm < 1)
        fail(CD_EINTERNAL, "fused phase: kernel does not fit an SM");
    const int grid = per_sm * ctx->num_sms;
    const int64_t warps = int64_t(grid) * (FUSED_THREADS / 32);
    // candidates per warp and round, as launch_tiers sizes them
    const int npw[4] = {4, 2, 1, 1};
    const int tiers[4] = {TIER_G8, TIER_G16, TIER_G32, TIER_WARP};
    for (int i = 0; i < 4; ++i) {
        const int64_t nodes = P.tend[tiers[i]] - P.tbeg[tiers[i]];
        const int64_t hi = std::min<int64_t>(32, 2LL * npw[i] * F.K);
        const int64_t lo = std::min<int64_t>(hi, static_cast<int64_t>(npw[i]) * F.K);
        F.chunk[i] = static_cast<int>(std::max(lo, std::min(hi, (nodes + warps - 1) / warps)));
    }
    void *args[] = {&P, &F};
    LaunchScope ls(ctx, MODE == MODE_PLP ? "plp_sweep.fused" : "plm_move.fused");
    CD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kfn), dim3(grid), dim3(FUSED_THREADS), args,
                                        0, ctx->stream));
}

int64_t fused_phase(cd_ctx *ctx, cd_graph *g, const SweepCall &c, uint64_t seed, uint64_t salt, int64_t max_passes,
                    int64_t theta, double stall, double qtol, FusedResult &out) {
    graph_ensure_bins(ctx, g);
    // the reference's caps are uint64 counts: saturate, never wrap; the
    // per-pass trace holds at most the report's record capacity
    max_passes = std::min<int64_t>(std::max<int64_t>(max_passes, 0), INT32_MAX);
    const int64_t cap = std::max<int64_t>(std::min<int64_t>(max_passes, CD_MAX_ITERATION_RECORDS), 1);
    DBuf<int32_t> ctr(ctx, 16);  // two passes' per-bucket counters (parity)
    DBuf<int2> mv(ctx, std::max<int64_t>(g->n, 1));
    DBuf<long long> result(ctx, 4), gain(ctx, 2), trace(ctx, cap);
    DBuf<unsigned long long> stamp(ctx, cap + 1);
    ctr.zero();
    gain.zero();
    SweepParams P{};
    P.off = g->off.p;
    P.col = g->col.p;
    P.w = g->weighted ? g->w.p : nullptr;
    P.vol = g->vol.p;
    P.z = c.z;
    P.active = c.active;
    P.vols = c.vols;
    P.csize = c.csize;
    P.gamma = c.gamma;
    P.inv_total = g->total > 0 ? 1.0 / g->total : 0.0;
    P.inv_sq2 = g->total > 0 ? 1.0 / (2.0 * g->total * g->total) : 0.0;
    P.guard = c.guard;
    P.buckets = c.buckets;
    P.tlist = g->tlist.p;
    for (int t = 0; t < NUM_TIERS; ++t) {
        P.tbeg[t] = g->tier_start[t];
        P.tend[t] = g->tier_start[t + 1];
    }
    P.own_lo = 0;
    P.own_hi = static_cast<int32_t>(g->n);
    P.pre_mask = 0;
    P.mv = mv.p;
    P.stats = ctx->dstats + (c.mode == MODE_PLP ? 0 : STAT_MODE_STRIDE);
    P.gain_fx = c.mode == MODE_PLM ? gain.p : nullptr;
    FusedPhase F{};
    F.K = c.buckets;
    F.seed = seed;
    F.salt = salt;
    F.max_passes = static_cast<int>(max_passes);
    F.theta = theta;
    F.stall = stall;
    F.qtol = qtol;
    F.ctr = ctr.p;
    F.gain = gain.p;
    F.result = result.p;
    F.trace = trace.p;
    F.stamp = stamp.p;
    F.trace_cap = static_cast<int>(cap);
    F.print = std::getenv("CD_TRACE") != nullptr;
    unsigned long long t0 = 0;
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    const int vc = !g->weighted ? VC_COUNT : (g->int_weights ? VC_INT : VC_REAL);
    const auto wall0 = std::chrono::steady_clock::now();
    if (c.mode == MODE_PLP) {
        if (vc == VC_COUNT)
            launch_fused<MODE_PLP, VC_COUNT>(ctx, P, F);
        else if (vc == VC_INT)
            launch_fused<MODE_PLP, VC_INT>(ctx, P, F);
        else
            launch_fused<MODE_PLP, VC_REAL>(ctx, P, F);
    } else {
        if (vc == VC_COUNT)
            launch_fused<MODE_PLM, VC_COUNT>(ctx, P, F);
        else if (vc == VC_INT)
            launch_fused<MODE_PLM, VC_INT>(ctx, P, F);
        else
            launch_fused<MODE_PLM, VC_REAL>(ctx, P, F);
    }
    long long h[3];
    CD_CUDA(cudaMemcpyAsync(h, result.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    out.trace.assign(static_cast<size_t>(std::min<long long>(h[0], cap)), 0);
    std::vector<unsigned long long> st(out.trace.size());
    if (!out.trace.empty()) {
        CD_CUDA(cudaMemcpyAsync(out.trace.data(), trace.p, out.trace.size() * sizeof(long long),
                                cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaMemcpyAsync(st.data(), stamp.p, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                ctx->stream));
    }
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    const double wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    // per-pass times from the device clock (the first pass also carries the launch)
    out.ms.assign(out.trace.size(), 0.0);
    for (size_t i = 0; i < st.size(); ++i)
        out.ms[i] = i ? static_cast<double>(st[i] - st[i - 1]) * 1e-6 : 0.0;
    if (!st.empty()) {
        double rest = 0.0;
        for (size_t i = 1; i < st.size(); ++i)
            rest += out.ms[i];
        out.ms[0] = std::max(0.0, wall_ms - rest);
    }
    (void)t0;
    out.passes = h[0];
    out.moves = h[1];
    out.changed = h[2] != 0;
    return h[0];
}

// Eligible: one device (no exchange), no pruning, no hubs (the block
// evaluator's table holds up to 8192 slots), and a graph small enough that
// launch and synchronisation overheads dominate (CD_SMALL_N, default 2^15).
bool small_move_eligible(const cd_ctx *ctx, const cd_graph *g, const SweepCall &c) {
    static const int64_t limit = [] {
        const char *e = std::getenv("CD_SMALL_N");
        return e ? std::atoll(e) : (int64_t(1) << 15);
    }();
    return ctx->comm == nullptr && !c.active && !c.dense_best && c.mode == MODE_PLM && g->n > 0 && g->n <= limit &&
           g->max_degree <= 4096 && c.buckets >= 1 && c.buckets <= 8;
}

template <int VC>
static void launch_small(cd_ctx *ctx, const SweepParams &P, const SmallPhase &S, size_t smem) {
    auto kfn = k_small_move<VC>;
    CD_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    CD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, SMALL_THREADS, smem));
    if (per_sm < 1)
        fail(CD_EINTERNAL, "small move phase: kernel does not fit an SM");
    // about CD_SMALL_DIV nodes per block (default 2, measured best: fewer,
    // busier blocks lengthen the per-block node queues more than they save
    // on the grid barriers)
    static const int div = [] {
        const char *e = std::getenv("CD_SMALL_DIV");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    const int grid = std::max(1, std::min<int>(per_sm * ctx->num_sms, static_cast<int>((S.nn + div - 1) / div)));
    SweepParams p = P;
    SmallPhase s = S;
    void *args[] = {&p, &s};
    LaunchScope ls(ctx, "plm_move.small");
    CD_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kfn), dim3(grid), dim3(SMALL_THREADS), args,
                                        smem, ctx->stream));
}

bool small_move_phase(cd_ctx *ctx, cd_graph *g, const SweepCall &c, uint64_t seed, uint64_t salt, int64_t max_passes,
                      int64_t theta, double stall, double qtol, int64_t *passes, int64_t *moves) {
    graph_ensure_bins(ctx, g);
    max_passes = std::min<int64_t>(std::max<int64_t>(max_passes, 0), INT32_MAX);  // saturate (uint64 caps)
    const int64_t nn = g->tier_start[NUM_TIERS];
    DBuf<int32_t> order(ctx, std::max<int64_t>(nn, 1)), bsel(ctx, std::max<int64_t>(nn, 1)),
        blist(ctx, std::max<int64_t>(nn, 1)), ctr(ctx, 64);  // two passes' counters (parity)
    DBuf<int2> mv(ctx, std::max<int64_t>(g->n, 1));
    DBuf<long long> result(ctx, 4), gain(ctx, 2);
    ctr.zero();
    gain.zero();
    // heaviest tiers first (longest-processing-time first over the work counter)
    int64_t pos = 0;
    for (int t = NUM_TIERS - 1; t >= 0; --t) {
        const int64_t cnt = g->tier_start[t + 1] - g->tier_start[t];
        if (cnt)
            CD_CUDA(cudaMemcpyAsync(order.p + pos, g->tlist.p + g->tier_start[t], cnt * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, ctx->stream));
        pos += cnt;
    }
    SweepParams P{};
    P.off = g->off.p;
    P.col = g->col.p;
    P.w = g->weighted ? g->w.p : nullptr;
    P.vol = g->vol.p;
    P.z = c.z;
    P.active = nullptr;
    P.vols = c.vols;
    P.csize = c.csize;
    P.gamma = c.gamma;
    P.inv_total = g->total > 0 ? 1.0 / g->total : 0.0;
    P.inv_sq2 = g->total > 0 ? 1.0 / (2.0 * g->total * g->total) : 0.0;
    P.guard = c.guard;
    P.buckets = c.buckets;
    P.own_lo = 0;
    P.own_hi = static_cast<int32_t>(g->n);
    P.mv = mv.p;
    P.stats = ctx->dstats + STAT_MODE_STRIDE;
    P.gain_fx = gain.p;
    SmallPhase S{};
    S.order = order.p;
    S.nn = static_cast<int32_t>(nn);
    S.bsel = bsel.p;
    S.blist = blist.p;
    S.ctr = ctr.p;
    S.seed = seed;
    S.salt = salt;
    S.K = c.buckets;
    S.max_passes = static_cast<int>(max_passes);
    S.theta = theta;
    S.stall = stall;
    S.qtol = qtol;
    S.gain = gain.p;
    S.cap_max = std::max<uint32_t>(64, static_cast<uint32_t>(next_pow2(static_cast<uint64_t>(2 * std::max<int64_t>(g->max_degree, 1)))));
    S.result = result.p;
    S.trace = std::getenv("CD_TRACE") != nullptr;
    const int vc = !g->weighted ? VC_COUNT : (g->int_weights ? VC_INT : VC_REAL);
    const size_t vbytes = vc == VC_REAL ? sizeof(double) : sizeof(unsigned int);
    const size_t smem = size_t(S.cap_max) * (vbytes + sizeof(int32_t)) + size_t(S.cap_max / 2) * sizeof(uint16_t);
    if (vc == VC_COUNT)
        launch_small<VC_COUNT>(ctx, P, S, smem);
    else if (vc == VC_INT)
        launch_small<VC_INT>(ctx, P, S, smem);
    else
        launch_small<VC_REAL>(ctx, P, S, smem);
    long long h[3];
    CD_CUDA(cudaMemcpyAsync(h, result.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (passes)
        *passes += h[0];
    if (moves)
        *moves += h[1];
    return h[2] != 0;
}

int64_t Sweeper::take_moves() {
    long long h = 0, gfx = 0;
    int32_t overflow = 0;
    CD_CUDA(cudaMemcpyAsync(&h, total_.p, sizeof(h), cudaMemcpyDeviceToHost, ctx_->stream));
    CD_CUDA(cudaMemsetAsync(total_.p, 0, sizeof(long long), ctx_->stream));
    if (exchange_)  // each rank summed its own movers' gains
        ctx_->comm->allreduce_sum_i64(ctx_, reinterpret_cast<int64_t *>(gain_.p), 1);
    CD_CUDA(cudaMemcpyAsync(&gfx, gain_.p, sizeof(gfx), cudaMemcpyDeviceToHost, ctx_->stream));
    CD_CUDA(cudaMemsetAsync(gain_.p, 0, sizeof(long long), ctx_->stream));
    if (g_->n_hubs) {
        const HubScratch *hs = hub_scratch_for(ctx_, g_);
        CD_CUDA(cudaMemcpyAsync(&overflow, hs ? hs->hp_flag.p : g_->hp_flag.p, sizeof(overflow),
                                cudaMemcpyDeviceToHost, ctx_->stream));
    }
    CD_CUDA(cudaStreamSynchronize(ctx_->stream));
    if (overflow)
        fail(CD_EINTERNAL, "hub partition table overflow (more distinct labels per partition than slots)");
    last_gain_fx_ = gfx;
    last_gain_ = static_cast<double>(gfx) / GAIN_FX_SCALE;
    return h;
}

}  // namespace cdk
