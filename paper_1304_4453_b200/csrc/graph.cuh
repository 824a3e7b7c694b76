// graph.cuh -- device-resident CSR graph (the reference's Graph,
// H/graph.hpp:38-272, laid out for HBM) and its work decomposition.
//
// HBM layout per graph (n nodes, D directed entries):
//   off  int64[n+1]   row offsets (int64: C5 has D ~ 8.5e9)
//   col  int32[D]     neighbour ids, rows strictly ascending (H/graph.hpp:177)
//   w    fp32[D]      only for weighted graphs (unweighted => 1.0 implied)
//   vol  fp64[n]      weighted degree, self-loop twice (H/graph.hpp:240-243)
//   loop fp64[n]      self-loop weight
// Work decomposition (built once per graph, lazily):
//   tier  uint8[n]    degree tier of each node (255 = isolated)
//   hubs  int32[H]    nodes of the hub tier, with a global hash region each
#pragma once

#include "common.cuh"

namespace cdk {

// Degree tiers of the sweep / move kernels.
enum Tier : int {
    TIER_G8 = 0,      // deg <= 8      : 8 lanes per node (4 nodes / warp)
    TIER_G16 = 1,     // deg <= 16     : 16 lanes per node
    TIER_G32 = 2,     // deg <= 32     : one warp per node, one pass
    TIER_WARP = 3,    // deg <= 256    : one warp per node, per-warp smem hash
    TIER_BLOCK = 4,   // deg <= 1024   : one block per node, 2048-slot smem hash
    TIER_BLOCK2 = 5,  // deg <= 4096   : one block per node, 8192-slot smem hash
    TIER_BLOCK3 = 6,  // deg <= 8192   : one 1024-thread block per node, 16384-slot smem hash
    TIER_CLUSTER = 7, // deg <= 32768  : one 4-CTA cluster per node, hash table in distributed smem
                      //                 (integer tallies only; fp64 graphs use HUB)
    TIER_HUB = 8,     // larger        : hash-partitioned multi-block tally
    NUM_TIERS = 9,
    TIER_NONE = 255
};
constexpr int WARP_TABLE_CAP = 512;     // per-warp smem hash slots (>= 2*256)
constexpr int BLOCK_TABLE_CAP = 2048;   // >= 2*1024
constexpr int BLOCK2_TABLE_CAP = 8192;  // >= 2*4096
constexpr int BLOCK3_TABLE_CAP = 16384; // >= 2*8192
constexpr int HUB_CHUNK = 4096;         // entries per hub chunk block
constexpr int HUB_PART = 512;           // target pairs per hub partition
constexpr int HUB_PART_CAP = 2048;      // smem slots of a partition block (4x HUB_PART)
constexpr int HUB_MAX_PBITS = 13;       // partitions per hub <= 8192 (smem histogram)
// partitions of a hub of degree d: 2^bits with HUB_PART << bits >= d
__host__ __device__ inline int hub_pbits_of(int64_t d) {
    int b = 0;
    while ((int64_t(HUB_PART) << b) < d && b < HUB_MAX_PBITS)
        ++b;
    return b;
}

#ifndef CD_CLUSTER_N
#define CD_CLUSTER_N 4
#endif
constexpr int CLUSTER_CTAS = CD_CLUSTER_N;                      // CTAs per node (16384 slots each)
constexpr int64_t CLUSTER_MAX_DEG = int64_t(CLUSTER_CTAS) * 8192;  // <= 50 % table load

// cluster_max: CLUSTER_MAX_DEG, or 0 when the cluster tier is not used
__host__ __device__ inline int tier_of_degree(int64_t d, int64_t cluster_max = CLUSTER_MAX_DEG) {
    if (d <= 0)
        return TIER_NONE;
    if (d <= 8)
        return TIER_G8;
    if (d <= 16)
        return TIER_G16;
    if (d <= 32)
        return TIER_G32;
    if (d <= 256)
        return TIER_WARP;
    if (d <= 1024)
        return TIER_BLOCK;
    if (d <= 4096)
        return TIER_BLOCK2;
    if (d <= 8192)
        return TIER_BLOCK3;
    if (d <= cluster_max)
        return TIER_CLUSTER;
    return TIER_HUB;
}

// Tally value class of a graph: 0 unweighted (counts), 1 integral weights
// whose row sums fit uint32 (exact integer tallies, native smem atomics),
// 2 general fp32 weights (fp64 tallies).
enum ValueClass : int { VC_COUNT = 0, VC_INT = 1, VC_REAL = 2 };

}  // namespace cdk

struct cd_graph {
    cd_ctx *ctx = nullptr;
    int64_t n = 0, D = 0, m = 0;
    double total = 0.0;
    bool weighted = false;
    bool int_weights = false;  // every weight integral and max vol < 2^31 (finalize)
    double max_vol = 0.0;
    int64_t max_degree = 0, isolated = 0;
    cdk::DBuf<int64_t> off;
    cdk::DBuf<int32_t> col;
    cdk::DBuf<float> w;
    cdk::DBuf<double> vol, loop;

    // work decomposition: every non-isolated node listed once, grouped by
    // tier, ascending id within a tier (stable partition by scan)
    bool binned = false;
    cdk::DBuf<uint8_t> tier;
    int64_t tier_nodes[cdk::NUM_TIERS] = {};
    int64_t tier_start[cdk::NUM_TIERS + 1] = {};
    cdk::DBuf<int32_t> tlist;  // [tier_start[NUM_TIERS]]
    // hub tier: a static chunk grid (HUB_CHUNK entries per block) and a
    // hash-partitioned pair scratch.  Hub h owns 2^hub_pbits[h] partitions
    // [hub_pbase[h], hub_pbase[h+1]) of about HUB_PART pairs each.
    int64_t n_hubs = 0, n_hub_chunks = 0, n_hub_parts = 0, hub_entries = 0;
    const int32_t *hubs = nullptr;  // [n_hubs] node ids (view into tlist)
    cdk::DBuf<int32_t> chunk_hub;   // [n_hub_chunks]
    cdk::DBuf<int32_t> chunk_part;  // [n_hub_chunks] chunk index within hub
    cdk::DBuf<int32_t> hub_pbits;   // [n_hubs]
    cdk::DBuf<int64_t> hub_pbase;   // [n_hubs + 1]
    cdk::DBuf<int32_t> part_hub;    // [n_hub_parts]
    cdk::DBuf<int32_t> hp_cnt;      // [n_hub_parts] pairs per partition (per sub-sweep)
    cdk::DBuf<int32_t> hp_cur;      // [n_hub_parts] scatter cursors
    cdk::DBuf<int64_t> hp_start;    // [n_hub_parts + 1]
    cdk::DBuf<int32_t> hp_key;      // [hub_entries] partitioned (label, weight) pairs
    cdk::DBuf<double> hp_val;       // [hub_entries]
    cdk::DBuf<int32_t> st_key;      // [hub_entries] the count pass's pairs, chunk-major (staging)
    cdk::DBuf<double> st_val;       // [hub_entries]
    cdk::DBuf<int32_t> chunk_np;    // [n_hub_chunks] pairs staged per chunk
    cdk::DBuf<double> hp_best_val;  // [n_hub_parts] per-partition best candidate
    cdk::DBuf<double> hp_second;    // [n_hub_parts] its runner-up (PLP margins)
    cdk::DBuf<int32_t> hp_best_key; // [n_hub_parts]
    cdk::DBuf<int64_t> hp_scan;     // scan scratch (2 x tiles)
    cdk::DBuf<int32_t> hp_flag;     // partition table overflow (sticky)
    cdk::DBuf<double> hub_aux;      // [n_hubs] per-hub w(u, C) accumulator (PLM)

    // row shard (comm.cuh): only rows [own_lo, own_hi) carry
    // entries (global column ids); every other row is empty.  vol, loop, m,
    // total, max_degree, isolated, int_weights and max_vol are the GLOBAL
    // graph's; D counts the local entries.  toff/tcol (built on first PLP use)
    // is the transposed block: for every node, its owned neighbours.
    bool rows_local = false;
    int shard_rank = 0, shard_size = 1;
    int64_t own_lo = 0, own_hi = 0;
    int64_t D_global = 0;
    cdk::DBuf<int64_t> toff;
    cdk::DBuf<int32_t> tcol;

    // edge-list ingest: dense id -> original id (ascending; H/io.hpp:220-235)
    cdk::DBuf<uint64_t> orig_ids;
};

namespace cdk {

// Duplicate handling of the row engine (H/graph.hpp:178-194).
enum DupMode : int { DUP_ERROR = 0, DUP_SUM = 1, DUP_ONE = 2 };

// graph.cu
// vol, loop, m, total, max degree.  integral_weights: the caller knows every
// weight is an integer (contraction of an integer-weight graph), so sums are
// order-free and computed entry-parallel
void graph_finalize(cd_ctx *ctx, cd_graph *g, bool integral_weights = false);
// Host columns (and weights) -> device in chunks of UPLOAD_CHUNK entries on
// the context's copy stream, each chunk validated (graph_validate_csr's
// checks) on the library stream while the next one copies; off_dev is already
// enqueued on the library stream.  Throws CD_EINPUT like graph_validate_csr.
constexpr int64_t UPLOAD_CHUNK = int64_t(1) << 25;        // largest chunk (128 MB of columns)
constexpr int64_t UPLOAD_MIN_ENTRIES = int64_t(1) << 22;  // chunked from 16 MB of columns
// about eight chunks for a mid-size graph (C2: 18.3M entries in five chunks of
// 2^22), so its checks, finalize and tiers also hide behind the copy
inline int64_t upload_chunk(int64_t D) {
    int64_t c = int64_t(1) << 21;
    while (c < UPLOAD_CHUNK && c * 8 < D)
        c <<= 1;
    return c;
}
// With g (an unweighted graph being built: n, D, off, col set), the upload
// also finalizes it -- every chunk's pass counts its self-loops and upper
// entries -- and builds its degree tiers from the offsets while the columns
// are still copying; g is then complete (graph_finalize is not needed).
void graph_upload_validate(cd_ctx *ctx, int64_t n, int64_t D, const int64_t *off_dev, int32_t *col_dev,
                           const int32_t *col_host, float *w_dev, const float *w_host, cd_graph *g = nullptr);
// row batching: cut[i] = first row in [lo, hi] whose prefix reaches an even
// split of [pre[lo], pre[hi]) into k parts (cut has k+1 entries)
__global__ void k_split_rows(const int64_t *pre, int64_t lo, int64_t hi, int k, int64_t *cut);
// dst[i] = src[i] - sub + add
__global__ void k_rebase(int64_t cnt, const int64_t *src, int64_t sub, int64_t add, int64_t *dst);
__global__ void k_fill_i64(int64_t cnt, int64_t value, int64_t *dst);
// host: the row batches of [lo, hi) holding at most ~`chunk` prefix units each
std::vector<int64_t> split_rows(cd_ctx *ctx, const int64_t *pre_dev, int64_t lo, int64_t hi, int64_t chunk);
// The hub tier's per-sub-sweep scratch.  A graph owns one (its hp_* fields);
// a child context running concurrently with others on the same graph gets a
// private copy (nullptr: use the graph's).
struct HubScratch {
    DBuf<int32_t> hp_cnt, hp_cur, hp_key, hp_best_key, hp_flag, st_key, chunk_np;
    DBuf<int64_t> hp_start, hp_scan;
    DBuf<double> hp_val, hp_best_val, hp_second, hub_aux, st_val;
};
HubScratch *hub_scratch_for(cd_ctx *ctx, const cd_graph *g);
// a context for one concurrent run on the parent's device (own stream,
// counters and hub scratch); ctx_child_destroy adds its launches to the parent
cd_ctx *ctx_child(const cd_ctx *parent);
void ctx_child_destroy(cd_ctx *parent, cd_ctx *child);
// free the tier lists and hub scratch (rebuilt on demand by graph_ensure_bins)
void graph_release_bins(cd_graph *g);
// graphs at least this large drop their work decomposition between phases
constexpr int64_t BIG_GRAPH_ENTRIES = int64_t(1) << 31;
// rows [lo, hi) built and finalized locally -> row shard with global node state
void shard_globalize(cd_ctx *ctx, cd_graph *g, int64_t lo, int64_t hi);
void graph_ensure_bins(cd_ctx *ctx, cd_graph *g);
cd_graph *graph_from_pairs(cd_ctx *ctx, int64_t n, int64_t m, const int32_t *u, const int32_t *v, const float *w,
                           DupMode mode);  // device arrays; symmetrises
void graph_validate_csr(cd_ctx *ctx, int64_t n, const int64_t *off, const int32_t *col, const float *w, int64_t D);

// text.cu (H/io.hpp:83-165, :190-237); `name` prefixes error messages
cd_graph *read_metis_dev(cd_ctx *ctx, const char *text, int64_t len, const std::string &name);
cd_graph *read_edge_list_dev(cd_ctx *ctx, const char *text, int64_t len, bool merge, const std::string &name);

// shard.cu
cd_graph *graph_shard_dev(cd_ctx *ctx, const cd_graph *full);  // rows of this rank (ctx->comm)
void graph_ensure_transpose(cd_ctx *ctx, cd_graph *g);         // toff / tcol of a row shard
// ownership range of this rank on a replicated graph (whole graph on one device)
void owned_range(cd_ctx *ctx, const cd_graph *g, int64_t &lo, int64_t &hi);
// sum of the row-shard partial coarse graphs of all ranks (replicated result)
cd_graph *coarsen_sharded_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc, bool sorted = true);

// quality.cu
void community_volumes_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, double *vols, int64_t ub);
// vols and sizes without range checks (driver-internal labels, always < ub)
void community_volumes_sizes_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, double *vols, int32_t *csize,
                                 int64_t ub);
void modularity_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double gamma, double *q,
                    double *cov);
double rand_index_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *a, const int32_t *b);

// partition.cu
int64_t max_label_dev(cd_ctx *ctx, int64_t n, const int32_t *z);  // max+1 (>= 1); -1 if a label < 0
int64_t compact_dev(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t ub, int32_t *out);
void prolong_dev(cd_ctx *ctx, int64_t nc, const int32_t *zc, int64_t n, const int32_t *pi, int32_t *out);
int64_t combine_hashed_dev(cd_ctx *ctx, int64_t b, int64_t n, const int32_t *const *sols_dev, int32_t *out);
void iota_dev(cd_ctx *ctx, int32_t *z, int64_t n);

// coarsen.cu.  sorted: rows ascending (the reference's CSR convention, the
// API); the detectors pass false -- their tallies do not depend on row order
// and the per-row sort is a third of a large contraction
cd_graph *coarsen_dev(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t nc, bool sorted = true);

}  // namespace cdk
