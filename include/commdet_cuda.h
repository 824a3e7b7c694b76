/*
 * commdet_cuda.h -- C ABI of the B200-native community-detection hot path.
 *
 * Drop-in boundary for the reference's detector interface
 * (/root/reference/proj/include/commdet, "H/" below).  Each entry point names
 * the reference function it replaces.  include/commdet/gpu.hpp wraps this ABI
 * in the reference's own C++ signatures and exception types; INTEGRATION.md
 * shows the bindings a maintainer adds.
 *
 * Conventions
 *  - node ids and community labels are int32 (n < 2^31), CSR offsets int64,
 *    stored edge weights fp32 (NULL = unweighted, weight 1.0), every sum that
 *    feeds a decision (tallies, volumes, modularity) is fp64 on the device.
 *  - every array argument may be a HOST pointer (pageable or pinned) or a
 *    DEVICE pointer on the context's GPU; the library detects which.  Host
 *    arguments are copied in / out inside the call (end-to-end use); device
 *    arguments are used in place (resident-in-HBM use).
 *  - calls are blocking (they return after the context stream is idle) and a
 *    context is not thread-safe: one cd_ctx per host thread.
 *  - errors: a cd_status code plus a thread-local message (cd_last_error).
 *    The C++ shim maps them back to the reference's exception types:
 *      CD_EINPUT  -> commdet::input_error      (H/graph.hpp:21-24)
 *      CD_EINVAL  -> std::invalid_argument
 *      CD_EDOMAIN -> std::domain_error
 *      CD_ERANGE  -> std::out_of_range
 */
#ifndef COMMDET_CUDA_H
#define COMMDET_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CD_API __attribute__((visibility("default")))

typedef enum cd_status {
    CD_OK = 0,
    CD_EINVAL = 1,
    CD_EDOMAIN = 2,
    CD_ERANGE = 3,
    CD_EINPUT = 4,
    CD_ENOMEM = 5,
    CD_ECUDA = 6,
    CD_ENCCL = 7,
    CD_EINTERNAL = 8
} cd_status;

typedef struct cd_ctx cd_ctx;
typedef struct cd_graph cd_graph;

enum { CD_ALGO_PLP = 0, CD_ALGO_PLM = 1, CD_ALGO_PLMR = 2 };

/* PlpConfig (H/plp.hpp:16-22).  randomize_order/workers are accepted for
 * source compatibility; the device order is the seeded bucket schedule. */
typedef struct cd_plp_config {
    int64_t theta;          /* <0: max(1, n/100000) (H/plp.hpp:24-28)        */
    int64_t max_iterations; /* 100                                            */
    int32_t randomize_order;
    int32_t workers;
    uint64_t seed;
    int32_t buckets; /* device: sub-sweeps per iteration (default 4)          */
    int32_t reserved;
} cd_plp_config;

/* LouvainConfig (H/louvain.hpp:15-22). */
typedef struct cd_louvain_config {
    double gamma;
    int64_t max_move_iterations; /* passes per move phase (32)               */
    int64_t max_levels;          /* 64                                       */
    uint64_t seed;
    int32_t workers;
    int32_t refine;          /* 0: PLM (run_plm), 1: PLMR (run_plmr)         */
    int32_t buckets;         /* device: sub-passes per pass; <= 0 (default): by graph,
                                8 if its max degree exceeds 4096, else 4     */
    int32_t singleton_guard; /* device: singleton->singleton only to smaller id */
    int64_t move_theta;      /* device: stop a move phase once a pass moves <= this;
                                <0: floor(n/100000) of the level's graph     */
    double move_tol;         /* device: ... or <= move_tol * n (0 disables)  */
    double move_stall;       /* device: ... or (from pass 8 on) when a pass moves more than
                                move_stall x the moves two passes earlier (0 disables) */
    int32_t prune;           /* device: re-evaluate a node only after a neighbour (or the node
                                itself) moved since its last evaluation; 1 (default) in the
                                input graph's move phases, 2 on every level, 0 never */
    int32_t reserved;
    double move_qtol;        /* device: ... or once a pass's summed gain is <= move_qtol x the
                                phase's summed gain so far (0 disables; < 0 (default): by
                                graph, 5e-3 if its max degree exceeds 4096, else 2e-3) */
} cd_louvain_config;

/* EnsembleConfig (H/ensemble.hpp:19-31), EPP(b, base, final). */
typedef struct cd_ensemble_config {
    int64_t ensemble_size;
    int32_t base;       /* CD_ALGO_*                                          */
    int32_t final_algo; /* CD_ALGO_*                                          */
    uint64_t seed;
    int32_t workers;
    int32_t reserved;
    cd_plp_config base_plp;
    cd_louvain_config final_louvain;
} cd_ensemble_config;

/* RunReport (H/report.hpp:26-41) with fixed-capacity traces. */
#define CD_MAX_ITERATION_RECORDS 1024
#define CD_MAX_LEVEL_RECORDS 64
typedef struct cd_iteration_record {
    int64_t updated;
    double ms;
} cd_iteration_record;
typedef struct cd_level_record {
    double move_ms, coarsen_ms, refine_ms;
    int64_t nodes, entries;   /* the level's graph                        */
    int64_t passes, moves;    /* move phase (+ refinement) passes and moves */
} cd_level_record;
typedef struct cd_report {
    char algorithm[16];
    int32_t workers;
    int32_t reserved;
    uint64_t seed;
    double total_ms;
    double modularity;
    double coverage;
    int64_t community_count;
    int64_t n_iterations;
    cd_iteration_record iterations[CD_MAX_ITERATION_RECORDS];
    int64_t n_levels;
    cd_level_record levels[CD_MAX_LEVEL_RECORDS];
    double base_ms, combine_ms, coarsen_ms, final_ms; /* EPP phases */
    int64_t kernel_launches;                          /* device launches in the call */
} cd_report;

typedef struct cd_graph_info {
    int64_t n;            /* node_count()        (H/graph.hpp:105) */
    int64_t D;            /* directed CSR entries                   */
    int64_t m;            /* edge_count()        (H/graph.hpp:106) */
    double total_weight;  /* total_edge_weight() (H/graph.hpp:107) */
    int32_t weighted;
    int32_t reserved;
    int64_t max_degree;
    int64_t isolated;
    /* row shard (cd_graph_shard): rows [own_lo, own_hi) of shard_rank / shard_size;
     * a whole graph reports 0 / 1 and [0, n).  D counts the local entries. */
    int32_t shard_rank, shard_size;
    int64_t own_lo, own_hi;
    int64_t D_global;
} cd_graph_info;

/* LFR-shaped benchmark spec (new generator; the reference has none). */
typedef struct cd_lfr_spec {
    int64_t n;
    double tau1, avg_degree;
    int32_t max_degree;
    double tau2;
    int32_t min_community, max_community;
    double mu;
} cd_lfr_spec;

/* Per-kernel-family device timing (CUDA events), enabled by cd_ctx_set_profiling. */
typedef struct cd_kernel_stat {
    char name[48];
    int64_t launches;
    double total_ms;
    double bytes; /* algorithmic bytes (DESIGN.md byte model)             */
    double items; /* nodes (sweeps) or entries processed                  */
} cd_kernel_stat;

/* ---- library / context --------------------------------------------------- */
CD_API const char *cd_last_error(void);
CD_API const char *cd_version(void);
CD_API void cd_plp_config_default(cd_plp_config *cfg);
CD_API void cd_louvain_config_default(cd_louvain_config *cfg);
/* The reference's stopping rule only (H/louvain.hpp:78, :136-137): a move
 * phase ends after a pass without moves or at max_move_iterations; every
 * non-isolated node is evaluated in every pass (no pruning).  The device
 * update order (buckets, singleton guard) is kept. */
CD_API void cd_louvain_config_reference(cd_louvain_config *cfg);
CD_API void cd_ensemble_config_default(cd_ensemble_config *cfg);
CD_API cd_status cd_ctx_create(int device, cd_ctx **out);
CD_API cd_status cd_ctx_destroy(cd_ctx *ctx);
CD_API cd_status cd_ctx_synchronize(cd_ctx *ctx);
CD_API cd_status cd_ctx_stream(cd_ctx *ctx, void **stream); /* cudaStream_t */
CD_API cd_status cd_ctx_set_profiling(cd_ctx *ctx, int enabled);
CD_API cd_status cd_ctx_reset_stats(cd_ctx *ctx);
CD_API cd_status cd_ctx_kernel_stats(cd_ctx *ctx, cd_kernel_stat *out, int32_t capacity, int32_t *count);
CD_API cd_status cd_ctx_launch_count(cd_ctx *ctx, int64_t *count);

/* ---- graphs (H/graph.hpp) ------------------------------------------------ */
/* Graph::from_edges (H/graph.hpp:48-81): validates endpoints and weights
 * (CD_EINPUT), symmetrises, sorts rows, duplicates -> CD_EINPUT unless
 * merge_duplicates (weights summed). */
CD_API cd_status cd_graph_from_edges(cd_ctx *ctx, int64_t n, int64_t m, const int32_t *u, const int32_t *v,
                                     const float *w, int32_t merge_duplicates, cd_graph **out);
/* Canonical symmetric CSR (rows strictly ascending).  Rows are validated
 * (range, order, weight > 0); symmetry is the caller's contract. */
CD_API cd_status cd_graph_from_csr(cd_ctx *ctx, int64_t n, const int64_t *off, const int32_t *col, const float *w,
                                   cd_graph **out);
/* generate_planted (H/generator.hpp:52-104), bit-exact edge set. */
CD_API cd_status cd_graph_generate_planted(cd_ctx *ctx, int64_t n, int64_t k, double p_in, double p_out,
                                           uint64_t seed, cd_graph **out, int32_t *truth);
/* Seeded R-MAT: symmetrised, deduplicated, no self-loops; weighted graphs get
 * dyadic weights (k+1)*2^-24, k uniform in [0, 2^24). */
CD_API cd_status cd_graph_generate_rmat(cd_ctx *ctx, int32_t scale, int32_t edge_factor, double a, double b,
                                        double c, int32_t weighted, uint64_t seed, cd_graph **out);
/* Seeded LFR-shaped graph (configuration-model style). */
CD_API cd_status cd_graph_generate_lfr(cd_ctx *ctx, const cd_lfr_spec *spec, uint64_t seed, cd_graph **out,
                                       int32_t *truth);
CD_API cd_status cd_graph_get_info(const cd_graph *g, cd_graph_info *out);
/* Any output may be NULL.  w is written only for weighted graphs. */
CD_API cd_status cd_graph_download(const cd_graph *g, int64_t *off, int32_t *col, float *w, double *vol,
                                   double *loop);
CD_API cd_status cd_graph_destroy(cd_graph *g);

/* ---- quality (H/quality.hpp) -------------------------------------------- */
/* modularity(g, z, gamma) (:35-51) and coverage(g, z) (:21-31).  Labels must
 * lie in [0, ub) (CD_ERANGE otherwise); w(E) == 0 -> CD_EDOMAIN, coverage 0. */
CD_API cd_status cd_modularity(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double gamma,
                               double *modularity, double *coverage);
/* graph_rand_index (H/quality.hpp:56-69): fraction of edges on which the two
 * partitions agree; w(E)-independent; CD_EDOMAIN for an edgeless graph. */
CD_API cd_status cd_rand_index(cd_ctx *ctx, const cd_graph *g, const int32_t *a, const int32_t *b, double *out);
/* community_volumes (H/louvain.hpp:27-31) */
CD_API cd_status cd_community_volumes(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double *vols);

/* ---- partitions (H/partition.hpp, H/louvain.hpp, H/ensemble.hpp) ---------- */
/* Partition::compacted (H/partition.hpp:39-53): first-appearance order. */
CD_API cd_status cd_compact(cd_ctx *ctx, int64_t n, const int32_t *z, int32_t *out, int64_t *k);
/* Partition::community_count (H/partition.hpp:55-60). */
CD_API cd_status cd_community_count(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t *k);
/* coarsen (H/louvain.hpp:154-220): z must be compact (CD_EINVAL otherwise);
 * pi_out (nullable) receives pi = z. */
CD_API cd_status cd_coarsen(cd_ctx *ctx, const cd_graph *g, const int32_t *z, cd_graph **coarse, int32_t *pi_out);
/* prolong (H/louvain.hpp:223-233): CD_ERANGE if pi[v] >= nc. */
CD_API cd_status cd_prolong(cd_ctx *ctx, int64_t nc, const int32_t *z_coarse, int64_t n, const int32_t *pi,
                            int32_t *out);
/* combine_hashed (H/ensemble.hpp:86-107): djb2 over 8 LE bytes per id. */
CD_API cd_status cd_combine_hashed(cd_ctx *ctx, int64_t b, int64_t n, const int32_t *const *solutions,
                                   int32_t *out, int64_t *k);

/* ---- deterministic sub-kernels (parity surface) --------------------------- */
/* One synchronous PLP sweep: z_out[u] = dominant_label(g, z_in, u)
 * (H/plp.hpp:32-53) for every u with deg > 0, else z_in[u]. */
CD_API cd_status cd_plp_sweep_sync(cd_ctx *ctx, const cd_graph *g, const int32_t *z_in, int32_t *z_out,
                                   int64_t *updated);
/* One synchronous move evaluation against frozen (z, vols): the decision
 * rule of move_phase (H/louvain.hpp:91-120) for every node.  best[u] = z[u]
 * and gain 0 for non-movers.  ub bounds the labels and sizes vols. */
CD_API cd_status cd_move_eval(cd_ctx *ctx, const cd_graph *g, const int32_t *z, const double *vols, int64_t ub,
                              double gamma, int32_t *best, double *gain);
/* move_phase (H/louvain.hpp:65-141) with the device's bucketed order. */
CD_API cd_status cd_move_phase(cd_ctx *ctx, const cd_graph *g, int32_t *z, const cd_louvain_config *cfg,
                               int32_t *changed);
/* MoveObserver (H/louvain.hpp:60): called after each applied move with
 * (node, source community, target community, predicted gain). */
typedef void (*cd_move_observer)(void *user, int32_t node, int32_t source, int32_t target, double gain);
/* move_phase (H/louvain.hpp:65-141) in the reference's one-worker order:
 * u = 0..n-1, each move applied before the next node is evaluated; a pass
 * without moves or cfg->max_move_iterations passes end it (cfg->gamma and
 * the pass cap are the only fields read).  Labels in [0, ub).  observer
 * (nullable) receives every applied move in order; the calls of a pass
 * arrive when that pass has finished on the device.  z is written when the
 * phase ends.  A serial test / debugging path (one warp walks the nodes). */
CD_API cd_status cd_move_phase_sequential(cd_ctx *ctx, const cd_graph *g, int32_t *z, int64_t ub,
                                          const cd_louvain_config *cfg, cd_move_observer observer, void *user,
                                          int32_t *changed);

/* ---- detectors (H/plp.hpp:67, H/louvain.hpp:290/297, H/ensemble.hpp:111) -- */
/* run_plp: labels raw (not compacted), like the reference (H/plp.hpp:148). */
CD_API cd_status cd_plp_run(cd_ctx *ctx, const cd_graph *g, const cd_plp_config *cfg, const int32_t *initial,
                            int32_t *labels, cd_report *report);
/* run_plm (cfg->refine == 0) / run_plmr (cfg->refine != 0); z compacted. */
CD_API cd_status cd_louvain_run(cd_ctx *ctx, const cd_graph *g, const cd_louvain_config *cfg, int32_t *z,
                                cd_report *report);
/* run_epp; z compacted. */
CD_API cd_status cd_epp_run(cd_ctx *ctx, const cd_graph *g, const cd_ensemble_config *cfg, int32_t *z,
                            cd_report *report);
/* run_epp with EnsembleConfig::base_override (H/ensemble.hpp:30, :127-128):
 * bases[i] (i < cfg->ensemble_size; n labels each, host or device memory)
 * replace the base detector's runs; combine, coarsen, final solver and
 * prolongation are run_epp's. */
CD_API cd_status cd_epp_run_bases(cd_ctx *ctx, const cd_graph *g, const cd_ensemble_config *cfg,
                                  const int32_t *const *bases, int32_t *z, cd_report *report);

/* ---- text ingest (H/io.hpp) ------------------------------------------------
 * The file's bytes (host or device memory) are parsed on the device with the
 * reference reader's rules and errors (CD_EINPUT + message). */
/* io::read_metis (H/io.hpp:83-165): header "n m [fmt]", '%' comments. */
CD_API cd_status cd_graph_read_metis(cd_ctx *ctx, const char *text, int64_t len, cd_graph **out);
/* io::read_edge_list (H/io.hpp:190-237): "u v [w]" lines, '#' comments, ids
 * densified in ascending order (cd_graph_original_ids). */
CD_API cd_status cd_graph_read_edge_list(cd_ctx *ctx, const char *text, int64_t len, int32_t merge_duplicates,
                                         cd_graph **out);
/* Same, reading the file at `path` first ("cannot open <path>" -> CD_EINPUT). */
CD_API cd_status cd_graph_load_metis(cd_ctx *ctx, const char *path, cd_graph **out);
CD_API cd_status cd_graph_load_edge_list(cd_ctx *ctx, const char *path, int32_t merge_duplicates, cd_graph **out);
/* The original id of every dense node of an edge-list graph (n entries). */
CD_API cd_status cd_graph_original_ids(const cd_graph *g, uint64_t *out);

/* ---- sharded execution --------------------------------------
 * One rank per GPU.  Attach a communicator to each rank's context; every
 * detector then evaluates only the rank's nodes (1D degree-balanced ranges,
 * cd_shard_bounds) and exchanges the per-sub-sweep move lists, so labels stay
 * replicated and equal to the one-device result.  The graph may be whole on
 * every rank (replicated) or a row shard (cd_graph_shard: owned rows only);
 * coarse levels are replicated.  Outputs are the full labels on every rank.
 * The reference's equivalent is its OpenMP `workers` (H/graph.hpp:34-36). */
typedef struct cd_loopback cd_loopback;
/* ncclGetUniqueId (libnccl.so.2 is loaded on first use). */
CD_API cd_status cd_nccl_unique_id(uint8_t id[128]);
/* ncclCommInitRank on the context's device; collective across the ranks. */
CD_API cd_status cd_ctx_attach_nccl(cd_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);
/* In-process emulation: nranks host threads, each with its own context on
 * one device, exchange through host barriers and device copies. */
CD_API cd_status cd_loopback_create(int32_t nranks, cd_loopback **out);
CD_API cd_status cd_loopback_destroy(cd_loopback *lb);
CD_API cd_status cd_ctx_attach_loopback(cd_ctx *ctx, cd_loopback *lb, int32_t rank);
CD_API cd_status cd_ctx_detach(cd_ctx *ctx);
CD_API cd_status cd_ctx_world(const cd_ctx *ctx, int32_t *rank, int32_t *size);
/* Ownership ranges: bounds[r] = first node whose offset reaches D*r/nranks
 * (host offsets, n+1 entries; bounds has nranks+1 entries).  No GPU needed. */
CD_API cd_status cd_shard_bounds(int64_t n, const int64_t *off, int32_t nranks, int64_t *bounds);
/* This rank's row shard of a whole graph (ranges of cd_shard_bounds). */
CD_API cd_status cd_graph_shard(cd_ctx *ctx, const cd_graph *full, cd_graph **out);
/* This rank's row shard straight from its own rows (no rank ever holds the
 * whole CSR): off = the whole graph's offsets (n+1, host or device), [lo, hi)
 * = this rank's range, which must equal cd_shard_bounds(off, world)[rank..];
 * col / w = the off[hi] - off[lo] entries of rows [lo, hi) (w NULL =
 * unweighted).  Rows are validated as in cd_graph_from_csr; node volumes,
 * loops, m and w(E) are summed over the ranks.  Collective over the
 * context's ranks; with no communicator it is cd_graph_from_csr. */
CD_API cd_status cd_graph_from_csr_rows(cd_ctx *ctx, int64_t n, const int64_t *off, int64_t lo, int64_t hi,
                                        const int32_t *col, const float *w, cd_graph **out);
/* This rank's row shard of the seeded R-MAT graph (cd_graph_generate_rmat),
 * built without ever holding the whole graph: rank r keeps the rows whose
 * raw (pre-deduplication) adjacency splits the stream evenly, i.e.
 * cd_shard_bounds over the raw adjacency lengths.  Collective over the
 * context's ranks; with no communicator it is cd_graph_generate_rmat.  Both
 * build in row chunks of bounded scratch (C5: scale 28 on one GPU). */
CD_API cd_status cd_graph_generate_rmat_shard(cd_ctx *ctx, int32_t scale, int32_t edge_factor, double a, double b,
                                              double c, int32_t weighted, uint64_t seed, cd_graph **out);

#ifdef __cplusplus
}
#endif

#endif /* COMMDET_CUDA_H */
