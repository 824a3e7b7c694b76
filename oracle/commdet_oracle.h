/*
 * commdet_oracle.h -- CPU oracle for the B200 community-detection hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1304_4453_b200/,
 * include/) may link, call or load this library.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it, and only as the checker.
 *
 * Two kinds of functions live here:
 *
 *  (1) Restatements of the reference algorithm (the headers under
 *      /root/reference/proj/include/commdet, abbreviated H/ below).  Each cites the file:line it
 *      follows.  These are pinned against the reference itself (compiled into
 *      oracle/_ref/ by oracle/Makefile) and against the reference's own KATs
 *      (tests/golden/, tests/test_oracle_*.py).
 *
 *  (2) Ports of the device algorithm's deterministic update order (the
 *      hash-bucketed semi-synchronous PLP / PLM drivers and the synthetic
 *      R-MAT / LFR-shaped generators, which the reference does not have).
 *      They let the GPU tests demand bit-exact end-to-end labels, while the
 *      reference (oracle/_ref) pins quality to +-0.005 modularity.
 *
 * Conventions: node ids and labels are int32 (n < 2^31), CSR offsets int64,
 * weights double (the reference's edgeweight, H/graph.hpp:18).  Unless noted
 * a function returns 0 on success and a negative CDO_* code on error.
 */
#ifndef COMMDET_ORACLE_H
#define COMMDET_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CDO_OK = 0,
    CDO_EINPUT = -1,  /* input_error   (H/graph.hpp:21-24)            */
    CDO_EINVAL = -2,  /* invalid_argument                             */
    CDO_EDOMAIN = -3, /* domain_error  (w(E) == 0)                    */
    CDO_ERANGE = -4,  /* out_of_range                                 */
    CDO_ENOMEM = -5
};

/* Host CSR graph, same conventions as H/graph.hpp:38-40, :263-267. */
typedef struct {
    int64_t n;      /* nodes                                   */
    int64_t D;      /* directed CSR entries                    */
    int64_t m;      /* undirected edges incl. loops (H/graph.hpp:241-249) */
    double total;   /* w(E)                                    */
    int64_t *off;   /* n+1                                     */
    int32_t *col;   /* D, rows ascending                       */
    double *w;      /* D                                       */
    double *vol;    /* n, loop counted twice (H/graph.hpp:240-243) */
    double *loop;   /* n                                       */
} cdo_graph;

void cdo_graph_free(cdo_graph *g);

/* ---- graph construction (H/graph.hpp:48-81, 85-103, 169-255) ---------- */
int cdo_graph_from_edges(int64_t n, int64_t m, const int32_t *eu, const int32_t *ev, const double *ew,
                         int merge_duplicates, cdo_graph *out);
/* Wrap an already canonical CSR (copies); recomputes finalize(). */
int cdo_graph_from_csr(int64_t n, const int64_t *off, const int32_t *col, const double *w, cdo_graph *out);
void cdo_finalize(cdo_graph *g);

/* ---- generators ------------------------------------------------------- */
uint64_t cdo_splitmix64(uint64_t x);                     /* H/generator.hpp:24-29 */
double cdo_row_uniform(uint64_t key, uint64_t v);        /* H/generator.hpp:35-37 */
/* H/generator.hpp:52-104; truth may be NULL. */
int cdo_generate_planted(int64_t n, int64_t k, double p_in, double p_out, uint64_t seed, cdo_graph *out,
                         int32_t *truth);
/* Device R-MAT generator port (not in the reference). */
int cdo_generate_rmat(int scale, int edge_factor, double a, double b, double c, int weighted, uint64_t seed,
                      cdo_graph *out);
/* Device LFR-shaped generator port (not in the reference). */
typedef struct {
    int64_t n;
    double tau1, avg_degree;
    int32_t max_degree;
    double tau2;
    int32_t min_community, max_community;
    double mu;
} cdo_lfr_spec;
int cdo_generate_lfr(const cdo_lfr_spec *spec, uint64_t seed, cdo_graph *out, int32_t *truth);

/* ---- quality (H/quality.hpp:21-51) ------------------------------------ */
int cdo_modularity(const cdo_graph *g, const int32_t *z, int64_t ub, double gamma, double *q);
double cdo_coverage(const cdo_graph *g, const int32_t *z);
void cdo_community_volumes(const cdo_graph *g, const int32_t *z, int64_t ub, double *vols); /* H/louvain.hpp:27-31 */

/* ---- partition (H/partition.hpp:39-60) -------------------------------- */
int64_t cdo_compact(int64_t n, const int32_t *z, int32_t *out); /* returns k */
int64_t cdo_community_count(int64_t n, const int32_t *z);

/* ---- PLP (H/plp.hpp:32-53, 111-126) ----------------------------------- */
int cdo_dominant_label(const cdo_graph *g, const int32_t *z, int32_t u, int32_t *out);
/* One synchronous sweep: every node with deg>0 takes dominant_label against
 * the frozen z_in.  Dense-scratch restatement of H/plp.hpp:111-126. */
int64_t cdo_plp_sweep_sync(const cdo_graph *g, const int32_t *z_in, int32_t *z_out);
int cdo_is_stable(const cdo_graph *g, const int32_t *z); /* H/plp.hpp:57-62 */

/* ---- Louvain (H/louvain.hpp) ------------------------------------------ */
double cdo_delta_mod(const cdo_graph *g, const int32_t *z, const double *vols, int32_t u, int32_t target,
                     double gamma); /* H/louvain.hpp:37-56 */
/* One synchronous move evaluation against frozen (z, vols): best target of
 * every node (H/louvain.hpp:91-120 decision rule) and its gain; isolated
 * nodes and non-movers return best = z[u], gain 0. */
void cdo_move_eval(const cdo_graph *g, const int32_t *z, const double *vols, int64_t ub, double gamma,
                   int32_t *best, double *gain);
/* Applied moves of a sequential move phase, in order (the MoveObserver's
 * arguments, H/louvain.hpp:60, :127-128).  count may exceed capacity. */
typedef struct {
    int32_t *node, *source, *target;
    double *gain;
    int64_t capacity, count;
} cdo_move_log;
/* move_phase (H/louvain.hpp:65-141) with workers == 1: u = 0..n-1 in place. */
int cdo_move_phase_sequential(const cdo_graph *g, int32_t *z, int64_t ub, double gamma, int64_t max_passes,
                              cdo_move_log *log, int32_t *changed);
/* H/louvain.hpp:154-220 (coarse weights double). Returns CDO_EINVAL if z is
 * not compact. */
int cdo_coarsen(const cdo_graph *g, const int32_t *z, cdo_graph *coarse);
int cdo_prolong(int64_t nc, const int32_t *zc, int64_t n, const int32_t *pi, int32_t *out); /* :223-233 */

/* ---- ensemble (H/ensemble.hpp:75-107) --------------------------------- */
uint64_t cdo_djb2(const uint8_t *data, uint64_t len);
int64_t cdo_combine_hashed(int64_t b, int64_t n, const int32_t *const *solutions, int32_t *out);

/* ---- ports of the device drivers (bucketed semi-synchronous order) ---- */
typedef struct {
    int64_t theta; /* <0: max(1, n/100000) (H/plp.hpp:24-28) */
    int64_t max_iterations;
    uint64_t seed;
    int32_t buckets;
} cdo_plp_config;

typedef struct {
    double gamma;
    int64_t max_move_iterations;
    int64_t max_levels;
    uint64_t seed;
    int32_t buckets;
    int32_t refine;
    int32_t singleton_guard;
    int64_t move_theta; /* <0: floor(n/100000) per level */
    double move_tol;    /* stop also once a pass moves <= move_tol * n */
    double move_stall;  /* ... or (pass >= 8) moves > move_stall * moves two passes earlier */
    int32_t prune;      /* evaluate only nodes whose neighbourhood changed (device prune):
                           1 = level-0 move phases, 2 = every level */
    double move_qtol;   /* ... or a pass's summed gain <= move_qtol x the phase's (fixed point 2^-44) */
} cdo_louvain_config;

/* bucket key / id: the order every device driver uses. */
uint64_t cdo_bucket_key(uint64_t seed, uint64_t salt);
int32_t cdo_bucket_of(uint64_t key, int32_t u, int32_t buckets);

int cdo_plp_bucketed(const cdo_graph *g, const cdo_plp_config *cfg, const int32_t *initial, int32_t *labels,
                     int64_t *iterations, int64_t *updated_trace, int64_t trace_cap);
int cdo_move_phase_bucketed(const cdo_graph *g, int32_t *z, const cdo_louvain_config *cfg, uint64_t salt,
                            int32_t *changed);
int cdo_louvain_bucketed(const cdo_graph *g, const cdo_louvain_config *cfg, int32_t *z, int64_t *k,
                         int64_t *levels);
/* Sharded protocol: one sub-sweep over the owned nodes
 * [lo, hi); returns the number of moves written (not applied). */
int64_t cdo_plp_subsweep(const cdo_graph *g, const int32_t *labels, uint8_t *active, uint64_t key, int32_t bucket,
                         int32_t buckets, int64_t lo, int64_t hi, int32_t *mv_u, int32_t *mv_l);
int64_t cdo_move_subsweep(const cdo_graph *g, const int32_t *z, const double *vols, const int32_t *csize,
                          uint8_t *active, const cdo_louvain_config *cfg, uint64_t key, int32_t bucket, int64_t lo,
                          int64_t hi, int32_t *mv_u, int32_t *mv_l, long long *gain_fx);
/* Activation after a sub-sweep's moves (PLP and pruned PLM): all nodes when
 * more than n/16 moved, else the neighbours of the moved nodes. */
void cdo_activate(const cdo_graph *g, int64_t nm, const int32_t *mv_u, uint8_t *active);
int cdo_epp_bucketed(const cdo_graph *g, int64_t ensemble_size, uint64_t seed, const cdo_plp_config *base,
                     const cdo_louvain_config *final_cfg, int32_t *z, int64_t *k);

#ifdef __cplusplus
}
#endif

#endif
