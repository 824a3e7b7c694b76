// detect.cuh -- device drivers of the detectors (run_plp, move_phase,
// run_plm / run_plmr, run_epp).  All label arrays are device pointers.
#pragma once

#include "sweep.cuh"

namespace cdk {

struct Report {
    cd_report *r;  // nullable
    void iteration(int64_t updated, double ms) {
        if (!r)
            return;
        if (r->n_iterations < CD_MAX_ITERATION_RECORDS)
            r->iterations[r->n_iterations] = {updated, ms};
        r->n_iterations++;
    }
    cd_level_record *level(int64_t l) {
        if (!r || l >= CD_MAX_LEVEL_RECORDS)
            return nullptr;
        if (r->n_levels < l + 1)
            r->n_levels = l + 1;
        return &r->levels[l];
    }
};

// wall-clock of device work on the context stream (CUDA events)
struct DevTimer {
    cd_ctx *ctx;
    cudaEvent_t a, b;
    explicit DevTimer(cd_ctx *c);
    ~DevTimer();
    void start();
    double stop_ms();  // syncs on the stop event
};

void plp_run_dev(cd_ctx *ctx, cd_graph *g, const cd_plp_config &cfg, const int32_t *initial, int32_t *labels,
                 Report rep);
int64_t plp_sweep_sync_dev(cd_ctx *ctx, cd_graph *g, const int32_t *z_in, int32_t *z_out);
void move_eval_dev(cd_ctx *ctx, cd_graph *g, const int32_t *z, const double *vols, double gamma, int32_t *best,
                   double *gain);
// buckets <= 0 / move_qtol < 0 resolved by the graph's degree skew (detect.cu)
constexpr int64_t SKEWED_MAX_DEGREE = 4096;
cd_louvain_config resolve_louvain_schedule(const cd_louvain_config &cfg, const cd_graph *g);
// from_singletons: z holds the node ids (the recursion's every level, H/louvain.hpp:242)
bool move_phase_dev(cd_ctx *ctx, cd_graph *g, int32_t *z, const cd_louvain_config &cfg, uint64_t salt,
                    int64_t *passes = nullptr, int64_t *moves = nullptr, bool from_singletons = false);
// the reference's one-worker move phase (sequential.cu): u = 0..n-1 in place,
// every applied move replayed to `observer` (may be null) after its pass
bool move_phase_sequential_dev(cd_ctx *ctx, cd_graph *g, int32_t *z, int64_t ub, double gamma, int64_t max_passes,
                               cd_move_observer observer, void *user);
int64_t louvain_run_dev(cd_ctx *ctx, cd_graph *g, const cd_louvain_config &cfg, int32_t *z, Report rep);
// given_bases: caller-supplied base partitions (ensemble_size device arrays of
// n labels) instead of running the base detector (EnsembleConfig::base_override)
int64_t epp_run_dev(cd_ctx *ctx, cd_graph *g, const cd_ensemble_config &cfg, int32_t *z, Report rep,
                    const int32_t *const *given_bases = nullptr);

bool is_compact_dev(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t nc);

inline uint64_t louvain_salt(int64_t level, int phase) {
    return (1ULL << 62) | (static_cast<uint64_t>(level) << 40) | (static_cast<uint64_t>(phase) << 32);
}

}  // namespace cdk
