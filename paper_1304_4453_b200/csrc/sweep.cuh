// sweep.cuh -- host interface of the degree-tiered label-propagation sweep
// (H/plp.hpp:106-133) and Louvain move evaluation (H/louvain.hpp:88-126).
#pragma once

#include "graph.cuh"

namespace cdk {

enum SweepMode : int { MODE_PLP = 0, MODE_PLM = 1 };

struct SweepState {
    cd_ctx *ctx = nullptr;
    cd_graph *g = nullptr;
    DBuf<int32_t> cnt;         // [8]: per-tier list counts [0..4], [5] moves
    DBuf<int32_t> mv_node;     // [n]
    DBuf<int32_t> mv_label;    // [n]
    DBuf<long long> total;     // [1] moves accumulated since last reset
};

void sweep_init(cd_ctx *ctx, cd_graph *g, SweepState &st);

// One bucket sub-sweep: every selected node (tier list, bucket, active) is
// evaluated against the frozen labels z; the decisions are then applied to z
// (PLP: and neighbours activated; PLM: vols / csize moved).  With dense_best
// set, decisions are written densely instead and nothing is applied.
struct SweepCall {
    int mode = MODE_PLP;
    int32_t *z = nullptr;
    uint8_t *active = nullptr;   // PLP active set (nullable: all active, no deactivation)
    double *vols = nullptr;      // PLM community volumes
    int32_t *csize = nullptr;    // PLM community sizes (singleton guard; nullable)
    double gamma = 1.0;
    int guard = 0;
    uint64_t key = 0;
    int bucket = 0, buckets = 1;
    int32_t *dense_best = nullptr;
    double *dense_gain = nullptr;
};
void sweep_bucket(SweepState &st, const SweepCall &c);

// host read of the accumulated move counter (syncs) and reset
int64_t sweep_read_total(SweepState &st);
void sweep_reset_total(SweepState &st);

}  // namespace cdk
