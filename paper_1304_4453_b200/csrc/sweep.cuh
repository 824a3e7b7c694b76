// sweep.cuh -- host interface of the degree-tiered label-propagation sweep
// (H/plp.hpp:106-133) and Louvain move evaluation (H/louvain.hpp:88-126).
#pragma once

#include "graph.cuh"

namespace cdk {

enum SweepMode : int { MODE_PLP = 0, MODE_PLM = 1 };

// Fixed for the lifetime of a Sweeper (one PLP run / one move phase).
struct SweepCall {
    int mode = MODE_PLP;
    int32_t *z = nullptr;
    uint8_t *active = nullptr;   // PLP active set (nullable: all active, no deactivation)
    // PLP on count tallies, in place of `active`: neighbour label changes since
    // the node's last evaluation and the margin of its decision then
    // (DESIGN.md "Margin-pruned active set"); both nullable
    int2 *chg = nullptr;  // (changes since the last evaluation, margin then)
    // PLP on count tallies from z = node ids over rows sorted ascending: the
    // first sub-sweep takes each node's smallest neighbour (identity_subsweep)
    bool identity_first = false;
    double *vols = nullptr;      // PLM community volumes
    int32_t *csize = nullptr;    // PLM community sizes (singleton guard; nullable)
    double gamma = 1.0;
    int guard = 0;
    int buckets = 1;
    int32_t *dense_best = nullptr;  // evaluation only: write decisions densely, apply nothing
    double *dense_gain = nullptr;
    // sharded execution: this rank evaluates [own_lo, own_hi) (-1: all nodes);
    // PLP activation walks (toff, tcol) when set (a row shard's transpose)
    int64_t own_lo = 0, own_hi = -1;
    const int64_t *toff = nullptr;
    const int32_t *tcol = nullptr;
};

// One iteration / pass = `buckets` sub-sweeps.  Each sub-sweep evaluates the
// selected nodes of every degree tier against the frozen labels (the tier
// kernels run as parallel branches) and then applies its moves.  After the
// first pass the launch sequence is replayed from a CUDA graph; the bucket key
// lives in device memory so the graph is reusable.
//
// With a communicator of size G > 1 (comm.cuh) every rank evaluates only the
// nodes it owns; after each sub-sweep the ranks allgather their move lists
// and every rank applies all of them in rank order, so labels, volumes and
// the move count stay replicated and identical to the one-device run.
class Sweeper {
  public:
    Sweeper(cd_ctx *ctx, cd_graph *g, const SweepCall &c);
    ~Sweeper();
    Sweeper(const Sweeper &) = delete;
    Sweeper &operator=(const Sweeper &) = delete;

    void pass(uint64_t key);   // enqueue one full pass with this bucket key
    int64_t take_moves();      // moves since the last call (syncs)
    double last_gain() const { return last_gain_; }        // their summed Δ
    long long last_gain_fx() const { return last_gain_fx_; }  // the same in units of 2^-44 (exact)

  private:
    void enqueue(bool capture, bool recording = false);
    void apply(const int2 *mv, const int32_t *counts, int nseg, int64_t stride);
    void exchange_and_apply(int b);
    cd_ctx *ctx_;
    cd_graph *g_;
    SweepCall c_;
    int world_ = 1;
    bool exchange_ = false;
    int64_t tbeg_[NUM_TIERS] = {}, tend_[NUM_TIERS] = {};
    // short tier lists are partitioned by bucket once per pass (balanced
    // sub-sweeps on coarse levels); see k_prebucket
    uint32_t pre_mask_ = 0;
    int pre_tiers_[NUM_TIERS] = {}, n_pre_ = 0;
    DBuf<int32_t> blist_, boff_, pb_cnt_, pb_cur_;
    DBuf<int32_t> cnt_;     // [8]: [b] moves of bucket b
    DBuf<int2> mv_;         // this rank's moves of the current bucket
    DBuf<int32_t> rcnt_;    // [G] gathered counts
    DBuf<int2> rmv_;        // [G][stride] gathered moves
    DBuf<long long> total_;
    DBuf<long long> gain_;
    double last_gain_ = 0.0;
    long long last_gain_fx_ = 0;
    DBuf<unsigned long long> key_;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t exec_ = nullptr;
    int64_t kernels_per_pass_ = 0;
    bool identity_pending_ = false;  // the first eager pass's bucket 0 (SweepCall::identity_first)
};

// Whole PLP run / PLM move phase of a graph with degrees <= 256 in one
// cooperative kernel (same decisions, order and stop rules as the Sweeper).
struct FusedResult {
    int64_t passes = 0, moves = 0;
    bool changed = false;
    std::vector<long long> trace;  // moves per pass
    std::vector<double> ms;        // device time per pass
};
bool fused_eligible(const cd_ctx *ctx, const cd_graph *g, const SweepCall &c);
int64_t fused_phase(cd_ctx *ctx, cd_graph *g, const SweepCall &c, uint64_t seed, uint64_t salt, int64_t max_passes,
                    int64_t theta, double stall, double qtol, FusedResult &out);

// Whole PLM move phase of a small graph in one cooperative kernel (same
// decisions, order and stop rules as the Sweeper path); returns `changed`.
bool small_move_eligible(const cd_ctx *ctx, const cd_graph *g, const SweepCall &c);
bool small_move_phase(cd_ctx *ctx, cd_graph *g, const SweepCall &c, uint64_t seed, uint64_t salt, int64_t max_passes,
                      int64_t theta, double stall, double qtol, int64_t *passes, int64_t *moves);

}  // namespace cdk
