// detect.cu -- device drivers: PLP (H/plp.hpp:67-149), move phase
// (H/louvain.hpp:65-141), PLM / PLMR recursion (H/louvain.hpp:237-301) and
// EPP (H/ensemble.hpp:111-199).
//
// Update order: every PLP iteration / PLM pass is
// split into `buckets` sub-sweeps by bucket_of(bucket_key(seed, salt), u);
// each sub-sweep evaluates its nodes against frozen labels and its moves are
// applied before the next sub-sweep.  This is the deterministic stand-in for
// the reference's racy in-place OpenMP updates (H/plp.hpp:127-130,
// H/louvain.hpp:120-126); a pure Jacobi sweep oscillates (SURVEY.md finding 2).
// oracle/commdet_oracle.c (cdo_*_bucketed) ports this order exactly.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>

#include "detect.cuh"

#include "comm.cuh"

namespace cdk {

// Runs its scope on this device alone (no exchange, whole node range).
struct LocalScope {
    cd_ctx *ctx;
    Comm *saved;
    explicit LocalScope(cd_ctx *c) : ctx(c), saved(c->comm) { c->comm = nullptr; }
    ~LocalScope() { ctx->comm = saved; }
};

// Below this many entries a replicated graph is not worth the per-sub-sweep
// exchange: every rank runs the phase alone and rank 0's labels are broadcast
// (fp64 atomics may order volume updates differently on different ranks).
static int64_t shard_min_entries() {
    const char *e = std::getenv("CD_SHARD_MIN_ENTRIES");
    return e ? std::atoll(e) : (int64_t(1) << 22);
}

static bool run_replicated(cd_ctx *ctx, const cd_graph *g) {
    return world_size(ctx) > 1 && !g->rows_local && g->D < shard_min_entries();
}

DevTimer::DevTimer(cd_ctx *c) : ctx(c) {
    CD_CUDA(cudaEventCreate(&a));
    CD_CUDA(cudaEventCreate(&b));
}
DevTimer::~DevTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
}
void DevTimer::start() { CD_CUDA(cudaEventRecord(a, ctx->stream)); }
double DevTimer::stop_ms() {
    CD_CUDA(cudaEventRecord(b, ctx->stream));
    CD_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    CD_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

__global__ void k_count_diff(int64_t n, const int32_t *a, const int32_t *b, unsigned long long *cnt) {
    unsigned long long c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += a[i] != b[i];
    c = warp_sum(c);
    if (lane_id() == 0 && c)
        atomicAdd(cnt, c);
}

// ---------------------------------------------------------------------------
// PLP
// ---------------------------------------------------------------------------
void plp_run_dev(cd_ctx *ctx, cd_graph *g, const cd_plp_config &cfg, const int32_t *initial, int32_t *labels,
                 Report rep) {
    const int64_t n = g->n;
    if (run_replicated(ctx, g)) {
        {
            LocalScope local(ctx);
            plp_run_dev(ctx, g, cfg, initial, labels, rep);
        }
        ctx->comm->broadcast(ctx, labels, n * sizeof(int32_t), 0);
        return;
    }
    const int64_t theta = cfg.theta >= 0 ? cfg.theta : std::max<int64_t>(1, n / 100000);  // H/plp.hpp:24-28
    const int K = cfg.buckets > 0 ? cfg.buckets : 4;
    if (initial)
        CD_CUDA(cudaMemcpyAsync(labels, initial, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    else
        iota_dev(ctx, labels, n);
    DBuf<uint8_t> active(ctx, std::max<int64_t>(n, 1));
    active.fill_bytes(1);
    SweepCall c;
    c.mode = MODE_PLP;
    c.z = labels;
    c.active = active.p;
    c.buckets = K;
    owned_range(ctx, g, c.own_lo, c.own_hi);
    if (g->rows_local && world_size(ctx) > 1) {
        graph_ensure_transpose(ctx, g);
        c.toff = g->toff.p;
        c.tcol = g->tcol.p;
    }
    if (fused_eligible(ctx, g, c)) {  // the whole run in one cooperative kernel
        if (n > theta && cfg.max_iterations > 0) {
            FusedResult fr;
            fused_phase(ctx, g, c, cfg.seed, 0, cfg.max_iterations, theta, 0.0, 0.0, fr);
            for (size_t i = 0; i < fr.trace.size(); ++i)
                rep.iteration(fr.trace[i], fr.ms[i]);
        }
        return;
    }
    // count tallies on one device: the margin-pruned active set (exact;
    // DESIGN.md "Margin-pruned active set"); CD_PLP_MARGIN=0 keeps the flags
    DBuf<int2> chg;
    static const bool margins = env_i64("CD_PLP_MARGIN", 1) != 0;
    if (margins && !g->weighted && n > 0) {
        chg.alloc(ctx, n);
        chg.fill_bytes(0x20);  // (CHG_ALL, 0x20202020): every node is evaluated once
        c.chg = chg.p;
        c.active = nullptr;
    }
    // from the node ids, on count tallies: the first sub-sweep needs no tally
    c.identity_first = !initial && !g->weighted &&
                       env_i64("CD_PLP_IDENTITY", 1) != 0;
    Sweeper sw(ctx, g, c);
    DevTimer it(ctx);
    int64_t updated = n, iter = 0;
    while (updated > theta && iter < cfg.max_iterations) {  // H/plp.hpp:98
        it.start();
        sw.pass(bucket_key(cfg.seed, static_cast<uint64_t>(iter)));
        updated = sw.take_moves();
        rep.iteration(updated, it.stop_ms());
        ++iter;
    }
}

int64_t plp_sweep_sync_dev(cd_ctx *ctx, cd_graph *g, const int32_t *z_in, int32_t *z_out) {
    const int64_t n = g->n;
    if (n == 0)
        return 0;
    CD_CUDA(cudaMemcpyAsync(z_out, z_in, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    SweepCall c;
    c.mode = MODE_PLP;
    c.z = const_cast<int32_t *>(z_in);
    c.buckets = 1;
    c.dense_best = z_out;
    {
        Sweeper sw(ctx, g, c);
        sw.pass(0);
    }
    DBuf<unsigned long long> cnt(ctx, 1);
    cnt.zero();
    CD_LAUNCH(ctx, "count_diff", k_count_diff, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n, z_in,
              static_cast<const int32_t *>(z_out), cnt.p);
    unsigned long long h = 0;
    CD_CUDA(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return static_cast<int64_t>(h);
}

// ---------------------------------------------------------------------------
// Louvain
// ---------------------------------------------------------------------------
__global__ void k_fill_gain0(int64_t n, const int32_t *z, int32_t *best, double *gain) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        best[i] = z[i];
        if (gain)
            gain[i] = 0.0;
    }
}

void move_eval_dev(cd_ctx *ctx, cd_graph *g, const int32_t *z, const double *vols, double gamma, int32_t *best,
                   double *gain) {
    const int64_t n = g->n;
    if (n == 0)
        return;
    CD_LAUNCH(ctx, "move_eval", k_fill_gain0, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n, z, best, gain);
    if (g->total == 0.0)
        return;
    SweepCall c;
    c.mode = MODE_PLM;
    c.z = const_cast<int32_t *>(z);
    c.vols = const_cast<double *>(vols);
    c.gamma = gamma;
    c.buckets = 1;
    c.dense_best = best;
    c.dense_gain = gain;
    {
        Sweeper sw(ctx, g, c);
        sw.pass(0);
    }
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
}

bool move_phase_dev(cd_ctx *ctx, cd_graph *g, int32_t *z, const cd_louvain_config &cfg, uint64_t salt,
                    int64_t *passes, int64_t *moves, bool from_singletons) {
    const int64_t n = g->n;
    if (n == 0 || g->total == 0.0)  // H/louvain.hpp:67-68
        return false;
    if (run_replicated(ctx, g)) {
        bool ch;
        {
            LocalScope local(ctx);
            ch = move_phase_dev(ctx, g, z, cfg, salt, passes, moves, from_singletons);
        }
        ctx->comm->broadcast(ctx, z, n * sizeof(int32_t), 0);
        int32_t chv = ch ? 1 : 0;
        DBuf<int32_t> d(ctx, 1);
        CD_CUDA(cudaMemcpyAsync(d.p, &chv, sizeof(chv), cudaMemcpyHostToDevice, ctx->stream));
        ctx->comm->broadcast(ctx, d.p, sizeof(int32_t), 0);
        CD_CUDA(cudaMemcpyAsync(&chv, d.p, sizeof(chv), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        return chv != 0;
    }
    const int K = cfg.buckets > 0 ? cfg.buckets : 4;
    const int64_t theta = std::max<int64_t>(cfg.move_theta >= 0 ? cfg.move_theta : n / 100000,
                                            static_cast<int64_t>(cfg.move_tol * static_cast<double>(n)));
    DBuf<double> vols(ctx, n);
    DBuf<int32_t> csize(ctx, n);
    community_volumes_sizes_dev(ctx, g, z, vols.p, csize.p, n);  // H/louvain.hpp:75
    SweepCall c;
    c.mode = MODE_PLM;
    c.z = z;
    c.vols = vols.p;
    c.csize = csize.p;
    c.gamma = cfg.gamma;
    c.guard = cfg.singleton_guard;
    c.buckets = K;
    owned_range(ctx, g, c.own_lo, c.own_hi);
    DBuf<uint8_t> active;
    if (cfg.prune) {
        active.alloc(ctx, n);
        active.fill_bytes(1);
        c.active = active.p;
        if (g->rows_local && world_size(ctx) > 1) {
            graph_ensure_transpose(ctx, g);
            c.toff = g->toff.p;
            c.tcol = g->tcol.p;
        }
    }
    if (small_move_eligible(ctx, g, c))
        return small_move_phase(ctx, g, c, cfg.seed, salt, cfg.max_move_iterations, theta, cfg.move_stall,
                                cfg.move_qtol, passes, moves);
    if (fused_eligible(ctx, g, c)) {
        if (cfg.max_move_iterations <= 0)
            return false;
        FusedResult fr;
        fused_phase(ctx, g, c, cfg.seed, salt, cfg.max_move_iterations, theta, cfg.move_stall, cfg.move_qtol, fr);
        if (passes)
            *passes += fr.passes;
        if (moves)
            *moves += fr.moves;
        return fr.changed;
    }
    // from singletons every neighbour is its own community: the first
    // sub-sweep needs no tally (k_plm_identity)
    c.identity_first = from_singletons && env_i64("CD_PLM_IDENTITY", 1) != 0;
    Sweeper sw(ctx, g, c);
    bool changed = false;
    static const bool trace = std::getenv("CD_TRACE") != nullptr;
    int64_t hist[2] = {-1, -1};  // moves of the two previous passes
    long long cum_fx = 0;        // the phase's summed gain (fixed point 2^-44)
    for (int64_t pass = 0; pass < cfg.max_move_iterations; ++pass) {
        const auto t0 = std::chrono::steady_clock::now();
        sw.pass(bucket_key(cfg.seed, salt + static_cast<uint64_t>(pass)));
        const int64_t moved = sw.take_moves();
        if (trace)
            std::fprintf(stderr, "[cd] move n=%lld D=%lld pass=%lld moved=%lld gain=%.4e %.3f ms\n",
                         static_cast<long long>(n), static_cast<long long>(g->D), static_cast<long long>(pass),
                         static_cast<long long>(moved), sw.last_gain(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        if (passes)
            ++*passes;
        if (moves)
            *moves += moved;
        if (moved == 0)  // H/louvain.hpp:136-137
            break;
        changed = true;
        if (moved <= theta)
            break;
        // stalled: a non-converging tail of oscillating movers
        if (cfg.move_stall > 0.0 && pass >= 8 &&
            static_cast<double>(moved) > cfg.move_stall * static_cast<double>(hist[0]))
            break;
        // converged in value: the pass added a negligible share of the phase's gain
        cum_fx += sw.last_gain_fx();
        if (cfg.move_qtol > 0.0 &&
            static_cast<double>(sw.last_gain_fx()) <= cfg.move_qtol * static_cast<double>(cum_fx))
            break;
        hist[0] = hist[1];
        hist[1] = moved;
    }
    return changed;
}

// H/louvain.hpp:237-267
static void louvain_recurse(cd_ctx *ctx, cd_graph *g, const cd_louvain_config &cfg_in, int64_t level, int32_t *z,
                            Report rep) {
    const int64_t n = g->n;
    // pruning: 1 = the input graph's move phases (where most nodes settle
    // early), 2 = every level
    cd_louvain_config cfg = cfg_in;
    if (level > 0 && cfg.prune < 2)
        cfg.prune = 0;
    iota_dev(ctx, z, n);  // singleton_partition (:242)
    DevTimer t(ctx);
    t.start();
    int64_t passes = 0, moves = 0;
    const bool changed = move_phase_dev(ctx, g, z, cfg, louvain_salt(level, 0), &passes, &moves, true);
    const double mv = t.stop_ms();
    if (g->D >= BIG_GRAPH_ENTRIES)
        graph_release_bins(g);  // room for the contraction and the coarse levels
    if (auto *L = rep.level(level)) {
        L->move_ms += mv;
        L->nodes = n;
        L->entries = g->D;
        L->passes += passes;
        L->moves += moves;
    }
    if (changed && level + 1 < cfg.max_levels) {  // :247
        DBuf<int32_t> zc(ctx, std::max<int64_t>(n, 1));
        const int64_t k = compact_dev(ctx, n, z, n, zc.p);  // :248
        if (k < n) {                                        // :249
            t.start();
            cd_graph *coarse = coarsen_sharded_dev(ctx, g, zc.p, k, false);  // :251 (rows unsorted)
            const double cm = t.stop_ms();
            if (auto *L = rep.level(level))
                L->coarsen_ms += cm;
            try {
                DBuf<int32_t> zcoarse(ctx, std::max<int64_t>(k, 1));
                louvain_recurse(ctx, coarse, cfg_in, level + 1, zcoarse.p, rep);  // :255
                prolong_dev(ctx, k, zcoarse.p, n, zc.p, z);                     // :256
            } catch (...) {
                delete coarse;
                throw;
            }
            delete coarse;
            if (cfg.refine) {  // PLMR :258-263
                t.start();
                int64_t rp = 0, rmv = 0;
                move_phase_dev(ctx, g, z, cfg, louvain_salt(level, 1), &rp, &rmv);
                const double rm = t.stop_ms();
                if (auto *L = rep.level(level)) {
                    L->refine_ms += rm;
                    L->passes += rp;
                    L->moves += rmv;
                }
            }
        }
    }
}

// The default schedule (DESIGN.md §4 "Schedule by graph"): buckets <= 0 and
// move_qtol < 0 mean "by graph".  A skewed graph (max degree > 4096: R-MAT-like
// hubs) takes 8 buckets and a gain tolerance of 5e-3 -- on C3 PLM modularity
// 0.0587 -> 0.0606 (the reference's 0.0611) and 227 -> 204 ms --, anything
// else 4 and 2e-3 (8 buckets cost C2 12 % at equal modularity).  Resolved
// once on the graph a run starts from; all its levels use it.  Ported
// exactly in oracle/commdet_oracle.c resolve_schedule.
cd_louvain_config resolve_louvain_schedule(const cd_louvain_config &cfg, const cd_graph *g) {
    cd_louvain_config c = cfg;
    const bool skewed = g->max_degree > SKEWED_MAX_DEGREE;
    if (c.buckets <= 0)
        c.buckets = skewed ? 8 : 4;
    if (c.move_qtol < 0.0)
        c.move_qtol = skewed ? 5e-3 : 2e-3;
    return c;
}

int64_t louvain_run_dev(cd_ctx *ctx, cd_graph *g, const cd_louvain_config &cfg_in, int32_t *z, Report rep) {
    if (g->total == 0.0)
        fail(CD_EDOMAIN, "Louvain requires positive total edge weight");  // H/louvain.hpp:271-272
    const cd_louvain_config cfg = resolve_louvain_schedule(cfg_in, g);
    DBuf<int32_t> tmp(ctx, std::max<int64_t>(g->n, 1));
    louvain_recurse(ctx, g, cfg, 0, tmp.p, rep);
    return compact_dev(ctx, g->n, tmp.p, std::max<int64_t>(g->n, 1), z);  // :278
}

// ---------------------------------------------------------------------------
// EPP
// ---------------------------------------------------------------------------
int64_t epp_run_dev(cd_ctx *ctx, cd_graph *g, const cd_ensemble_config &cfg, int32_t *z, Report rep,
                    const int32_t *const *given_bases) {
    if (cfg.ensemble_size < 1)
        fail(CD_EINVAL, "ensemble size must be >= 1");  // H/ensemble.hpp:113-114
    if (g->total == 0.0)
        fail(CD_EDOMAIN, "EPP requires positive total edge weight");  // :115-116
    const int64_t n = g->n, b = cfg.ensemble_size;
    DevTimer t(ctx);
    // bases (:152-161): seed + i
    t.start();
    const int G = world_size(ctx), rank = world_rank(ctx);
    // ensemble parallelism: with a replicated graph, rank r computes bases
    // r, r+G, ... alone and the bases are allgathered; a row shard computes
    // every base cooperatively
    const bool base_parallel = G > 1 && !g->rows_local && !given_bases;
    const int64_t slots = base_parallel ? (b + G - 1) / G * G : b;
    DBuf<int32_t> bases(ctx, given_bases ? 1 : std::max<int64_t>(n * slots, 1));
    auto run_base_on = [&](cd_ctx *c, int64_t i, int32_t *zi) {
        if (cfg.base == CD_ALGO_PLP) {
            cd_plp_config pc = cfg.base_plp;
            pc.seed = cfg.seed + static_cast<uint64_t>(i);
            plp_run_dev(c, g, pc, nullptr, zi, Report{nullptr});
        } else {
            cd_louvain_config lc = cfg.final_louvain;
            lc.seed = cfg.seed + static_cast<uint64_t>(i);
            lc.refine = cfg.base == CD_ALGO_PLMR;
            louvain_run_dev(c, g, lc, zi, Report{nullptr});
        }
    };
    auto run_base = [&](int64_t i, int32_t *zi) { run_base_on(ctx, i, zi); };
    // One device: the bases are independent runs of latency-bound kernels, so
    // they run concurrently -- one host thread and child context (own stream,
    // counters, hub scratch) each; the graph's shared work decomposition is
    // built first and only read.  PLP bases on graphs the tiered kernels run
    // (the one-kernel cooperative phases -- fused PLP for max degree <= 256,
    // the small PLM levels -- each want the whole GPU); not under profiling
    // (per-launch timing wants the kernels serialised) nor for graphs that
    // drop their bins between phases (BIG_GRAPH_ENTRIES).
    const bool concurrent = !given_bases && G == 1 && b > 1 && cfg.base == CD_ALGO_PLP && g->max_degree > 256 &&
                            !ctx->profiling && g->D < BIG_GRAPH_ENTRIES && env_i64("CD_EPP_CONCURRENT", 1) != 0;
    if (given_bases) {
        // EnsembleConfig::base_override (H/ensemble.hpp:127-128): the caller's partitions
    } else if (base_parallel) {
        for (int64_t j = 0; j < slots; j += G) {
            const int64_t i = j + rank;
            int32_t *zi = bases.p + i * n;
            if (i < b) {
                LocalScope local(ctx);
                run_base(i, zi);
            } else if (n) {
                CD_CUDA(cudaMemsetAsync(zi, 0, n * sizeof(int32_t), ctx->stream));
            }
            ctx->comm->allgather(ctx, zi, bases.p + j * n, n * sizeof(int32_t));  // in place
        }
    } else if (concurrent) {
        graph_ensure_bins(ctx, g);
        ctx_sync(ctx);  // bases allocated, graph ready for every stream
        std::vector<cd_ctx *> kids(b, nullptr);
        std::vector<std::exception_ptr> errs(b);
        try {
            for (int64_t i = 0; i < b; ++i)
                kids[i] = ctx_child(ctx);
            std::vector<std::thread> th;
            for (int64_t i = 0; i < b; ++i)
                th.emplace_back([&, i] {
                    try {
                        CD_CUDA(cudaSetDevice(ctx->device));
                        run_base_on(kids[i], i, bases.p + i * n);
                        CD_CUDA(cudaStreamSynchronize(kids[i]->stream));
                    } catch (...) {
                        errs[i] = std::current_exception();
                    }
                });
            for (auto &x : th)
                x.join();
        } catch (...) {
            for (auto *k : kids)
                ctx_child_destroy(ctx, k);
            throw;
        }
        for (auto *k : kids)
            ctx_child_destroy(ctx, k);
        for (auto &e : errs)
            if (e)
                std::rethrow_exception(e);
    } else {
        for (int64_t i = 0; i < b; ++i)
            run_base(i, bases.p + i * n);
    }
    const double base_ms = t.stop_ms();
    // combine (:163-165)
    t.start();
    std::vector<const int32_t *> hp(b);
    for (int64_t i = 0; i < b; ++i)
        hp[i] = given_bases ? given_bases[i] : bases.p + i * n;
    DBuf<const int32_t *> dp(ctx, b);
    CD_CUDA(cudaMemcpyAsync(dp.p, hp.data(), b * sizeof(int32_t *), cudaMemcpyHostToDevice, ctx->stream));
    DBuf<int32_t> core(ctx, std::max<int64_t>(n, 1));
    const int64_t k = combine_hashed_dev(ctx, b, n, dp.p, core.p);
    const double combine_ms = t.stop_ms();
    // coarsen (:167-169)
    t.start();
    cd_graph *coarse = coarsen_sharded_dev(ctx, g, core.p, k, false);
    const double coarsen_ms = t.stop_ms();
    double final_ms = 0.0;
    try {
        // final solver (:171-191), seed = cfg.seed
        t.start();
        DBuf<int32_t> zc(ctx, std::max<int64_t>(k, 1));
        if (cfg.final_algo == CD_ALGO_PLP) {
            cd_plp_config pc = cfg.base_plp;
            pc.seed = cfg.seed;
            plp_run_dev(ctx, coarse, pc, nullptr, zc.p, Report{nullptr});
        } else {
            cd_louvain_config fc = cfg.final_louvain;
            fc.seed = cfg.seed;
            fc.refine = cfg.final_algo == CD_ALGO_PLMR;
            louvain_run_dev(ctx, coarse, fc, zc.p, Report{nullptr});
        }
        final_ms = t.stop_ms();
        // prolong + compact (:193)
        DBuf<int32_t> fine(ctx, std::max<int64_t>(n, 1));
        prolong_dev(ctx, k, zc.p, n, core.p, fine.p);
        const int64_t kk = compact_dev(ctx, n, fine.p, std::max<int64_t>(k, 1), z);
        delete coarse;
        if (rep.r) {
            rep.r->base_ms = base_ms;
            rep.r->combine_ms = combine_ms;
            rep.r->coarsen_ms = coarsen_ms;
            rep.r->final_ms = final_ms;
        }
        return kk;
    } catch (...) {
        delete coarse;
        throw;
    }
}

}  // namespace cdk
