// capi.cu -- the extern "C" boundary (include/commdet_cuda.h).  Each entry
// point validates like the reference function it replaces, moves host
// arguments in / out and maps C++ errors to cd_status codes.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>

#include "comm.cuh"
#include "detect.cuh"

namespace cdk {
cd_graph *generate_planted_dev(cd_ctx *ctx, int64_t n, int64_t k, double p_in, double p_out, uint64_t seed,
                               int32_t *truth_dev);
cd_graph *generate_rmat_dev(cd_ctx *ctx, int scale, int edge_factor, double a, double b, double c, int weighted,
                            uint64_t seed, bool shard);
cd_graph *generate_lfr_dev(cd_ctx *ctx, const cd_lfr_spec &sp, uint64_t seed, int32_t *truth_dev);

namespace {
thread_local char g_err[1024] = "";

void set_err(const char *m) {
    std::snprintf(g_err, sizeof(g_err), "%s", m);
}
}  // namespace

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaEvent_t ctx_event(cd_ctx *ctx) {
    if (!ctx->free_events.empty()) {
        cudaEvent_t e = ctx->free_events.back();
        ctx->free_events.pop_back();
        return e;
    }
    cudaEvent_t e;
    CD_CUDA(cudaEventCreate(&e));
    return e;
}

void ctx_flush_stats(cd_ctx *ctx) {
    if (ctx->pending.empty())
        return;
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto &p : ctx->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            auto &s = ctx->stats[p.name];
            s.launches += 1;
            s.total_ms += ms;
        }
        ctx->free_events.push_back(p.a);
        ctx->free_events.push_back(p.b);
    }
    ctx->pending.clear();
}

void ctx_sync(cd_ctx *ctx) { CD_CUDA(cudaStreamSynchronize(ctx->stream)); }

}  // namespace cdk

using namespace cdk;

#define CD_GUARD(ctxp, ...)                                                                          \
    try {                                                                                            \
        if (ctxp)                                                                                    \
            CD_CUDA(cudaSetDevice((ctxp)->device));                                                  \
        __VA_ARGS__;                                                                                 \
        return CD_OK;                                                                                \
    } catch (const ::cdk::Error &e) {                                                                \
        set_err(e.what());                                                                           \
        return e.code;                                                                               \
    } catch (const std::bad_alloc &) {                                                               \
        set_err("host allocation failed");                                                           \
        return CD_ENOMEM;                                                                            \
    } catch (const std::exception &e) {                                                              \
        set_err(e.what());                                                                           \
        return CD_EINTERNAL;                                                                         \
    }

#define CD_REQUIRE(cond, code, msg)                                                                  \
    do {                                                                                             \
        if (!(cond))                                                                                 \
            ::cdk::fail(code, msg);                                                                  \
    } while (0)

namespace {

void report_begin(cd_report *r, const char *algo, int workers, uint64_t seed) {
    if (!r)
        return;
    std::memset(r, 0, sizeof(*r));
    std::snprintf(r->algorithm, sizeof(r->algorithm), "%s", algo);
    r->workers = workers;
    r->seed = seed;
}

// quality figures of a finished run (H/plp.hpp:143-147, H/louvain.hpp:280-282)
void report_quality(cd_ctx *ctx, cd_graph *g, const int32_t *z, int64_t ub, double gamma, cd_report *r) {
    if (!r)
        return;
    if (g->total > 0) {
        modularity_dev(ctx, g, z, ub, gamma, &r->modularity, &r->coverage);
    } else {
        r->modularity = 0.0;
        r->coverage = 0.0;
    }
}

}  // namespace

extern "C" {

const char *cd_last_error(void) { return g_err; }
const char *cd_version(void) { return "commdet-b200 0.1 (sm_100a)"; }

void cd_plp_config_default(cd_plp_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->theta = -1;
    c->max_iterations = 100;
    c->randomize_order = 0;
    c->workers = 1;
    c->seed = 1;
    c->buckets = 4;
}

void cd_louvain_config_default(cd_louvain_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->gamma = 1.0;
    c->max_move_iterations = 32;
    c->max_levels = 64;
    c->seed = 1;
    c->workers = 1;
    c->refine = 0;
    c->buckets = 0;  // by graph: 8 if the max degree exceeds 4096, else 4 (resolve_louvain_schedule)
    c->singleton_guard = 1;
    c->move_theta = -1;
    c->move_tol = 1e-3;  // stop a level's passes below 0.1% movers
    c->move_stall = 0.95;  // ... or once the movers stop shrinking (oscillating tail)
    c->prune = 1;          // ... and skip nodes whose neighbourhood did not change
    c->move_qtol = -1.0;   // ... or once a pass adds < 0.5% (skewed) / 0.2% of the phase's gain (by graph)
}

void cd_louvain_config_reference(cd_louvain_config *c) {
    cd_louvain_config_default(c);
    c->move_theta = 0;
    c->move_tol = 0.0;
    c->move_stall = 0.0;
    c->prune = 0;
    c->move_qtol = 0.0;
}

void cd_ensemble_config_default(cd_ensemble_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->ensemble_size = 4;
    c->base = CD_ALGO_PLP;
    c->final_algo = CD_ALGO_PLMR;
    c->seed = 1;
    c->workers = 1;
    cd_plp_config_default(&c->base_plp);
    c->base_plp.randomize_order = 1;  // H/ensemble.hpp:27
    cd_louvain_config_default(&c->final_louvain);
}

cd_status cd_ctx_create(int device, cd_ctx **out) {
    cd_ctx *ctx = nullptr;
    try {
        CD_REQUIRE(out, CD_EINVAL, "null output");
        int ndev = 0;
        CD_CUDA(cudaGetDeviceCount(&ndev));
        CD_REQUIRE(device >= 0 && device < ndev, CD_EINVAL, "no such CUDA device");
        CD_CUDA(cudaSetDevice(device));
        ctx = new cd_ctx();
        ctx->device = device;
        CD_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        CD_CUDA(cudaDeviceGetDefaultMemPool(&ctx->pool, device));
        uint64_t thr = UINT64_MAX;
        CD_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr));
        // Reserve device memory in the stream-ordered pool once: growing the
        // pool inside a run maps pages (tens to hundreds of ms for large
        // temporaries).  CD_POOL_RESERVE_FRAC (default 0.5) of free memory.
        {
            double frac = 0.5;
            if (const char *e = std::getenv("CD_POOL_RESERVE_FRAC"))
                frac = std::atof(e);
            size_t free_b = 0, total_b = 0;
            CD_CUDA(cudaMemGetInfo(&free_b, &total_b));
            const size_t want = static_cast<size_t>(frac * static_cast<double>(free_b)) & ~size_t(0xFFFFF);
            if (want > 0) {
                void *p = nullptr;
                if (cudaMallocAsync(&p, want, ctx->stream) == cudaSuccess) {
                    cudaFreeAsync(p, ctx->stream);
                    CD_CUDA(cudaStreamSynchronize(ctx->stream));
                } else {
                    cudaGetLastError();
                }
            }
        }
        cudaDeviceProp prop;
        CD_CUDA(cudaGetDeviceProperties(&prop, device));
        ctx->num_sms = prop.multiProcessorCount;
        ctx->smem_optin = prop.sharedMemPerBlockOptin;
        ctx->use_graphs = std::getenv("CD_NO_GRAPHS") == nullptr;
        CD_CUDA(cudaMalloc(reinterpret_cast<void **>(&ctx->dstats), DSTATS * sizeof(unsigned long long)));
        CD_CUDA(cudaMemset(ctx->dstats, 0, DSTATS * sizeof(unsigned long long)));
        *out = ctx;
        return CD_OK;
    } catch (const ::cdk::Error &e) {
        set_err(e.what());
        if (ctx) {
            if (ctx->stream)
                cudaStreamDestroy(ctx->stream);
            delete ctx;
        }
        return e.code;
    } catch (const std::exception &e) {
        set_err(e.what());
        delete ctx;
        return CD_EINTERNAL;
    }
}

cd_status cd_ctx_destroy(cd_ctx *ctx) {
    if (!ctx)
        return CD_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &p : ctx->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : ctx->free_events)
        cudaEventDestroy(e);
    if (ctx->dstats)
        cudaFree(ctx->dstats);
    if (ctx->copy_stream)
        cudaStreamDestroy(ctx->copy_stream);
    delete ctx->comm;
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return CD_OK;
}

cd_status cd_ctx_synchronize(cd_ctx *ctx) { CD_GUARD(ctx, CD_REQUIRE(ctx, CD_EINVAL, "null context"); ctx_sync(ctx)) }

cd_status cd_ctx_stream(cd_ctx *ctx, void **stream) {
    CD_GUARD(ctx, CD_REQUIRE(ctx && stream, CD_EINVAL, "null argument"); *stream = ctx->stream)
}

cd_status cd_ctx_set_profiling(cd_ctx *ctx, int enabled) {
    CD_GUARD(ctx, CD_REQUIRE(ctx, CD_EINVAL, "null context"); ctx_flush_stats(ctx); ctx->profiling = enabled < 0 ? 0 : (enabled > 2 ? 1 : enabled))
}

cd_status cd_ctx_reset_stats(cd_ctx *ctx) {
    CD_GUARD(ctx, CD_REQUIRE(ctx, CD_EINVAL, "null context"); ctx_flush_stats(ctx); ctx->stats.clear();
             CD_CUDA(cudaMemsetAsync(ctx->dstats, 0, DSTATS * sizeof(unsigned long long), ctx->stream));
             ctx_sync(ctx))
}

cd_status cd_ctx_kernel_stats(cd_ctx *ctx, cd_kernel_stat *out, int32_t capacity, int32_t *count) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && count, CD_EINVAL, "null argument");
        ctx_flush_stats(ctx);
        // algorithmic bytes of the sweep families (DESIGN.md byte model):
        //   plp_sweep: 17 B / evaluated node + (8 + 4W) B / entry
        //   plm_move:  24 B / evaluated node + (8 + 4W) B / entry
        unsigned long long ds[DSTATS];
        CD_CUDA(cudaMemcpyAsync(ds, ctx->dstats, sizeof(ds), cudaMemcpyDeviceToHost, ctx->stream));
        ctx_sync(ctx);
        // aggregate sub-families ("plm_move.warp", "coarsen.sort", ...) into
        // their base ("plm_move", "coarsen"); a base never has its own launches
        {
            std::map<std::string, KStat> agg;
            for (auto &kv : ctx->stats) {
                const size_t dot = kv.first.find('.');
                if (dot == std::string::npos)
                    continue;
                auto &t = agg[kv.first.substr(0, dot)];
                t.launches += kv.second.launches;
                t.total_ms += kv.second.total_ms;
            }
            for (auto &kv : agg)
                ctx->stats[kv.first] = kv.second;
            auto model = ctx->stats.find("coarsen.model");  // contraction byte model (coarsen_dev)
            if (model != ctx->stats.end() && ctx->stats.count("coarsen")) {
                ctx->stats["coarsen"].bytes = model->second.bytes;
                ctx->stats["coarsen"].items = model->second.items;
            }
        }
        // per-kernel algorithmic bytes (DESIGN.md byte model), from the
        // per-tier work counters: plp 17 B / node, plm 24 B / node, plus
        // 8 (unweighted) or 12 (weighted) B / entry
        static const char *slot_name[STAT_SLOTS] = {"g8",     "g16",     "g32",     "warp",  "block", "block2",
                                                    "block3", "cluster", "hub",     "small", "fused"};
        for (int m = 0; m < 2; ++m) {
            const std::string base = m == 0 ? "plp_sweep" : "plm_move";
            const double per_node = m == 0 ? 17.0 : 24.0;
            // the hub tier runs as several kernels: time it as one family
            KStat hub;
            for (auto &kv : ctx->stats)
                if (kv.first.compare(0, base.size() + 5, base + ".hub_") == 0) {
                    hub.launches = std::max(hub.launches, kv.second.launches);
                    hub.total_ms += kv.second.total_ms;
                }
            if (hub.total_ms > 0)
                ctx->stats[base + ".hub"] = hub;
            double tb = 0.0, ti = 0.0;
            for (int sl = 0; sl < STAT_SLOTS; ++sl) {
                const unsigned long long *c = ds + m * STAT_MODE_STRIDE + 3 * sl;
                const double bytes = per_node * c[0] + 8.0 * c[1] + 12.0 * c[2];
                const double items = static_cast<double>(c[1] + c[2]);
                tb += bytes;
                ti += items;
                auto it = ctx->stats.find(base + "." + slot_name[sl]);
                if (it != ctx->stats.end()) {
                    it->second.bytes = bytes;
                    it->second.items = items;
                }
            }
            auto it = ctx->stats.find(base);
            if (it != ctx->stats.end()) {
                it->second.bytes = tb;
                it->second.items = ti;
            }
        }
        int32_t i = 0;
        for (auto &kv : ctx->stats) {
            if (out && i < capacity) {
                std::snprintf(out[i].name, sizeof(out[i].name), "%s", kv.first.c_str());
                out[i].launches = kv.second.launches;
                out[i].total_ms = kv.second.total_ms;
                out[i].bytes = kv.second.bytes;
                out[i].items = kv.second.items;
            }
            ++i;
        }
        *count = i;
    })
}

cd_status cd_ctx_launch_count(cd_ctx *ctx, int64_t *count) {
    CD_GUARD(ctx, CD_REQUIRE(ctx && count, CD_EINVAL, "null argument"); *count = ctx->launches)
}

// ---- graphs ------------------------------------------------------------------

__global__ void k_check_edges(int64_t m, int64_t n, const int32_t *u, const int32_t *v, const float *w, int *flag) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (u[i] < 0 || v[i] < 0 || u[i] >= n || v[i] >= n)
            *flag = 1;
        if (w && !(w[i] > 0.0f))
            *flag = 2;
    }
}

cd_status cd_graph_from_edges(cd_ctx *ctx, int64_t n, int64_t m, const int32_t *u, const int32_t *v, const float *w,
                              int32_t merge_duplicates, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && n >= 0 && m >= 0 && n < INT32_MAX, CD_EINVAL, "invalid argument");
        CD_REQUIRE(m == 0 || (u && v), CD_EINVAL, "null edge arrays");
        InArr<int32_t> du(ctx, u, m), dv(ctx, v, m);
        InArr<float> dw(ctx, w, m);
        if (m > 0) {
            DBuf<int> flag(ctx, 1);
            flag.zero();
            CD_LAUNCH(ctx, "validate", k_check_edges, grid_for(m, 256, ctx->num_sms * 8), 256, 0, m, n, du.d, dv.d,
                      dw.d, flag.p);
            int h = 0;
            CD_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            CD_CUDA(cudaStreamSynchronize(ctx->stream));
            if (h == 1)
                fail(CD_EINPUT, "edge endpoint out of range");  // H/graph.hpp:50-51
            if (h == 2)
                fail(CD_EINPUT, "nonpositive edge weight");  // H/graph.hpp:52-53
        }
        *out = graph_from_pairs(ctx, n, m, du.d, dv.d, dw.d, merge_duplicates ? DUP_SUM : DUP_ERROR);
    })
}

cd_status cd_graph_from_csr(cd_ctx *ctx, int64_t n, const int64_t *off, const int32_t *col, const float *w,
                            cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && off && n >= 0 && n < INT32_MAX, CD_EINVAL, "invalid argument");
        int64_t D = 0;
        if (is_device_ptr(off)) {
            CD_CUDA(cudaMemcpy(&D, off + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
        } else {
            D = off[n];
        }
        CD_REQUIRE(D >= 0, CD_EINPUT, "negative entry count");
        CD_REQUIRE(D == 0 || col, CD_EINVAL, "null column array");
        auto *g = new cd_graph();
        try {
            g->ctx = ctx;
            g->n = n;
            g->D = D;
            g->weighted = w != nullptr;
            g->off.alloc(ctx, n + 1);
            g->col.alloc(ctx, std::max<int64_t>(D, 1));
            if (w)
                g->w.alloc(ctx, std::max<int64_t>(D, 1));
            CD_CUDA(cudaMemcpyAsync(g->off.p, off, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, ctx->stream));
            if (D && !is_device_ptr(col) && D >= UPLOAD_MIN_ENTRIES) {
                // host columns: chunked copies, each chunk validated while the next one copies;
                // an unweighted graph is finalized and binned during the copy as well
                graph_upload_validate(ctx, n, D, g->off.p, g->col.p, col, w ? g->w.p : nullptr, w, w ? nullptr : g);
                if (!w) {
                    *out = g;
                    return CD_OK;
                }
            } else {
                if (D)
                    CD_CUDA(cudaMemcpyAsync(g->col.p, col, D * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
                if (w && D)
                    CD_CUDA(cudaMemcpyAsync(g->w.p, w, D * sizeof(float), cudaMemcpyDefault, ctx->stream));
                graph_validate_csr(ctx, n, g->off.p, g->col.p, g->weighted ? g->w.p : nullptr, D);
            }
            graph_finalize(ctx, g);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    })
}

cd_status cd_graph_generate_planted(cd_ctx *ctx, int64_t n, int64_t k, double p_in, double p_out, uint64_t seed,
                                    cd_graph **out, int32_t *truth) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && n >= 0 && n < INT32_MAX, CD_EINVAL, "invalid argument");
        OutArr<int32_t> t(ctx, truth, n);
        *out = generate_planted_dev(ctx, n, k, p_in, p_out, seed, t.d);
        t.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_graph_generate_rmat(cd_ctx *ctx, int32_t scale, int32_t edge_factor, double a, double b, double c,
                                 int32_t weighted, uint64_t seed, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out, CD_EINVAL, "invalid argument");
        *out = generate_rmat_dev(ctx, scale, edge_factor, a, b, c, weighted, seed, false);
    })
}

cd_status cd_graph_generate_rmat_shard(cd_ctx *ctx, int32_t scale, int32_t edge_factor, double a, double b, double c,
                                       int32_t weighted, uint64_t seed, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out, CD_EINVAL, "invalid argument");
        *out = generate_rmat_dev(ctx, scale, edge_factor, a, b, c, weighted, seed, true);
    })
}

cd_status cd_graph_generate_lfr(cd_ctx *ctx, const cd_lfr_spec *spec, uint64_t seed, cd_graph **out,
                                int32_t *truth) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && spec && spec->n < INT32_MAX, CD_EINVAL, "invalid argument");
        OutArr<int32_t> t(ctx, truth, spec->n);
        *out = generate_lfr_dev(ctx, *spec, seed, t.d);
        t.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_graph_get_info(const cd_graph *g, cd_graph_info *out) {
    CD_GUARD(static_cast<cd_ctx *>(nullptr), {
        CD_REQUIRE(g && out, CD_EINVAL, "null argument");
        out->n = g->n;
        out->D = g->D;
        out->m = g->m;
        out->total_weight = g->total;
        out->weighted = g->weighted ? 1 : 0;
        out->reserved = 0;
        out->max_degree = g->max_degree;
        out->isolated = g->isolated;
        out->shard_rank = g->rows_local ? g->shard_rank : 0;
        out->shard_size = g->rows_local ? g->shard_size : 1;
        out->own_lo = g->rows_local ? g->own_lo : 0;
        out->own_hi = g->rows_local ? g->own_hi : g->n;
        out->D_global = g->rows_local ? g->D_global : g->D;
    })
}

cd_status cd_graph_download(const cd_graph *g, int64_t *off, int32_t *col, float *w, double *vol, double *loop) {
    cd_ctx *ctx = g ? g->ctx : nullptr;
    CD_GUARD(ctx, {
        CD_REQUIRE(g, CD_EINVAL, "null graph");
        if (off)
            CD_CUDA(cudaMemcpyAsync(off, g->off.p, (g->n + 1) * sizeof(int64_t), cudaMemcpyDefault, ctx->stream));
        if (col && g->D)
            CD_CUDA(cudaMemcpyAsync(col, g->col.p, g->D * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
        if (w && g->weighted && g->D)
            CD_CUDA(cudaMemcpyAsync(w, g->w.p, g->D * sizeof(float), cudaMemcpyDefault, ctx->stream));
        if (vol && g->n)
            CD_CUDA(cudaMemcpyAsync(vol, g->vol.p, g->n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        if (loop && g->n)
            CD_CUDA(cudaMemcpyAsync(loop, g->loop.p, g->n * sizeof(double), cudaMemcpyDefault, ctx->stream));
        ctx_sync(ctx);
    })
}

cd_status cd_graph_destroy(cd_graph *g) {
    if (!g)
        return CD_OK;
    cd_ctx *ctx = g->ctx;
    cudaSetDevice(ctx->device);
    delete g;
    cudaStreamSynchronize(ctx->stream);
    return CD_OK;
}

// ---- quality --------------------------------------------------------------------

cd_status cd_modularity(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double gamma, double *q,
                        double *coverage) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && z && ub >= 1, CD_EINVAL, "invalid argument");
        InArr<int32_t> dz(ctx, z, g->n);
        modularity_dev(ctx, const_cast<cd_graph *>(g), dz.d, ub, gamma, q, coverage);
    })
}

cd_status cd_rand_index(cd_ctx *ctx, const cd_graph *g, const int32_t *a, const int32_t *b, double *out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && out && (g->n == 0 || (a && b)), CD_EINVAL, "invalid argument");
        InArr<int32_t> da(ctx, a, g->n), db(ctx, b, g->n);
        *out = rand_index_dev(ctx, g, da.d, db.d);
    })
}

cd_status cd_community_volumes(cd_ctx *ctx, const cd_graph *g, const int32_t *z, int64_t ub, double *vols) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && z && vols && ub >= 1, CD_EINVAL, "invalid argument");
        InArr<int32_t> dz(ctx, z, g->n);
        OutArr<double> dv(ctx, vols, ub);
        community_volumes_dev(ctx, g, dz.d, dv.d, ub);
        dv.finish();
        ctx_sync(ctx);
    })
}

// ---- partitions -----------------------------------------------------------------

cd_status cd_compact(cd_ctx *ctx, int64_t n, const int32_t *z, int32_t *out, int64_t *k) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && (n == 0 || (z && out)) && n >= 0, CD_EINVAL, "invalid argument");
        InArr<int32_t> dz(ctx, z, n);
        OutArr<int32_t> dout(ctx, out, n);
        const int64_t ub = max_label_dev(ctx, n, dz.d);
        CD_REQUIRE(ub >= 0, CD_EINVAL, "negative community id");
        const int64_t kk = compact_dev(ctx, n, dz.d, ub, dout.d);
        dout.finish();
        ctx_sync(ctx);
        if (k)
            *k = kk;
    })
}

cd_status cd_community_count(cd_ctx *ctx, int64_t n, const int32_t *z, int64_t *k) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && (n == 0 || z) && n >= 0 && k, CD_EINVAL, "invalid argument");
        InArr<int32_t> dz(ctx, z, n);
        DBuf<int32_t> tmp(ctx, std::max<int64_t>(n, 1));
        const int64_t ub = max_label_dev(ctx, n, dz.d);
        CD_REQUIRE(ub >= 0, CD_EINVAL, "negative community id");
        *k = compact_dev(ctx, n, dz.d, ub, tmp.p);
    })
}

cd_status cd_coarsen(cd_ctx *ctx, const cd_graph *g, const int32_t *z, cd_graph **coarse, int32_t *pi_out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && coarse && (g->n == 0 || z), CD_EINVAL, "invalid argument");
        InArr<int32_t> dz(ctx, z, g->n);
        const int64_t nc = g->n ? max_label_dev(ctx, g->n, dz.d) : 0;
        CD_REQUIRE(nc >= 0, CD_EINVAL, "coarsen requires a compacted partition");
        CD_REQUIRE(g->n == 0 || is_compact_dev(ctx, g->n, dz.d, nc), CD_EINVAL,
                   "coarsen requires a compacted partition");  // H/louvain.hpp:156-157
        *coarse = coarsen_sharded_dev(ctx, g, dz.d, nc);  // a row shard's coarse graph is the ranks' sum
        if (pi_out && g->n)
            CD_CUDA(cudaMemcpyAsync(pi_out, dz.d, g->n * sizeof(int32_t), cudaMemcpyDefault, ctx->stream));
        ctx_sync(ctx);
    })
}

cd_status cd_prolong(cd_ctx *ctx, int64_t nc, const int32_t *z_coarse, int64_t n, const int32_t *pi,
                     int32_t *out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && n >= 0 && nc >= 0 && (n == 0 || (pi && out)), CD_EINVAL, "invalid argument");
        InArr<int32_t> dzc(ctx, z_coarse, nc), dpi(ctx, pi, n);
        OutArr<int32_t> dout(ctx, out, n);
        prolong_dev(ctx, nc, dzc.d, n, dpi.d, dout.d);
        dout.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_combine_hashed(cd_ctx *ctx, int64_t b, int64_t n, const int32_t *const *solutions, int32_t *out,
                            int64_t *k) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && b >= 1 && solutions, CD_EINVAL, "empty ensemble");  // H/ensemble.hpp:33-35
        CD_REQUIRE(n >= 0 && (n == 0 || out), CD_EINVAL, "invalid argument");
        std::vector<InArr<int32_t> *> ins;
        std::vector<const int32_t *> ptrs;
        try {
            for (int64_t i = 0; i < b; ++i) {
                ins.push_back(new InArr<int32_t>(ctx, solutions[i], n));
                ptrs.push_back(ins.back()->d);
            }
            DBuf<const int32_t *> dp(ctx, b);
            CD_CUDA(cudaMemcpyAsync(dp.p, ptrs.data(), b * sizeof(int32_t *), cudaMemcpyHostToDevice, ctx->stream));
            OutArr<int32_t> dout(ctx, out, n);
            const int64_t kk = combine_hashed_dev(ctx, b, n, dp.p, dout.d);
            dout.finish();
            ctx_sync(ctx);
            if (k)
                *k = kk;
        } catch (...) {
            for (auto *p : ins)
                delete p;
            throw;
        }
        for (auto *p : ins)
            delete p;
    })
}

// ---- sub-kernels ------------------------------------------------------------------

cd_status cd_plp_sweep_sync(cd_ctx *ctx, const cd_graph *g, const int32_t *z_in, int32_t *z_out, int64_t *updated) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && (g->n == 0 || (z_in && z_out)), CD_EINVAL, "invalid argument");
        CD_REQUIRE(!g->rows_local || g->shard_size == 1, CD_EINVAL, "sub-kernel needs a whole graph, not a row shard");
        InArr<int32_t> dzi(ctx, z_in, g->n);
        OutArr<int32_t> dzo(ctx, z_out, g->n);
        const int64_t upd = plp_sweep_sync_dev(ctx, const_cast<cd_graph *>(g), dzi.d, dzo.d);
        dzo.finish();
        ctx_sync(ctx);
        if (updated)
            *updated = upd;
    })
}

cd_status cd_move_eval(cd_ctx *ctx, const cd_graph *g, const int32_t *z, const double *vols, int64_t ub, double gamma,
                       int32_t *best, double *gain) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && (g->n == 0 || (z && vols && best)) && ub >= 1, CD_EINVAL, "invalid argument");
        CD_REQUIRE(!g->rows_local || g->shard_size == 1, CD_EINVAL, "sub-kernel needs a whole graph, not a row shard");
        InArr<int32_t> dz(ctx, z, g->n);
        InArr<double> dv(ctx, vols, ub);
        const int64_t mx = max_label_dev(ctx, g->n, dz.d);
        CD_REQUIRE(mx >= 0 && mx <= ub, CD_ERANGE, "community id outside [0, ub)");
        OutArr<int32_t> db(ctx, best, g->n);
        OutArr<double> dg(ctx, gain, g->n);
        move_eval_dev(ctx, const_cast<cd_graph *>(g), dz.d, dv.d, gamma, db.d, dg.d);
        db.finish();
        dg.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_move_phase(cd_ctx *ctx, const cd_graph *g, int32_t *z, const cd_louvain_config *cfg, int32_t *changed) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || z), CD_EINVAL, "invalid argument");
        OutArr<int32_t> dz(ctx, z, g->n);
        if (dz.host && g->n)
            CD_CUDA(cudaMemcpyAsync(dz.d, z, g->n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        const int64_t mx = max_label_dev(ctx, g->n, dz.d);
        CD_REQUIRE(mx >= 0 && mx <= std::max<int64_t>(g->n, 1), CD_ERANGE, "device move phase needs labels < n");
        const bool ch = move_phase_dev(ctx, const_cast<cd_graph *>(g), dz.d, resolve_louvain_schedule(*cfg, g),
                                       louvain_salt(0, 0));
        dz.finish();
        ctx_sync(ctx);
        if (changed)
            *changed = ch ? 1 : 0;
    })
}

cd_status cd_move_phase_sequential(cd_ctx *ctx, const cd_graph *g, int32_t *z, int64_t ub, const cd_louvain_config *cfg,
                                   cd_move_observer observer, void *user, int32_t *changed) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || z) && ub >= 1, CD_EINVAL, "invalid argument");
        CD_REQUIRE(!g->rows_local || g->shard_size == 1, CD_EINVAL, "sub-kernel needs a whole graph, not a row shard");
        OutArr<int32_t> dz(ctx, z, g->n);
        if (dz.host && g->n)
            CD_CUDA(cudaMemcpyAsync(dz.d, z, g->n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        const int64_t mx = max_label_dev(ctx, g->n, dz.d);
        CD_REQUIRE(mx >= 0 && mx <= ub, CD_ERANGE, "community id outside [0, ub)");
        const bool ch = move_phase_sequential_dev(ctx, const_cast<cd_graph *>(g), dz.d, ub, cfg->gamma,
                                                  cfg->max_move_iterations, observer, user);
        dz.finish();
        ctx_sync(ctx);
        if (changed)
            *changed = ch ? 1 : 0;
    })
}

// ---- detectors -------------------------------------------------------------------

cd_status cd_plp_run(cd_ctx *ctx, const cd_graph *g, const cd_plp_config *cfg, const int32_t *initial,
                     int32_t *labels, cd_report *report) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || labels), CD_EINVAL, "invalid argument");
        cd_graph *gg = const_cast<cd_graph *>(g);
        const int64_t launches0 = ctx->launches;
        report_begin(report, "plp", cfg->workers, cfg->seed);
        InArr<int32_t> di(ctx, initial, g->n);
        int64_t ub = std::max<int64_t>(g->n, 1);
        if (initial) {
            ub = max_label_dev(ctx, g->n, di.d);
            CD_REQUIRE(ub >= 0, CD_EINVAL, "initial partition has negative ids");
            ub = std::max<int64_t>(ub, 1);
        }
        OutArr<int32_t> dl(ctx, labels, g->n);
        DevTimer t(ctx);
        t.start();
        plp_run_dev(ctx, gg, *cfg, initial ? di.d : nullptr, dl.d, Report{report});
        const double ms = t.stop_ms();
        if (report) {
            report->total_ms = ms;  // excludes quality evaluation (H/plp.hpp:142)
            report_quality(ctx, gg, dl.d, ub, 1.0, report);
            DBuf<int32_t> tmp(ctx, std::max<int64_t>(g->n, 1));
            report->community_count = compact_dev(ctx, g->n, dl.d, ub, tmp.p);
            report->kernel_launches = ctx->launches - launches0;
        }
        dl.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_louvain_run(cd_ctx *ctx, const cd_graph *g, const cd_louvain_config *cfg, int32_t *z,
                         cd_report *report) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || z), CD_EINVAL, "invalid argument");
        cd_graph *gg = const_cast<cd_graph *>(g);
        const int64_t launches0 = ctx->launches;
        report_begin(report, cfg->refine ? "plmr" : "plm", cfg->workers, cfg->seed);
        OutArr<int32_t> dz(ctx, z, g->n);
        DevTimer t(ctx);
        t.start();
        const int64_t k = louvain_run_dev(ctx, gg, *cfg, dz.d, Report{report});
        const double ms = t.stop_ms();
        if (report) {
            report->total_ms = ms;
            report_quality(ctx, gg, dz.d, std::max<int64_t>(k, 1), cfg->gamma, report);
            report->community_count = k;
            report->kernel_launches = ctx->launches - launches0;
        }
        dz.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_epp_run(cd_ctx *ctx, const cd_graph *g, const cd_ensemble_config *cfg, int32_t *z, cd_report *report) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || z), CD_EINVAL, "invalid argument");
        cd_graph *gg = const_cast<cd_graph *>(g);
        const int64_t launches0 = ctx->launches;
        report_begin(report, "epp", cfg->workers, cfg->seed);
        OutArr<int32_t> dz(ctx, z, g->n);
        DevTimer t(ctx);
        t.start();
        const int64_t k = epp_run_dev(ctx, gg, *cfg, dz.d, Report{report});
        const double ms = t.stop_ms();
        if (report) {
            report->total_ms = ms;
            report_quality(ctx, gg, dz.d, std::max<int64_t>(k, 1), 1.0, report);
            report->community_count = k;
            report->kernel_launches = ctx->launches - launches0;
        }
        dz.finish();
        ctx_sync(ctx);
    })
}

cd_status cd_epp_run_bases(cd_ctx *ctx, const cd_graph *g, const cd_ensemble_config *cfg,
                           const int32_t *const *bases, int32_t *z, cd_report *report) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && g && cfg && (g->n == 0 || z), CD_EINVAL, "invalid argument");
        CD_REQUIRE(cfg->ensemble_size >= 1, CD_EINVAL, "ensemble size must be >= 1");  // H/ensemble.hpp:113-114
        CD_REQUIRE(bases, CD_EINVAL, "empty ensemble");
        cd_graph *gg = const_cast<cd_graph *>(g);
        const int64_t launches0 = ctx->launches, b = cfg->ensemble_size;
        report_begin(report, "epp", cfg->workers, cfg->seed);
        std::vector<std::unique_ptr<InArr<int32_t>>> ins;
        std::vector<const int32_t *> ptrs;
        for (int64_t i = 0; i < b; ++i) {
            CD_REQUIRE(g->n == 0 || bases[i], CD_EINVAL, "invalid argument");
            ins.emplace_back(new InArr<int32_t>(ctx, bases[i], g->n));
            ptrs.push_back(ins.back()->d);
        }
        OutArr<int32_t> dz(ctx, z, g->n);
        DevTimer t(ctx);
        t.start();
        const int64_t k = epp_run_dev(ctx, gg, *cfg, dz.d, Report{report}, ptrs.data());
        const double ms = t.stop_ms();
        if (report) {
            report->total_ms = ms;
            report_quality(ctx, gg, dz.d, std::max<int64_t>(k, 1), 1.0, report);
            report->community_count = k;
            report->kernel_launches = ctx->launches - launches0;
        }
        dz.finish();
        ctx_sync(ctx);
    })
}

// ---- text ingest -------------------------------------------------------------------

namespace {
std::vector<char> read_file(const char *path) {
    FILE *f = std::fopen(path, "rb");
    if (!f)
        fail(CD_EINPUT, std::string("cannot open ") + path);  // H/io.hpp:23-28
    std::vector<char> buf;
    char tmp[1 << 16];
    size_t r;
    while ((r = std::fread(tmp, 1, sizeof(tmp), f)) > 0)
        buf.insert(buf.end(), tmp, tmp + r);
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad)
        fail(CD_EINPUT, std::string("cannot read ") + path);
    return buf;
}
}  // namespace

cd_status cd_graph_read_metis(cd_ctx *ctx, const char *text, int64_t len, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && len >= 0 && (len == 0 || text), CD_EINVAL, "invalid argument");
        *out = read_metis_dev(ctx, text, len, "<metis>");
    })
}

cd_status cd_graph_read_edge_list(cd_ctx *ctx, const char *text, int64_t len, int32_t merge, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && len >= 0 && (len == 0 || text), CD_EINVAL, "invalid argument");
        *out = read_edge_list_dev(ctx, text, len, merge != 0, "<edge list>");
    })
}

cd_status cd_graph_load_metis(cd_ctx *ctx, const char *path, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && path, CD_EINVAL, "invalid argument");
        const std::vector<char> buf = read_file(path);
        *out = read_metis_dev(ctx, buf.data(), static_cast<int64_t>(buf.size()), path);
    })
}

cd_status cd_graph_load_edge_list(cd_ctx *ctx, const char *path, int32_t merge, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && path, CD_EINVAL, "invalid argument");
        const std::vector<char> buf = read_file(path);
        *out = read_edge_list_dev(ctx, buf.data(), static_cast<int64_t>(buf.size()), merge != 0, path);
    })
}

cd_status cd_graph_original_ids(const cd_graph *g, uint64_t *out) {
    cd_ctx *ctx = g ? g->ctx : nullptr;
    CD_GUARD(ctx, {
        CD_REQUIRE(g && out, CD_EINVAL, "invalid argument");
        CD_REQUIRE(g->orig_ids.p != nullptr || g->n == 0, CD_EINVAL, "graph was not read from an edge list");
        if (g->n)
            CD_CUDA(cudaMemcpyAsync(out, g->orig_ids.p, g->n * sizeof(uint64_t), cudaMemcpyDefault, ctx->stream));
        ctx_sync(ctx);
    })
}

// ---- sharded execution ----------------------------------------------------------

cd_status cd_nccl_unique_id(uint8_t id[128]) {
    CD_GUARD(static_cast<cd_ctx *>(nullptr), CD_REQUIRE(id, CD_EINVAL, "null argument"); nccl_unique_id(id))
}

cd_status cd_ctx_attach_nccl(cd_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t id[128]) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && id && nranks >= 1 && rank >= 0 && rank < nranks, CD_EINVAL, "invalid argument");
        Comm *c = comm_nccl_create(nranks, rank, id);
        delete ctx->comm;
        ctx->comm = c;
    })
}

cd_status cd_loopback_create(int32_t nranks, cd_loopback **out) {
    CD_GUARD(static_cast<cd_ctx *>(nullptr), {
        CD_REQUIRE(out && nranks >= 1, CD_EINVAL, "invalid argument");
        auto *lb = new cd_loopback();
        lb->nranks = nranks;
        lb->slot.assign(nranks, nullptr);
        lb->host.resize(nranks);
        *out = lb;
    })
}

cd_status cd_loopback_destroy(cd_loopback *lb) {
    delete lb;
    return CD_OK;
}

cd_status cd_ctx_attach_loopback(cd_ctx *ctx, cd_loopback *lb, int32_t rank) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && lb && rank >= 0 && rank < lb->nranks, CD_EINVAL, "invalid argument");
        Comm *c = comm_loopback_create(lb, rank);
        delete ctx->comm;
        ctx->comm = c;
    })
}

cd_status cd_ctx_detach(cd_ctx *ctx) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx, CD_EINVAL, "null context");
        delete ctx->comm;
        ctx->comm = nullptr;
    })
}

cd_status cd_ctx_world(const cd_ctx *ctx, int32_t *rank, int32_t *size) {
    CD_GUARD(static_cast<cd_ctx *>(nullptr), {
        CD_REQUIRE(ctx, CD_EINVAL, "null context");
        if (rank)
            *rank = world_rank(ctx);
        if (size)
            *size = world_size(ctx);
    })
}

cd_status cd_shard_bounds(int64_t n, const int64_t *off, int32_t nranks, int64_t *bounds) {
    CD_GUARD(static_cast<cd_ctx *>(nullptr), {
        CD_REQUIRE(n >= 0 && off && bounds && nranks >= 1, CD_EINVAL, "invalid argument");
        shard_bounds_host(n, off, nranks, bounds);
    })
}

cd_status cd_graph_shard(cd_ctx *ctx, const cd_graph *full, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && full && out, CD_EINVAL, "invalid argument");
        *out = graph_shard_dev(ctx, full);
    })
}

cd_status cd_graph_from_csr_rows(cd_ctx *ctx, int64_t n, const int64_t *off, int64_t lo, int64_t hi,
                                 const int32_t *col, const float *w, cd_graph **out) {
    CD_GUARD(ctx, {
        CD_REQUIRE(ctx && out && off && n >= 0 && n < INT32_MAX, CD_EINVAL, "invalid argument");
        CD_REQUIRE(0 <= lo && lo <= hi && hi <= n, CD_EINVAL, "row range out of bounds");
        *out = graph_from_rows_dev(ctx, n, off, lo, hi, col, w);
    })
}

}  // extern "C"
