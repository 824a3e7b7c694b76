// ref_capi.cpp -- C ABI over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile from the
// reference's own headers where they lie (/root/reference/proj/include) into
// oracle/_ref/libcommdet_ref.so (git-ignored; it travels to the GPU box as a
// built artefact).  No reference source is copied into this repository.
// Used by tests/ (to pin the C oracle and the GPU path) and by
// bench.py --impl reference / cpu_baseline (the reference's CPU timing).
//
// Every entry point calls the reference's public API unchanged:
//   Graph::from_edges            H/graph.hpp:48
//   generate_planted             H/generator.hpp:52
//   run_plp / dominant_label / is_stable   H/plp.hpp:67, :32, :57
//   run_plm / run_plmr / move_phase / coarsen / delta_mod   H/louvain.hpp
//   run_epp / combine_hashed     H/ensemble.hpp:111, :86
//   modularity / coverage        H/quality.hpp:35, :21
//   io::read_metis / read_edge_list   H/io.hpp:83, :190
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include <commdet/ensemble.hpp>
#include <commdet/generator.hpp>
#include <commdet/io.hpp>
#include <commdet/louvain.hpp>
#include <commdet/plp.hpp>
#include <commdet/quality.hpp>

namespace cd = commdet;

namespace {
thread_local char g_err[512];

int fail(const std::exception &e, int code) {
    std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
    return code;
}

template <typename F>
int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const cd::input_error &e) {
        return fail(e, -1);
    } catch (const std::invalid_argument &e) {
        return fail(e, -2);
    } catch (const std::domain_error &e) {
        return fail(e, -3);
    } catch (const std::out_of_range &e) {
        return fail(e, -4);
    } catch (const std::exception &e) {
        return fail(e, -9);
    }
}

cd::Partition to_partition(int64_t n, const int32_t *z, int64_t ub) {
    cd::Partition p;
    p.data().resize(static_cast<size_t>(n));
    cd::index mx = 0;
    for (int64_t u = 0; u < n; ++u) {
        p[u] = static_cast<cd::index>(static_cast<uint32_t>(z[u]));
        mx = std::max(mx, p[u] + 1);
    }
    p.set_upper_bound(ub > 0 ? static_cast<cd::index>(ub) : std::max<cd::index>(mx, 1));
    return p;
}

void from_partition(const cd::Partition &p, int32_t *out) {
    for (size_t u = 0; u < p.size(); ++u)
        out[u] = static_cast<int32_t>(p[u]);
}

struct Report {
    double total_ms, modularity, coverage;
    int64_t community_count, iterations, levels;
    double base_ms, combine_ms, coarsen_ms, final_ms;
};

void fill_report(const cd::RunReport &r, Report *out) {
    if (!out)
        return;
    out->total_ms = r.total_ms;
    out->modularity = r.modularity;
    out->coverage = r.coverage;
    out->community_count = static_cast<int64_t>(r.community_count);
    out->iterations = static_cast<int64_t>(r.iterations.size());
    out->levels = static_cast<int64_t>(r.levels.size());
    out->base_ms = r.base_ms;
    out->combine_ms = r.combine_ms;
    out->coarsen_ms = r.coarsen_ms;
    out->final_ms = r.final_ms;
}
} // namespace

extern "C" {

const char *ref_last_error(void) { return g_err; }

void ref_graph_free(void *g) { delete static_cast<cd::Graph *>(g); }

// Graph::from_edges (H/graph.hpp:48-81)
int ref_graph_from_edges(int64_t n, int64_t m, const int32_t *eu, const int32_t *ev, const double *ew,
                         int merge, void **out) {
    return guarded([&] {
        cd::EdgeList edges(static_cast<size_t>(m));
        for (int64_t i = 0; i < m; ++i)
            edges[i] = {static_cast<cd::node>(static_cast<uint32_t>(eu[i])),
                        static_cast<cd::node>(static_cast<uint32_t>(ev[i])), ew ? ew[i] : 1.0};
        *out = new cd::Graph(cd::Graph::from_edges(static_cast<cd::count>(n), edges, merge != 0));
    });
}

// Canonical CSR -> reference Graph via from_edges over u <= v entries.
int ref_graph_from_csr(int64_t n, const int64_t *off, const int32_t *col, const double *w, void **out) {
    return guarded([&] {
        cd::EdgeList edges;
        edges.reserve(static_cast<size_t>(off[n] / 2 + 1));
        for (int64_t u = 0; u < n; ++u)
            for (int64_t i = off[u]; i < off[u + 1]; ++i)
                if (col[i] >= u)
                    edges.push_back({static_cast<cd::node>(u), static_cast<cd::node>(col[i]), w ? w[i] : 1.0});
        *out = new cd::Graph(cd::Graph::from_edges(static_cast<cd::count>(n), edges));
    });
}

void ref_graph_info(const void *gp, int64_t *n, int64_t *D, int64_t *m, double *total) {
    const auto &g = *static_cast<const cd::Graph *>(gp);
    *n = static_cast<int64_t>(g.node_count());
    int64_t d = 0;
    for (cd::node u = 0; u < g.node_count(); ++u)
        d += static_cast<int64_t>(g.degree(u));
    *D = d;
    *m = static_cast<int64_t>(g.edge_count());
    *total = g.total_edge_weight();
}

// CSR through the public iteration API (for_neighbors, H/graph.hpp:125-129).
void ref_graph_csr(const void *gp, int64_t *off, int32_t *col, double *w, double *vol, double *loop) {
    const auto &g = *static_cast<const cd::Graph *>(gp);
    int64_t pos = 0;
    off[0] = 0;
    for (cd::node u = 0; u < g.node_count(); ++u) {
        g.for_neighbors(u, [&](cd::node v, cd::edgeweight wt) {
            col[pos] = static_cast<int32_t>(v);
            w[pos] = wt;
            ++pos;
        });
        off[u + 1] = pos;
        vol[u] = g.volume(u);
        loop[u] = g.loop_weight(u);
    }
}

// generate_planted (H/generator.hpp:52-104)
int ref_generate_planted(int64_t n, int64_t k, double p_in, double p_out, uint64_t seed, int workers, void **out,
                         int32_t *truth) {
    return guarded([&] {
        cd::PlantedPartitionSpec s{static_cast<cd::count>(n), static_cast<cd::count>(k), p_in, p_out, seed};
        auto [g, t] = cd::generate_planted(s, workers);
        if (truth)
            from_partition(t, truth);
        *out = new cd::Graph(std::move(g));
    });
}

int ref_modularity(const void *gp, const int32_t *z, int64_t ub, double gamma, double *q, double *cov) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::Partition p = to_partition(static_cast<int64_t>(g.node_count()), z, ub);
        *cov = cd::coverage(g, p);
        *q = cd::modularity(g, p, gamma);
    });
}

int ref_dominant_label(const void *gp, const int32_t *z, int64_t u, int32_t *out) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        *out = static_cast<int32_t>(
            cd::dominant_label(g, to_partition(static_cast<int64_t>(g.node_count()), z, 0), static_cast<cd::node>(u)));
    });
}

int ref_is_stable(const void *gp, const int32_t *z) {
    const auto &g = *static_cast<const cd::Graph *>(gp);
    return cd::is_stable(g, to_partition(static_cast<int64_t>(g.node_count()), z, 0)) ? 1 : 0;
}

// run_plp (H/plp.hpp:67-149)
int ref_run_plp(const void *gp, int64_t theta, int64_t max_iterations, int randomize, uint64_t seed, int workers,
                const int32_t *initial, int32_t *labels, void *report, int64_t *updated_trace, int64_t trace_cap) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::PlpConfig cfg;
        cfg.theta = theta;
        cfg.max_iterations = static_cast<cd::count>(max_iterations);
        cfg.randomize_order = randomize != 0;
        cfg.seed = seed;
        cfg.workers = workers;
        std::optional<cd::Partition> init;
        if (initial)
            init = to_partition(static_cast<int64_t>(g.node_count()), initial, 0);
        auto [z, r] = cd::run_plp(g, cfg, init);
        from_partition(z, labels);
        fill_report(r, static_cast<Report *>(report));
        for (size_t i = 0; updated_trace && i < r.iterations.size() && static_cast<int64_t>(i) < trace_cap; ++i)
            updated_trace[i] = static_cast<int64_t>(r.iterations[i].updated);
    });
}

// run_plm / run_plmr (H/louvain.hpp:290-301)
int ref_run_louvain(const void *gp, double gamma, int64_t max_move_iterations, int64_t max_levels, uint64_t seed,
                    int workers, int refine, int32_t *z_out, void *report) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::LouvainConfig cfg;
        cfg.gamma = gamma;
        cfg.max_move_iterations = static_cast<cd::count>(max_move_iterations);
        cfg.max_levels = static_cast<cd::count>(max_levels);
        cfg.seed = seed;
        cfg.workers = workers;
        auto [z, r] = refine ? cd::run_plmr(g, cfg) : cd::run_plm(g, cfg);
        from_partition(z, z_out);
        fill_report(r, static_cast<Report *>(report));
    });
}

// move_phase (H/louvain.hpp:65-141), sequential when workers == 1
int ref_move_phase(const void *gp, int32_t *z, int64_t ub, double gamma, int64_t max_move_iterations, int workers,
                   int *changed) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::Partition p = to_partition(static_cast<int64_t>(g.node_count()), z, ub);
        cd::LouvainConfig cfg;
        cfg.gamma = gamma;
        cfg.max_move_iterations = static_cast<cd::count>(max_move_iterations);
        cfg.workers = workers;
        *changed = cd::move_phase(g, p, cfg) ? 1 : 0;
        from_partition(p, z);
    });
}

// move_phase with a MoveObserver (H/louvain.hpp:60, :127-128) that logs every
// applied move and the modularity of the partition right after it
int ref_move_phase_log(const void *gp, int32_t *z, int64_t ub, double gamma, int64_t max_move_iterations,
                       int workers, int32_t *lu, int32_t *lc, int32_t *ld, double *lgain, double *lq, int64_t cap,
                       int64_t *count, int *changed) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::Partition p = to_partition(static_cast<int64_t>(g.node_count()), z, ub);
        cd::LouvainConfig cfg;
        cfg.gamma = gamma;
        cfg.max_move_iterations = static_cast<cd::count>(max_move_iterations);
        cfg.workers = workers;
        int64_t k = 0;
        *changed = cd::move_phase(g, p, cfg,
                                  [&](cd::node u, cd::index c, cd::index d, double gain) {
                                      if (k < cap) {
                                          lu[k] = static_cast<int32_t>(u);
                                          lc[k] = static_cast<int32_t>(c);
                                          ld[k] = static_cast<int32_t>(d);
                                          lgain[k] = gain;
                                          if (lq)
                                              lq[k] = cd::modularity(g, p);
                                      }
                                      ++k;
                                  })
                       ? 1
                       : 0;
        *count = k;
        from_partition(p, z);
    });
}

// delta_mod (H/louvain.hpp:37-56)
int ref_delta_mod(const void *gp, const int32_t *z, int64_t ub, int64_t u, int64_t target, double gamma,
                  double *out) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::Partition p = to_partition(static_cast<int64_t>(g.node_count()), z, ub);
        auto vols = cd::community_volumes(g, p);
        *out = cd::delta_mod(g, p, vols, static_cast<cd::node>(u), static_cast<cd::index>(target), gamma);
    });
}

// coarsen (H/louvain.hpp:154-220); pi written to pi_out
int ref_coarsen(const void *gp, const int32_t *z, int workers, void **coarse, int32_t *pi_out) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::Partition p = to_partition(static_cast<int64_t>(g.node_count()), z, 0);
        auto cr = cd::coarsen(g, p, workers);
        for (size_t v = 0; v < cr.pi.size(); ++v)
            pi_out[v] = static_cast<int32_t>(cr.pi[v]);
        *coarse = new cd::Graph(std::move(cr.coarse));
    });
}

// Partition::compacted (H/partition.hpp:39-53) and community_count (:55-60)
int64_t ref_compacted(int64_t n, const int32_t *z, int32_t *out) {
    cd::Partition p = to_partition(n, z, 0);
    cd::Partition c = p.compacted();
    from_partition(c, out);
    return static_cast<int64_t>(p.community_count());
}

// combine_hashed (H/ensemble.hpp:86-107)
int ref_combine_hashed(int64_t b, int64_t n, const int32_t *const *solutions, int workers, int32_t *out) {
    return guarded([&] {
        std::vector<cd::Partition> sols;
        for (int64_t i = 0; i < b; ++i)
            sols.push_back(to_partition(n, solutions[i], 0));
        from_partition(cd::combine_hashed(sols, workers), out);
    });
}

int ref_combine_exact(int64_t b, int64_t n, const int32_t *const *solutions, int32_t *out) {
    return guarded([&] {
        std::vector<cd::Partition> sols;
        for (int64_t i = 0; i < b; ++i)
            sols.push_back(to_partition(n, solutions[i], 0));
        from_partition(cd::combine_exact(sols), out);
    });
}

uint64_t ref_djb2(const uint8_t *data, uint64_t len) { return cd::djb2(data, static_cast<size_t>(len)); }

// run_epp (H/ensemble.hpp:111-199): EPP(b, PLP, PLMR)
int ref_run_epp(const void *gp, int64_t ensemble_size, uint64_t seed, int workers, int32_t *z_out, void *report) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::EnsembleConfig cfg;
        cfg.ensemble_size = static_cast<cd::count>(ensemble_size);
        cfg.seed = seed;
        cfg.workers = workers;
        auto [z, r] = cd::run_epp(g, cfg);
        from_partition(z, z_out);
        fill_report(r, static_cast<Report *>(report));
    });
}

int ref_max_threads(void) { return omp_get_max_threads(); }

// io::write_metis / write_partition / write_community_graph (H/io.hpp:168, :248, :279)
int ref_write_metis(const void *gp, const char *path) {
    return guarded([&] { cd::io::write_metis(*static_cast<const cd::Graph *>(gp), path); });
}

int ref_write_partition(int64_t n, const int32_t *z, const char *path) {
    return guarded([&] { cd::io::write_partition(to_partition(n, z, 0), path); });
}

int ref_write_community_graph(const void *gp, const int32_t *z, const char *path) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        cd::io::write_community_graph(g, to_partition(static_cast<int64_t>(g.node_count()), z, 0), path);
    });
}

// graph_rand_index (H/quality.hpp:56-69)
int ref_graph_rand_index(const void *gp, const int32_t *a, const int32_t *b, double *out) {
    return guarded([&] {
        const auto &g = *static_cast<const cd::Graph *>(gp);
        const int64_t n = static_cast<int64_t>(g.node_count());
        *out = cd::graph_rand_index(g, to_partition(n, a, 0), to_partition(n, b, 0));
    });
}

// io::read_metis (H/io.hpp:83-165)
int ref_read_metis(const char *path, void **out) {
    return guarded([&] { *out = new cd::Graph(cd::io::read_metis(path)); });
}

// io::read_edge_list (H/io.hpp:190-237); ids (nullable) receives n original ids
int ref_read_edge_list(const char *path, int merge, void **out, uint64_t *ids, int64_t ids_cap) {
    return guarded([&] {
        std::vector<std::uint64_t> orig;
        *out = new cd::Graph(cd::io::read_edge_list(path, merge != 0, &orig));
        if (ids)
            for (size_t i = 0; i < orig.size() && static_cast<int64_t>(i) < ids_cap; ++i)
                ids[i] = orig[i];
    });
}

} // extern "C"
