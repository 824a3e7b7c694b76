// Reference-style caller compiled against the drop-in C++ shim
// (include/commdet/gpu.hpp).  The code reads like the reference's own unit
// tests (T/test_*.cpp); only the include changes.  Exit code 0 = all pass.
#define COMMDET_GPU_DROP_IN
#include <commdet/gpu.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

using namespace commdet;

static int failures = 0;
#define CHECK(cond)                                                                                  \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                              \
            ++failures;                                                                              \
        }                                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                  \
    do {                                                                                             \
        bool thrown_ = false;                                                                        \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const type &) {                                                                     \
            thrown_ = true;                                                                          \
        } catch (...) {                                                                              \
        }                                                                                            \
        if (!thrown_) {                                                                              \
            std::printf("FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #type);      \
            ++failures;                                                                              \
        }                                                                                            \
    } while (0)

static Graph barbell() {
    return Graph::from_edges(6, {{0, 1, 1}, {0, 2, 1}, {1, 2, 1}, {3, 4, 1}, {3, 5, 1}, {4, 5, 1}, {2, 3, 1}});
}
static Graph two_triangles() {
    return Graph::from_edges(6, {{0, 1, 1}, {0, 2, 1}, {1, 2, 1}, {3, 4, 1}, {3, 5, 1}, {4, 5, 1}});
}
static Partition triangles() {
    Partition z;
    z.data() = {0, 0, 0, 1, 1, 1};
    z.set_upper_bound(2);
    return z;
}

int main() {
    // graph (T/test_graph.cpp)
    Graph g = barbell();
    CHECK(g.node_count() == 6 && g.edge_count() == 7 && g.total_edge_weight() == 7.0);
    CHECK(g.volume(2) == 3.0 && g.degree(2) == 3);
    Graph loop = Graph::from_edges(1, {{0, 0, 2.0}});
    CHECK(loop.total_edge_weight() == 2.0 && loop.volume(0) == 4.0 && loop.loop_weight(0) == 2.0);
    CHECK_THROWS_AS(Graph::from_edges(2, {{0, 2, 1}}), input_error);
    CHECK_THROWS_AS(Graph::from_edges(2, {{0, 1, 1}, {1, 0, 1}}), input_error);
    Graph merged = Graph::from_edges(2, {{0, 1, 1}, {1, 0, 1}}, true);
    CHECK(merged.edge_count() == 1 && merged.total_edge_weight() == 2.0);
    CHECK_THROWS_AS(g.volume(6), std::out_of_range);

    // quality (T/test_quality.cpp)
    CHECK(std::abs(modularity(g, Partition(6, 0))) < 1e-15);
    CHECK(std::abs(modularity(g, triangles()) - 5.0 / 14.0) < 1e-15);
    CHECK(std::abs(modularity(two_triangles(), triangles()) - 0.5) < 1e-15);
    CHECK(std::abs(coverage(g, triangles()) - 6.0 / 7.0) < 1e-15);
    Graph empty = Graph::from_edges(4, {});
    CHECK_THROWS_AS(modularity(empty, singleton_partition(empty)), std::domain_error);

    // PLP (T/test_plp.cpp)
    Graph star = Graph::from_edges(6, {{0, 1, 5}, {0, 2, 1}, {0, 3, 1}, {0, 4, 1}, {0, 5, 1}});
    Partition zs;
    zs.data() = {0, 1, 7, 7, 7, 7};
    zs.set_upper_bound(8);
    CHECK(dominant_label(star, zs, 0) == 1);
    CHECK(dominant_label(g, singleton_partition(g), 0) == 1);
    CHECK_THROWS_AS(dominant_label(Graph::from_edges(2, {}), singleton_partition(Graph::from_edges(2, {})), 0),
                    std::invalid_argument);
    PlpConfig pc;
    pc.theta = 0;
    auto [zp, rp] = run_plp(two_triangles(), pc);
    CHECK(zp.community_count() == 2);
    CHECK(std::abs(modularity(two_triangles(), zp.compacted()) - 0.5) < 1e-12);
    CHECK(is_stable(two_triangles(), zp));
    auto [ze, re] = run_plp(Graph::from_edges(5, {}), PlpConfig{.theta = 1});
    CHECK(re.iterations.size() == 1 && re.iterations[0].updated == 0);

    // Louvain (T/test_louvain.cpp)
    auto cr = coarsen(g, triangles());
    CHECK(cr.coarse.node_count() == 2 && cr.coarse.total_edge_weight() == 7.0);
    CHECK(cr.coarse.loop_weight(0) == 3.0 && cr.coarse.volume(1) == 7.0);
    CHECK((cr.pi == std::vector<node>{0, 0, 0, 1, 1, 1}));
    Partition nc;
    nc.data() = {5, 5, 5, 9, 9, 9};
    nc.set_upper_bound(10);
    CHECK_THROWS_AS(coarsen(g, nc), std::invalid_argument);
    Partition coarse;
    coarse.data() = {4, 9};
    coarse.set_upper_bound(10);
    // commdet::index collides with POSIX index() under a using-directive, as in
    // the reference's own tests (T/test_louvain.cpp:21)
    CHECK((prolong(coarse, {0, 0, 0, 1, 1, 1}).data() == std::vector<commdet::index>{4, 4, 4, 9, 9, 9}));
    CHECK_THROWS_AS(prolong(coarse, {0, 2}), std::out_of_range);
    LouvainConfig lc;
    auto [zl, rl] = run_plm(g, lc);
    CHECK(std::abs(rl.modularity - 5.0 / 14.0) < 1e-12 && rl.algorithm == "plm");
    auto [zr, rr] = run_plmr(two_triangles(), lc);
    CHECK(std::abs(rr.modularity - 0.5) < 1e-12 && rr.algorithm == "plmr");
    CHECK_THROWS_AS(run_plm(Graph::from_edges(3, {}), lc), std::domain_error);
    Partition sing = singleton_partition(two_triangles());
    CHECK(move_phase(two_triangles(), sing, lc));

    // ensemble (T/test_ensemble.cpp)
    const std::uint8_t one[] = {1};
    CHECK(djb2(nullptr, 0) == 5381 && djb2(one, 1) == 5381 * 33 + 1);
    Partition a, b;
    a.data() = {0, 0, 1, 1};
    b.data() = {0, 1, 1, 0};
    CHECK(combine_hashed({a, b}).upper_bound() == 4);
    CHECK_THROWS_AS(combine_hashed({Partition(3, 0), Partition(4, 0)}), std::invalid_argument);
    EnsembleConfig ec;
    auto [zx, rx] = run_epp(two_triangles(), ec);
    CHECK(std::abs(rx.modularity - 0.5) < 1e-12 && rx.algorithm == "epp");
    ec.ensemble_size = 0;
    CHECK_THROWS_AS(run_epp(g, ec), std::invalid_argument);

    // generator (T/test_generator.cpp)
    auto [pg, truth] = generate_planted({6, 2, 1.0, 0.0, 1});
    CHECK(pg == two_triangles());
    CHECK_THROWS_AS(generate_planted({10, 0, 0.5, 0.1, 1}), std::invalid_argument);

    // io (T/test_io.cpp): METIS / edge-list readers, parsed on the device
    {
        const char *mp = "/tmp/shim_kat_tri.metis";
        if (FILE *f = std::fopen(mp, "w")) {
            std::fputs("% two triangles\n6 6\n2 3\n1 3\n1 2\n5 6\n4 6\n4 5\n", f);
            std::fclose(f);
        }
        CHECK(io::read_metis(mp) == two_triangles());
        const char *bad = "/tmp/shim_kat_bad.metis";
        if (FILE *f = std::fopen(bad, "w")) {
            std::fputs("2 1\n2\n\n", f);
            std::fclose(f);
        }
        CHECK_THROWS_AS(io::read_metis(bad), input_error);  // asymmetric adjacency
        CHECK_THROWS_AS(io::read_metis("/tmp/shim_kat_missing.metis"), input_error);
        const char *ep = "/tmp/shim_kat.edges";
        if (FILE *f = std::fopen(ep, "w")) {
            std::fputs("# c\n10 20\n20 30 2.5\n", f);
            std::fclose(f);
        }
        std::vector<std::uint64_t> ids;
        Graph eg = io::read_edge_list(ep, false, &ids);
        CHECK((eg.node_count() == 3 && eg.edge_count() == 2 && ids == std::vector<std::uint64_t>{10, 20, 30}));
        std::remove(mp);
        std::remove(bad);
        std::remove(ep);
    }

    {
        // sequential moves strictly increase modularity (T/test_louvain.cpp:85-98 with a MoveObserver)
        std::mt19937_64 rng(404);
        std::uniform_real_distribution<double> coin(0.0, 1.0);
        int observed = 0;
        for (int i = 0; i < 20; ++i) {
            const count n = 8 + i % 12;
            EdgeList edges;
            for (node u = 0; u < n; ++u)
                for (node v = u + 1; v < n; ++v)
                    if (coin(rng) < 0.35)
                        edges.push_back({u, v, 1.0});
            if (edges.empty())
                edges.push_back({0, 1, 1.0});
            Graph rg = Graph::from_edges(n, edges);
            Partition z = singleton_partition(rg);
            double last = modularity(rg, z);
            LouvainConfig cfg;
            cfg.workers = 1;
            move_phase(rg, z, cfg, [&](node u, commdet::index c, commdet::index d, double gain) {
                const double now = modularity(rg, z);
                CHECK(now > last);
                CHECK(z[u] == d && c != d && gain > 0.0);
                last = now;
                ++observed;
            });
        }
        CHECK(observed > 0);
        // no moves on the optimum; an observer that throws propagates
        Partition zt = triangles();
        CHECK(!move_phase(two_triangles(), zt, LouvainConfig{}, [](node, commdet::index, commdet::index, double) {}));
        Partition zs = singleton_partition(g);
        CHECK_THROWS_AS(move_phase(g, zs, LouvainConfig{},
                                   [](node, commdet::index, commdet::index, double) { throw std::runtime_error("x"); }),
                        std::runtime_error);
    }
    {
        // epp with singleton base stub equals plain plm (T/test_ensemble.cpp:101-113)
        EnsembleConfig cfg;
        cfg.ensemble_size = 1;
        cfg.final_algo = Algo::plm;
        cfg.workers = 1;
        int calls = 0;
        cfg.base_override = [&](const Graph &graph, std::uint64_t) {
            ++calls;
            return singleton_partition(graph);
        };
        auto [ze, re] = run_epp(g, cfg);
        LouvainConfig lc;
        lc.workers = 1;
        auto [zp, rp] = run_plm(g, lc);
        CHECK(calls == 1);
        CHECK(ze == zp.compacted());
        CHECK(std::abs(re.modularity - rp.modularity) < 1e-12);
        // the hook's partitions must cover the graph
        cfg.ensemble_size = 2;
        cfg.base_override = [](const Graph &, std::uint64_t s) { return Partition::singletons(s == 1 ? 6 : 5); };
        CHECK_THROWS_AS(run_epp(g, cfg), std::invalid_argument);
    }

    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
