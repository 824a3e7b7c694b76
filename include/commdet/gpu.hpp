// commdet/gpu.hpp -- header-only C++ drop-in for the reference detector
// interface (/root/reference/proj/include/commdet, "H/" below), implemented
// over the C ABI of libcommdet_cuda.so (include/commdet_cuda.h).
//
// Same names, signatures, value types and exception types as the reference:
//   Graph::from_edges / from_adjacency      H/graph.hpp:48, :85
//   Partition (+ compacted, community_count) H/partition.hpp:13-91
//   run_plp / run_plm / run_plmr / run_epp   H/plp.hpp:67, H/louvain.hpp:290/297, H/ensemble.hpp:111
//   modularity / coverage                    H/quality.hpp:35, :21
//   coarsen / prolong / move_phase           H/louvain.hpp:154, :223, :65
//   combine_hashed / dominant_label / is_stable / generate_planted
// The types live in namespace commdet::gpu; define COMMDET_GPU_DROP_IN before
// including to also export them as namespace commdet (then do not include
// the reference headers in the same translation unit).
//
// Differences a caller can observe:
//   * node ids / labels must fit int32 (std::out_of_range otherwise);
//   * stored edge weights are fp32 (decisions and sums are fp64);
//   * PLP/PLM update order is the device's seeded bucket schedule, so
//     `workers` and `randomize_order` do not change the result;
//   * move_phase with a MoveObserver runs the reference's one-worker order
//     (cd_move_phase_sequential), whose move sequence the reference defines
//     only for workers == 1 (H/louvain.hpp:58-60).
#pragma once

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <numeric>
#include <vector>

#include "../commdet_cuda.h"

namespace commdet {
namespace gpu {

using node = std::uint64_t;
using index = std::uint64_t;
using count = std::uint64_t;
using edgeweight = double;

/// Thrown on malformed input data (H/graph.hpp:21-24).
class input_error : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(cd_status s) {
    if (s == CD_OK)
        return;
    const std::string msg = cd_last_error();
    switch (s) {
    case CD_EINPUT:
        throw input_error(msg);
    case CD_EINVAL:
        throw std::invalid_argument(msg);
    case CD_EDOMAIN:
        throw std::domain_error(msg);
    case CD_ERANGE:
        throw std::out_of_range(msg);
    case CD_ENOMEM:
        throw std::bad_alloc();
    default:
        throw std::runtime_error("commdet gpu: " + msg);
    }
}

inline int32_t to_i32(std::uint64_t v, const char *what) {
    if (v > static_cast<std::uint64_t>(INT32_MAX))
        throw std::out_of_range(std::string(what) + " does not fit the device's int32 ids");
    return static_cast<int32_t>(v);
}
}  // namespace detail

/// One CUDA device context (stream + memory pool).  Not thread-safe.
class Context {
  public:
    explicit Context(int device = 0) { detail::check(cd_ctx_create(device, &ctx_)); }
    ~Context() { cd_ctx_destroy(ctx_); }
    Context(const Context &) = delete;
    Context &operator=(const Context &) = delete;
    cd_ctx *get() const { return ctx_; }
    static Context &instance() {
        static Context c(0);
        return c;
    }

  private:
    cd_ctx *ctx_ = nullptr;
};

struct Edge {
    node u;
    node v;
    edgeweight w;
};
using EdgeList = std::vector<Edge>;

inline int resolve_workers(int workers) { return workers > 0 ? workers : 1; }

/// Device-resident undirected weighted graph (H/graph.hpp:38-272).
class Graph {
  public:
    Graph() = default;

    static Graph from_edges(count node_count, const EdgeList &edges, bool merge_duplicates = false) {
        const int32_t n = detail::to_i32(node_count, "node count");
        std::vector<int32_t> u(edges.size()), v(edges.size());
        std::vector<float> w(edges.size());
        bool weighted = false;
        for (std::size_t i = 0; i < edges.size(); ++i) {
            const Edge &e = edges[i];
            if (e.u >= node_count || e.v >= node_count)
                throw input_error("edge endpoint out of range: " + std::to_string(e.u) + "," + std::to_string(e.v));
            if (!(e.w > 0.0))
                throw input_error("nonpositive edge weight on edge " + std::to_string(e.u) + "," +
                                  std::to_string(e.v));
            u[i] = static_cast<int32_t>(e.u);
            v[i] = static_cast<int32_t>(e.v);
            w[i] = static_cast<float>(e.w);
            weighted = weighted || e.w != 1.0;
        }
        cd_graph *h = nullptr;
        detail::check(cd_graph_from_edges(Context::instance().get(), n, static_cast<int64_t>(edges.size()),
                                          u.empty() ? nullptr : u.data(), v.empty() ? nullptr : v.data(),
                                          weighted ? w.data() : nullptr, merge_duplicates ? 1 : 0, &h));
        return Graph(h);
    }

    /// Full symmetric adjacency, rows sorted (H/graph.hpp:85-103).
    static Graph from_adjacency(const std::vector<std::vector<std::pair<node, edgeweight>>> &adj) {
        const int64_t n = detail::to_i32(adj.size(), "node count");
        std::vector<int64_t> off(n + 1, 0);
        std::vector<int32_t> col;
        std::vector<float> w;
        bool weighted = false;
        for (int64_t u = 0; u < n; ++u) {
            for (auto [v, wt] : adj[u]) {
                col.push_back(detail::to_i32(v, "node id"));
                w.push_back(static_cast<float>(wt));
                weighted = weighted || wt != 1.0;
            }
            off[u + 1] = static_cast<int64_t>(col.size());
        }
        cd_graph *h = nullptr;
        detail::check(cd_graph_from_csr(Context::instance().get(), n, off.data(), col.empty() ? nullptr : col.data(),
                                        weighted ? w.data() : nullptr, &h));
        return Graph(h);
    }

    count node_count() const { return h_ ? static_cast<count>(info().n) : 0; }
    count edge_count() const { return h_ ? static_cast<count>(info().m) : 0; }
    edgeweight total_edge_weight() const { return h_ ? info().total_weight : 0.0; }

    count degree(node u) const {
        check_node(u);
        const auto &c = host();
        return static_cast<count>(c.off[u + 1] - c.off[u]);
    }
    edgeweight volume(node u) const {
        check_node(u);
        return host().vol[u];
    }
    edgeweight loop_weight(node u) const {
        check_node(u);
        return host().loop[u];
    }

    template <typename F>
    void for_neighbors(node u, F &&f) const {
        const auto &c = host();
        for (int64_t i = c.off[u]; i < c.off[u + 1]; ++i)
            f(static_cast<node>(c.col[i]), c.w.empty() ? 1.0 : static_cast<edgeweight>(c.w[i]));
    }
    template <typename F>
    void for_nodes(F &&f) const {
        for (node u = 0; u < node_count(); ++u)
            f(u);
    }
    template <typename F>
    void for_nodes_parallel(F &&f, int = 0) const {
        for_nodes(std::forward<F>(f));
    }
    template <typename F>
    void for_edges(F &&f) const {
        const auto &c = host();
        for (node u = 0; u < node_count(); ++u)
            for (int64_t i = c.off[u]; i < c.off[u + 1]; ++i)
                if (static_cast<node>(c.col[i]) >= u)
                    f(u, static_cast<node>(c.col[i]), c.w.empty() ? 1.0 : static_cast<edgeweight>(c.w[i]));
    }

    bool operator==(const Graph &o) const {
        const auto &a = host(), &b = o.host();
        auto wa = a.w.empty() ? std::vector<float>(a.col.size(), 1.0f) : a.w;
        auto wb = b.w.empty() ? std::vector<float>(b.col.size(), 1.0f) : b.w;
        return a.off == b.off && a.col == b.col && wa == wb;
    }

    const cd_graph *handle() const { return h_.get(); }

  private:
    struct Deleter {
        void operator()(cd_graph *g) const { cd_graph_destroy(g); }
    };
    struct Host {
        std::vector<int64_t> off;
        std::vector<int32_t> col;
        std::vector<float> w;
        std::vector<double> vol, loop;
    };
    explicit Graph(cd_graph *h) : h_(h, Deleter()) {}
    friend struct CoarseningResult;
    template <class>
    friend struct GraphFactory;
    friend Graph adopt_graph(cd_graph *);

    cd_graph_info info() const {
        cd_graph_info i{};
        detail::check(cd_graph_get_info(h_.get(), &i));
        return i;
    }
    void check_node(node u) const {
        if (u >= node_count())
            throw std::out_of_range("node id " + std::to_string(u) + " out of range");
    }
    const Host &host() const {
        if (!host_) {
            auto hc = std::make_shared<Host>();
            const cd_graph_info i = h_ ? info() : cd_graph_info{};
            hc->off.assign(i.n + 1, 0);
            hc->col.resize(i.D);
            if (i.weighted)
                hc->w.resize(i.D);
            hc->vol.resize(i.n);
            hc->loop.resize(i.n);
            if (h_)
                detail::check(cd_graph_download(h_.get(), hc->off.data(), hc->col.data(),
                                                i.weighted ? hc->w.data() : nullptr, hc->vol.data(),
                                                hc->loop.data()));
            host_ = hc;
        }
        return *host_;
    }

    std::shared_ptr<cd_graph> h_;
    mutable std::shared_ptr<Host> host_;
};

inline Graph adopt_graph(cd_graph *h) { return Graph(h); }

/// Dense node -> community assignment (H/partition.hpp:13-91).
class Partition {
  public:
    Partition() = default;
    explicit Partition(count n, index initial = 0) : data_(n, initial), upper_(initial + 1) {}

    // every node its own community; the bound stays >= 1 for n = 0
    static Partition singletons(count n) {
        Partition z;
        z.data_.assign(n, 0);
        std::iota(z.data_.begin(), z.data_.end(), index{0});
        z.upper_ = std::max<index>(n, 1);
        return z;
    }

    count size() const { return data_.size(); }
    index upper_bound() const { return upper_; }
    void set_upper_bound(index ub) { upper_ = ub; }
    index operator[](node u) const { return data_[u]; }
    index &operator[](node u) { return data_[u]; }
    const std::vector<index> &data() const { return data_; }
    std::vector<index> &data() { return data_; }

    /// First-appearance compaction on the device (cd_compact).
    Partition compacted() const {
        std::vector<int32_t> z = to_device_labels(), out(z.size());
        int64_t k = 0;
        detail::check(cd_compact(Context::instance().get(), static_cast<int64_t>(z.size()), z.data(), out.data(), &k));
        Partition p = from_device_labels(out);
        p.upper_ = k > 0 ? static_cast<index>(k) : 1;
        return p;
    }
    count community_count() const {
        std::vector<int32_t> z = to_device_labels();
        int64_t k = 0;
        detail::check(cd_community_count(Context::instance().get(), static_cast<int64_t>(z.size()), z.data(), &k));
        return static_cast<count>(k);
    }
    // histogram over [0, largest id]; empty ids get 0
    std::vector<count> community_sizes() const {
        const index top = data_.empty() ? 0 : *std::max_element(data_.begin(), data_.end()) + 1;
        std::vector<count> hist(top, 0);
        for (index c : data_)
            hist[c] += 1;
        return hist;
    }
    // compact <=> the ids in use are exactly 0..k-1
    bool is_compact() const {
        const std::vector<count> h = community_sizes();
        return std::find(h.begin(), h.end(), count{0}) == h.end();
    }
    bool operator==(const Partition &o) const { return data_ == o.data_; }

    std::vector<int32_t> to_device_labels() const {
        std::vector<int32_t> z(data_.size());
        for (std::size_t u = 0; u < data_.size(); ++u)
            z[u] = detail::to_i32(data_[u], "community id");
        return z;
    }
    static Partition from_device_labels(const std::vector<int32_t> &z, index ub = 0) {
        Partition p;
        p.data_.resize(z.size());
        index mx = 0;
        for (std::size_t u = 0; u < z.size(); ++u) {
            p.data_[u] = static_cast<index>(z[u]);
            mx = std::max<index>(mx, p.data_[u] + 1);
        }
        p.upper_ = ub ? ub : std::max<index>(mx, 1);
        return p;
    }

  private:
    std::vector<index> data_;
    index upper_ = 1;
};

inline Partition singleton_partition(const Graph &g) { return Partition::singletons(g.node_count()); }

// ---- configs and report (H/plp.hpp:16-22, H/louvain.hpp:15-22, H/report.hpp) ----
struct PlpConfig {
    long long theta = -1;
    count max_iterations = 100;
    bool randomize_order = false;
    std::uint64_t seed = 1;
    int workers = 1;
};

struct LouvainConfig {
    double gamma = 1.0;
    count max_move_iterations = 32;
    count max_levels = 64;
    std::uint64_t seed = 1;
    int workers = 1;
    bool refine = false;
    // device only (not in the reference): false = the device's default early
    // stopping and pruning (cd_louvain_config_default: move_tol 1e-3,
    // move_stall 0.95, move_qtol 2e-3, prune 1); true = the reference's rule
    // alone, a move phase ends after a pass without moves or at
    // max_move_iterations (cd_louvain_config_reference)
    bool reference_stopping = false;
};

enum class Algo { plp, plm, plmr };

struct EnsembleConfig {
    count ensemble_size = 4;
    Algo base = Algo::plp;
    Algo final_algo = Algo::plmr;
    std::uint64_t seed = 1;
    int workers = 1;
    PlpConfig base_plp{.randomize_order = true};
    LouvainConfig final_louvain;
    /// Test hook (H/ensemble.hpp:30): replaces the base algorithm when set; called as f(g, seed).
    std::function<Partition(const Graph &, std::uint64_t)> base_override;
};

struct LevelTiming {
    double move_ms = 0.0;
    double coarsen_ms = 0.0;
    double refine_ms = 0.0;
};

struct IterationRecord {
    count updated = 0;
    double ms = 0.0;
};

/// Minimal JSON value (objects keep sorted keys, like nlohmann::json's
/// default std::map), enough for RunReport::to_json and the CLI reports.
class Json {
  public:
    enum class Kind { null, number, integer, string, array, object };
    Json() = default;
    Json(double v) : kind_(Kind::number), num_(v) {}  // NOLINT
    Json(long long v) : kind_(Kind::integer), int_(v) {}  // NOLINT
    Json(int v) : kind_(Kind::integer), int_(v) {}  // NOLINT
    Json(unsigned long long v) : kind_(Kind::integer), int_(static_cast<long long>(v)) {}  // NOLINT
    Json(unsigned long v) : kind_(Kind::integer), int_(static_cast<long long>(v)) {}  // NOLINT
    Json(const std::string &v) : kind_(Kind::string), str_(v) {}  // NOLINT
    Json(const char *v) : kind_(Kind::string), str_(v) {}  // NOLINT
    static Json array() {
        Json j;
        j.kind_ = Kind::array;
        return j;
    }
    static Json object() {
        Json j;
        j.kind_ = Kind::object;
        return j;
    }
    Json &operator[](const std::string &k) {
        if (kind_ == Kind::null)
            kind_ = Kind::object;
        return obj_[k];
    }
    void push_back(Json v) {
        if (kind_ == Kind::null)
            kind_ = Kind::array;
        arr_.push_back(std::move(v));
    }
    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

  private:
    static void esc(std::string &o, const std::string &s) {
        o += '"';
        for (char c : s) {
            if (c == '"' || c == '\\') {
                o += '\\';
                o += c;
            } else if (static_cast<unsigned char>(c) < 0x20) {
                char b[8];
                std::snprintf(b, sizeof(b), "\\u%04x", c);
                o += b;
            } else {
                o += c;
            }
        }
        o += '"';
    }
    void write(std::string &o, int indent, int depth) const {
        const std::string nl = indent >= 0 ? "\n" : "";
        const std::string pad = indent >= 0 ? std::string(size_t(indent) * (depth + 1), ' ') : "";
        const std::string pad0 = indent >= 0 ? std::string(size_t(indent) * depth, ' ') : "";
        switch (kind_) {
        case Kind::null:
            o += "null";
            break;
        case Kind::integer:
            o += std::to_string(int_);
            break;
        case Kind::number: {
            if (!std::isfinite(num_)) {
                o += "null";
                break;
            }
            char b[64];
            auto r = std::to_chars(b, b + sizeof(b), num_);  // shortest round trip
            std::string t(b, r.ptr);
            if (t.find_first_of(".eE") == std::string::npos)
                t += ".0";
            o += t;
            break;
        }
        case Kind::string:
            esc(o, str_);
            break;
        case Kind::array: {
            if (arr_.empty()) {
                o += "[]";
                break;
            }
            o += "[" + nl;
            for (size_t i = 0; i < arr_.size(); ++i) {
                o += pad;
                arr_[i].write(o, indent, depth + 1);
                o += (i + 1 < arr_.size() ? "," : "") + nl;
            }
            o += pad0 + "]";
            break;
        }
        case Kind::object: {
            if (obj_.empty()) {
                o += "{}";
                break;
            }
            o += "{" + nl;
            size_t i = 0;
            for (const auto &kv : obj_) {
                o += pad;
                esc(o, kv.first);
                o += indent >= 0 ? ": " : ":";
                kv.second.write(o, indent, depth + 1);
                o += (++i < obj_.size() ? "," : "") + nl;
            }
            o += pad0 + "}";
            break;
        }
        }
    }
    Kind kind_ = Kind::null;
    double num_ = 0.0;
    long long int_ = 0;
    std::string str_;
    std::vector<Json> arr_;
    std::map<std::string, Json> obj_;
};

struct RunReport {
    std::string algorithm;
    std::string input;
    int workers = 1;
    std::uint64_t seed = 0;
    double total_ms = 0.0;
    double modularity = 0.0;
    double coverage = 0.0;
    count community_count = 0;
    std::vector<LevelTiming> levels;
    std::vector<IterationRecord> iterations;
    double base_ms = 0.0;
    double combine_ms = 0.0;
    double coarsen_ms = 0.0;
    double final_ms = 0.0;

    /// RunReport::to_json (H/report.hpp:42-70): same fields and nesting.
    Json to_json() const {
        Json j = Json::object();
        j["algorithm"] = algorithm;
        j["input"] = input;
        j["workers"] = workers;
        j["seed"] = static_cast<unsigned long long>(seed);
        j["total_ms"] = total_ms;
        j["modularity"] = modularity;
        j["coverage"] = coverage;
        j["communities"] = static_cast<unsigned long long>(community_count);
        if (!levels.empty()) {
            Json arr = Json::array();
            for (const auto &l : levels) {
                Json e = Json::object();
                e["move_ms"] = l.move_ms;
                e["coarsen_ms"] = l.coarsen_ms;
                e["refine_ms"] = l.refine_ms;
                arr.push_back(e);
            }
            j["levels"] = arr;
        }
        if (!iterations.empty()) {
            Json arr = Json::array();
            for (const auto &it : iterations) {
                Json e = Json::object();
                e["updated"] = static_cast<unsigned long long>(it.updated);
                e["ms"] = it.ms;
                arr.push_back(e);
            }
            j["iterations"] = arr;
        }
        if (algorithm == "epp") {
            Json ph = Json::object();
            ph["base_ms"] = base_ms;
            ph["combine_ms"] = combine_ms;
            ph["coarsen_ms"] = coarsen_ms;
            ph["final_ms"] = final_ms;
            j["phases"] = ph;
        }
        return j;
    }
};

namespace detail {
// the reference's caps are uint64 counts; the C ABI takes int64: saturate
inline int64_t sat64(count c) {
    return c > static_cast<count>(INT64_MAX) ? INT64_MAX : static_cast<int64_t>(c);
}
inline cd_plp_config plp_c(const PlpConfig &c) {
    cd_plp_config o;
    cd_plp_config_default(&o);
    o.theta = c.theta;
    o.max_iterations = sat64(c.max_iterations);
    o.randomize_order = c.randomize_order ? 1 : 0;
    o.seed = c.seed;
    o.workers = c.workers;
    return o;
}
inline cd_louvain_config louvain_c(const LouvainConfig &c) {
    cd_louvain_config o;
    if (c.reference_stopping)
        cd_louvain_config_reference(&o);
    else
        cd_louvain_config_default(&o);
    o.gamma = c.gamma;
    o.max_move_iterations = sat64(c.max_move_iterations);
    o.max_levels = sat64(c.max_levels);
    o.seed = c.seed;
    o.workers = c.workers;
    o.refine = c.refine ? 1 : 0;
    return o;
}
inline int algo_c(Algo a) { return a == Algo::plp ? CD_ALGO_PLP : (a == Algo::plm ? CD_ALGO_PLM : CD_ALGO_PLMR); }
inline RunReport report_of(const cd_report &r) {
    RunReport o;
    o.algorithm = r.algorithm;
    o.workers = r.workers;
    o.seed = r.seed;
    o.total_ms = r.total_ms;
    o.modularity = r.modularity;
    o.coverage = r.coverage;
    o.community_count = static_cast<count>(r.community_count);
    for (int64_t i = 0; i < std::min<int64_t>(r.n_levels, CD_MAX_LEVEL_RECORDS); ++i)
        o.levels.push_back({r.levels[i].move_ms, r.levels[i].coarsen_ms, r.levels[i].refine_ms});
    for (int64_t i = 0; i < std::min<int64_t>(r.n_iterations, CD_MAX_ITERATION_RECORDS); ++i)
        o.iterations.push_back({static_cast<count>(r.iterations[i].updated), r.iterations[i].ms});
    o.base_ms = r.base_ms;
    o.combine_ms = r.combine_ms;
    o.coarsen_ms = r.coarsen_ms;
    o.final_ms = r.final_ms;
    return o;
}
inline void check_cover(const Graph &g, const Partition &z) {
    if (z.size() != g.node_count())
        throw std::invalid_argument("partition length " + std::to_string(z.size()) + " does not match node count " +
                                    std::to_string(g.node_count()));
}
}  // namespace detail

// ---- quality (H/quality.hpp) ------------------------------------------------------
inline double coverage(const Graph &g, const Partition &z) {
    detail::check_cover(g, z);
    if (g.total_edge_weight() == 0.0)
        return 0.0;
    auto l = z.to_device_labels();
    double q = 0.0, c = 0.0;
    detail::check(cd_modularity(Context::instance().get(), g.handle(), l.data(),
                                static_cast<int64_t>(std::max<index>(z.upper_bound(), 1)), 1.0, &q, &c));
    return c;
}

/// Dense int32 relabelling that preserves label equality (ids may exceed int32).
inline std::vector<int32_t> dense_labels(const Partition &z) {
    std::unordered_map<index, int32_t> m;
    std::vector<int32_t> out(z.size());
    for (std::size_t u = 0; u < z.size(); ++u) {
        auto it = m.find(z[u]);
        if (it == m.end())
            it = m.emplace(z[u], static_cast<int32_t>(m.size())).first;
        out[u] = it->second;
    }
    return out;
}

/// graph_rand_index (H/quality.hpp:56-69), on the device.
inline double graph_rand_index(const Graph &g, const Partition &a, const Partition &b) {
    detail::check_cover(g, a);
    detail::check_cover(g, b);
    const auto la = dense_labels(a), lb = dense_labels(b);
    double r = 0.0;
    detail::check(cd_rand_index(Context::instance().get(), g.handle(), la.empty() ? nullptr : la.data(),
                                lb.empty() ? nullptr : lb.data(), &r));
    return r;
}

inline double modularity(const Graph &g, const Partition &z, double gamma = 1.0) {
    detail::check_cover(g, z);
    auto l = z.to_device_labels();
    double q = 0.0, c = 0.0;
    detail::check(cd_modularity(Context::instance().get(), g.handle(), l.data(),
                                static_cast<int64_t>(std::max<index>(z.upper_bound(), 1)), gamma, &q, &c));
    return q;
}

struct QualityReport {
    double modularity = 0.0;
    double coverage = 0.0;
    count community_count = 0;
    std::map<count, count> size_histogram;  // community size -> number of communities

    /// QualityReport::to_text (H/quality.hpp:78-88).
    std::string to_text() const {
        char b[64];
        std::string os;
        std::snprintf(b, sizeof(b), "%.15g", modularity);
        os += std::string("modularity ") + b + "\n";
        std::snprintf(b, sizeof(b), "%.15g", coverage);
        os += std::string("coverage ") + b + "\n";
        os += "communities " + std::to_string(community_count) + "\n";
        for (auto [size, n] : size_histogram)
            os += "size_" + std::to_string(size) + " " + std::to_string(n) + "\n";
        return os;
    }
};

/// evaluate (H/quality.hpp:91-102).
inline QualityReport evaluate(const Graph &g, const Partition &z, double gamma = 1.0) {
    QualityReport r;
    r.coverage = coverage(g, z);
    r.modularity = g.total_edge_weight() > 0 ? modularity(g, z, gamma) : 0.0;
    const Partition zc = z.compacted();
    const auto sizes = zc.community_sizes();
    r.community_count = sizes.size();
    for (count sz : sizes)
        ++r.size_histogram[sz];
    return r;
}

// ---- PLP (H/plp.hpp) ------------------------------------------------------------------
inline count resolved_theta(const PlpConfig &cfg, count n) {
    if (cfg.theta >= 0)
        return static_cast<count>(cfg.theta);
    return std::max<count>(1, n / 100000);
}

inline std::pair<Partition, RunReport> run_plp(const Graph &g, const PlpConfig &cfg,
                                               const std::optional<Partition> &initial = std::nullopt) {
    if (initial && initial->size() != g.node_count())
        throw std::invalid_argument("initial partition does not cover the graph");
    std::vector<int32_t> init = initial ? initial->to_device_labels() : std::vector<int32_t>();
    std::vector<int32_t> labels(g.node_count());
    cd_plp_config c = detail::plp_c(cfg);
    auto rep = std::make_unique<cd_report>();
    detail::check(cd_plp_run(Context::instance().get(), g.handle(), &c, initial ? init.data() : nullptr,
                             labels.data(), rep.get()));
    return {Partition::from_device_labels(labels), detail::report_of(*rep)};
}

inline index dominant_label(const Graph &g, const Partition &z, node u) {
    if (g.degree(u) == 0)
        throw std::invalid_argument("dominant_label: node " + std::to_string(u) + " is isolated");
    auto l = z.to_device_labels();
    std::vector<int32_t> out(l.size());
    int64_t upd = 0;
    detail::check(cd_plp_sweep_sync(Context::instance().get(), g.handle(), l.data(), out.data(), &upd));
    return static_cast<index>(out[u]);
}

inline bool is_stable(const Graph &g, const Partition &z) {
    auto l = z.to_device_labels();
    std::vector<int32_t> out(l.size());
    int64_t upd = 0;
    detail::check(cd_plp_sweep_sync(Context::instance().get(), g.handle(), l.data(), out.data(), &upd));
    return upd == 0;
}

// ---- Louvain (H/louvain.hpp) --------------------------------------------------------
using CommunityVolumes = std::vector<edgeweight>;

inline CommunityVolumes community_volumes(const Graph &g, const Partition &z) {
    auto l = z.to_device_labels();
    CommunityVolumes vols(std::max<index>(z.upper_bound(), 1));
    detail::check(cd_community_volumes(Context::instance().get(), g.handle(), l.data(),
                                       static_cast<int64_t>(vols.size()), vols.data()));
    return vols;
}

/// H/louvain.hpp:37-56 (scalar; evaluated on the host mirror of the graph).
inline double delta_mod(const Graph &g, const Partition &z, const CommunityVolumes &vols, node u, index target,
                        double gamma) {
    const index c = z[u];
    if (target == c)
        return 0.0;
    edgeweight w_c = 0.0, w_d = 0.0;
    g.for_neighbors(u, [&](node v, edgeweight w) {
        if (v == u)
            return;
        if (z[v] == c)
            w_c += w;
        else if (z[v] == target)
            w_d += w;
    });
    const edgeweight total = g.total_edge_weight();
    const edgeweight vol_u = g.volume(u);
    return (w_d - w_c) / total + gamma * ((vols[c] - vol_u) - vols[target]) * vol_u / (2.0 * total * total);
}

/// Called after each applied move: (node, source, target, predicted gain) (H/louvain.hpp:58-60).
using MoveObserver = std::function<void(node, index, index, double)>;

namespace detail {
struct ObserverCall {
    Partition *z;
    const MoveObserver *observer;
    std::exception_ptr error;
};
inline void observer_trampoline(void *user, int32_t u, int32_t c, int32_t d, double gain) {
    auto *oc = static_cast<ObserverCall *>(user);
    if (oc->error)
        return;
    try {
        (*oc->z)[static_cast<node>(u)] = static_cast<index>(d);  // the partition after this move
        (*oc->observer)(static_cast<node>(u), static_cast<index>(c), static_cast<index>(d), gain);
    } catch (...) {
        oc->error = std::current_exception();
    }
}
}  // namespace detail

/// move_phase (H/louvain.hpp:65-141) with the device's bucketed order, or,
/// given an observer, in the reference's one-worker order with every move
/// reported as it is applied to z.
inline bool move_phase(const Graph &g, Partition &z, const LouvainConfig &cfg, const MoveObserver &observer = {}) {
    detail::check_cover(g, z);
    if (observer) {
        auto l = z.to_device_labels();
        cd_louvain_config c = detail::louvain_c(cfg);
        const index ub = z.upper_bound();
        detail::ObserverCall oc{&z, &observer, nullptr};
        int32_t changed = 0;
        detail::check(cd_move_phase_sequential(Context::instance().get(), g.handle(), l.data(),
                                               static_cast<int64_t>(std::max<index>(ub, 1)), &c,
                                               &detail::observer_trampoline, &oc, &changed));
        if (oc.error)
            std::rethrow_exception(oc.error);
        z = Partition::from_device_labels(l, ub);
        return changed != 0;
    }
    auto l = z.to_device_labels();
    cd_louvain_config c = detail::louvain_c(cfg);
    int32_t changed = 0;
    detail::check(cd_move_phase(Context::instance().get(), g.handle(), l.data(), &c, &changed));
    const index ub = z.upper_bound();
    z = Partition::from_device_labels(l, ub);
    return changed != 0;
}

struct CoarseningResult {
    Graph coarse;
    std::vector<node> pi;
};

inline CoarseningResult coarsen(const Graph &g, const Partition &z, int = 1) {
    detail::check_cover(g, z);
    auto l = z.to_device_labels();
    std::vector<int32_t> pi(l.size());
    cd_graph *h = nullptr;
    detail::check(cd_coarsen(Context::instance().get(), g.handle(), l.data(), &h, pi.data()));
    CoarseningResult r{adopt_graph(h), {}};
    r.pi.assign(pi.begin(), pi.end());
    return r;
}

inline Partition prolong(const Partition &z_coarse, const std::vector<node> &pi) {
    auto zc = z_coarse.to_device_labels();
    std::vector<int32_t> p(pi.size()), out(pi.size());
    for (std::size_t v = 0; v < pi.size(); ++v) {
        if (pi[v] >= z_coarse.size())
            throw std::out_of_range("prolong: contraction map entry out of range");
        p[v] = static_cast<int32_t>(pi[v]);
    }
    detail::check(cd_prolong(Context::instance().get(), static_cast<int64_t>(zc.size()), zc.data(),
                             static_cast<int64_t>(p.size()), p.data(), out.data()));
    return Partition::from_device_labels(out, z_coarse.upper_bound());
}

inline std::pair<Partition, RunReport> run_plm(const Graph &g, const LouvainConfig &cfg) {
    cd_louvain_config c = detail::louvain_c(cfg);
    c.refine = 0;
    std::vector<int32_t> z(g.node_count());
    auto rep = std::make_unique<cd_report>();
    detail::check(cd_louvain_run(Context::instance().get(), g.handle(), &c, z.data(), rep.get()));
    return {Partition::from_device_labels(z), detail::report_of(*rep)};
}

inline std::pair<Partition, RunReport> run_plmr(const Graph &g, const LouvainConfig &cfg) {
    cd_louvain_config c = detail::louvain_c(cfg);
    c.refine = 1;
    std::vector<int32_t> z(g.node_count());
    auto rep = std::make_unique<cd_report>();
    detail::check(cd_louvain_run(Context::instance().get(), g.handle(), &c, z.data(), rep.get()));
    return {Partition::from_device_labels(z), detail::report_of(*rep)};
}

// ---- ensemble (H/ensemble.hpp) ------------------------------------------------------
inline std::uint64_t djb2(const std::uint8_t *data, std::size_t len) {
    std::uint64_t h = 5381;
    for (std::size_t i = 0; i < len; ++i)
        h = h * 33 + data[i];
    return h;
}

inline Partition combine_hashed(const std::vector<Partition> &solutions, int = 1) {
    if (solutions.empty())
        throw std::invalid_argument("empty ensemble");
    std::vector<std::vector<int32_t>> l;
    std::vector<const int32_t *> p;
    for (const Partition &s : solutions) {
        if (s.size() != solutions.front().size())
            throw std::invalid_argument("ensemble partitions cover different node sets");
        l.push_back(s.to_device_labels());
    }
    for (auto &v : l)
        p.push_back(v.data());
    std::vector<int32_t> out(solutions.front().size());
    int64_t k = 0;
    detail::check(cd_combine_hashed(Context::instance().get(), static_cast<int64_t>(p.size()),
                                    static_cast<int64_t>(out.size()), p.data(), out.data(), &k));
    return Partition::from_device_labels(out, k > 0 ? static_cast<index>(k) : 1);
}

inline std::pair<Partition, RunReport> run_epp(const Graph &g, const EnsembleConfig &cfg) {
    cd_ensemble_config c;
    cd_ensemble_config_default(&c);
    c.ensemble_size = static_cast<int64_t>(cfg.ensemble_size);
    c.base = detail::algo_c(cfg.base);
    c.final_algo = detail::algo_c(cfg.final_algo);
    c.seed = cfg.seed;
    c.workers = cfg.workers;
    c.base_plp = detail::plp_c(cfg.base_plp);
    c.final_louvain = detail::louvain_c(cfg.final_louvain);
    std::vector<int32_t> z(g.node_count());
    auto rep = std::make_unique<cd_report>();
    if (!cfg.base_override) {
        detail::check(cd_epp_run(Context::instance().get(), g.handle(), &c, z.data(), rep.get()));
        return {Partition::from_device_labels(z), detail::report_of(*rep)};
    }
    // base_override (H/ensemble.hpp:127-128): the hook's partitions replace the base runs
    if (cfg.ensemble_size < 1)
        throw std::invalid_argument("ensemble size must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::vector<int32_t>> bases;
    for (count i = 0; i < cfg.ensemble_size; ++i) {
        Partition p = cfg.base_override(g, cfg.seed + static_cast<std::uint64_t>(i));
        if (!bases.empty() && p.size() != bases.front().size())
            throw std::invalid_argument("ensemble partitions cover different node sets");  // :33-39
        detail::check_cover(g, p);
        bases.push_back(p.to_device_labels());
    }
    const double base_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::vector<const int32_t *> ptrs;
    for (auto &b : bases)
        ptrs.push_back(b.data());
    detail::check(cd_epp_run_bases(Context::instance().get(), g.handle(), &c, ptrs.data(), z.data(), rep.get()));
    RunReport r = detail::report_of(*rep);
    r.base_ms = base_ms;
    r.total_ms += base_ms;
    return {Partition::from_device_labels(z), std::move(r)};
}

// ---- generator (H/generator.hpp) ------------------------------------------------------
struct PlantedPartitionSpec {
    count n = 0;
    count k = 1;
    double p_in = 0.0;
    double p_out = 0.0;
    std::uint64_t seed = 1;
};

inline index planted_block(node u, count n, count k) {
    return static_cast<index>((static_cast<unsigned __int128>(u) * k) / n);
}

inline std::pair<Graph, Partition> generate_planted(const PlantedPartitionSpec &spec, int = 1) {
    std::vector<int32_t> truth(spec.n);
    cd_graph *h = nullptr;
    detail::check(cd_graph_generate_planted(Context::instance().get(), static_cast<int64_t>(spec.n),
                                            static_cast<int64_t>(spec.k), spec.p_in, spec.p_out, spec.seed, &h,
                                            truth.empty() ? nullptr : truth.data()));
    Partition t = Partition::from_device_labels(truth, spec.n > 0 ? spec.k : 1);
    return {adopt_graph(h), t};
}

// ---- text readers (H/io.hpp) -- parsed on the device ------------------------------------
namespace io {

/// io::read_metis (H/io.hpp:83-165).
inline Graph read_metis(const std::string &path) {
    cd_graph *h = nullptr;
    detail::check(cd_graph_load_metis(Context::instance().get(), path.c_str(), &h));
    return adopt_graph(h);
}

/// io::read_edge_list (H/io.hpp:190-237).
inline Graph read_edge_list(const std::string &path, bool merge_duplicates = false,
                            std::vector<std::uint64_t> *original_ids = nullptr) {
    cd_graph *h = nullptr;
    detail::check(cd_graph_load_edge_list(Context::instance().get(), path.c_str(), merge_duplicates ? 1 : 0, &h));
    Graph g = adopt_graph(h);
    if (original_ids) {
        original_ids->resize(g.node_count());
        detail::check(cd_graph_original_ids(h, original_ids->empty() ? nullptr : original_ids->data()));
    }
    return g;
}

namespace detail {
inline std::string format_weight(double w) {  // io::detail::format_weight (H/io.hpp:70-77)
    char buf[32];
    if (w == std::floor(w) && std::abs(w) < 1e15)
        std::snprintf(buf, sizeof(buf), "%.0f", w);
    else
        std::snprintf(buf, sizeof(buf), "%.17g", w);
    return buf;
}
inline std::ofstream open_output(const std::string &path) {
    std::ofstream out(path);
    if (!out)
        throw input_error("cannot open " + path + " for writing");
    return out;
}
// runs `emit` on the opened file, then checks the stream once
template <class F>
inline void write_text(const std::string &path, F &&emit) {
    std::ofstream out = open_output(path);
    emit(out);
    out.flush();
    if (!out)
        throw input_error("write failed: " + path);
}
}  // namespace detail

/// io::write_metis (H/io.hpp:168-183): fmt 1, 1-based neighbours with weights.
inline void write_metis(const Graph &g, const std::string &path) {
    detail::write_text(path, [&](std::ostream &out) {
        out << g.node_count() << ' ' << g.edge_count() << " 1\n";
        std::string row;
        for (node u = 0; u < g.node_count(); ++u) {
            row.clear();
            g.for_neighbors(u, [&](node v, edgeweight w) {
                row += row.empty() ? "" : " ";
                row += std::to_string(v + 1);
                row += ' ';
                row += detail::format_weight(w);
            });
            out << row << '\n';
        }
    });
}

/// io::write_edge_list (H/io.hpp:239-245): "u v w", one line per undirected edge.
inline void write_edge_list(const Graph &g, const std::string &path) {
    detail::write_text(path, [&](std::ostream &out) {
        for (node u = 0; u < g.node_count(); ++u)
            g.for_neighbors(u, [&](node v, edgeweight w) {
                if (v < u)
                    return;  // each undirected edge once, from its smaller endpoint
                out << u << ' ' << v << ' ' << detail::format_weight(w) << '\n';
            });
    });
}

/// io::write_partition (H/io.hpp:248-255).
inline void write_partition(const Partition &z, const std::string &path) {
    detail::write_text(path, [&](std::ostream &out) {
        for (index c : z.data())
            out << c << '\n';
    });
}

/// io::read_partition (H/io.hpp:257-275).
inline Partition read_partition(const std::string &path) {
    std::ifstream in(path);
    if (!in)
        throw input_error("cannot open " + path);
    Partition z;
    std::string line;
    std::size_t lineno = 0;
    index ub = 0;
    while (std::getline(in, line)) {
        ++lineno;
        std::vector<std::string> toks;
        std::size_t i = 0;
        while (i < line.size()) {
            while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i])))
                ++i;
            std::size_t j = i;
            while (j < line.size() && !std::isspace(static_cast<unsigned char>(line[j])))
                ++j;
            if (j > i)
                toks.push_back(line.substr(i, j - i));
            i = j;
        }
        if (toks.empty())
            continue;
        const std::string ctx = path + ":" + std::to_string(lineno);
        if (toks.size() != 1)
            throw input_error(ctx + ": expected one community id per line");
        std::uint64_t c = 0;
        auto [p, ec] = std::from_chars(toks[0].data(), toks[0].data() + toks[0].size(), c);
        if (ec != std::errc{} || p != toks[0].data() + toks[0].size())
            throw input_error("malformed integer '" + toks[0] + "' in " + ctx);
        z.data().push_back(c);
        ub = std::max<index>(ub, c + 1);
    }
    z.set_upper_bound(ub > 0 ? ub : 1);
    return z;
}

/// io::write_community_graph (H/io.hpp:279-289): the contraction (on the
/// device) in METIS format, plus "<path>.sizes" with "community_id size" lines.
inline void write_community_graph(const Graph &g, const Partition &z, const std::string &path) {
    const Partition zc = z.is_compact() ? z : z.compacted();
    write_metis(coarsen(g, zc).coarse, path);
    const std::vector<count> sizes = zc.community_sizes();
    detail::write_text(path + ".sizes", [&](std::ostream &out) {
        index c = 0;
        for (count s : sizes)
            out << c++ << ' ' << s << '\n';
    });
}

}  // namespace io

}  // namespace gpu

#ifdef COMMDET_GPU_DROP_IN
using namespace gpu;
#endif

}  // namespace commdet
