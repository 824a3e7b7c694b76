// commdet_gpu -- command-line front end of the B200 library with the
// reference CLI's contract (P/tools/commdet.cpp: subcommands, flag names,
// printed keys, report JSON fields, exit codes).
// Every computation goes through the drop-in C++ shim (include/commdet/gpu.hpp)
// and therefore through the C ABI onto the device.
//
//   detect    --input F [--algo plp|plm|plmr|epp] [--format metis|edges]
//             [--merge-duplicates] [--shuffle] [--threads N] [--theta T]
//             [--gamma G] [--ensemble B] [--seed S] [--runs R] [--output P]
//             [--report J] [--community-graph C]
//   score     --input F --partition P [--reference Q] [--format] [--gamma G]
//   generate  --n N --k K --pin P --pout Q --output F [--seed S] [--threads N]
//             [--ground-truth T]
//   bench     [--mode strong|weak] [--algo A] (--input F | --gen-n N [--gen-k
//             K --gen-pin P --gen-pout Q]) [--threads-list 1,2,..] [--seed S]
//             [--theta T] [--gamma G] [--ensemble B] [--data TSV]
//
// Worker counts are accepted and reported like the reference's OpenMP worker
// count; the device ignores them (one GPU per context).  Exit status: 0 ok,
// 2 bad usage or bad input, 3 anything else.
#define COMMDET_GPU_DROP_IN
#include <commdet/gpu.hpp>

#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace {

using namespace commdet;

enum Exit { kOk = 0, kBadInput = 2, kInternal = 3 };

struct BadUsage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// option tables: one row per accepted flag of a subcommand
// ---------------------------------------------------------------------------
struct FlagSpec {
    const char *name;
    bool takes_value;
};

const std::map<std::string, std::vector<FlagSpec>> &command_table() {
    static const std::map<std::string, std::vector<FlagSpec>> t = {
        {"detect",
         {{"algo", true}, {"input", true}, {"format", true}, {"merge-duplicates", false}, {"shuffle", false},
          {"threads", true}, {"theta", true}, {"gamma", true}, {"ensemble", true}, {"seed", true}, {"runs", true},
          {"output", true}, {"report", true}, {"community-graph", true}}},
        {"score", {{"input", true}, {"format", true}, {"partition", true}, {"reference", true}, {"gamma", true}}},
        {"generate",
         {{"n", true}, {"k", true}, {"pin", true}, {"pout", true}, {"seed", true}, {"threads", true},
          {"output", true}, {"ground-truth", true}}},
        {"bench",
         {{"mode", true}, {"algo", true}, {"input", true}, {"format", true}, {"gen-n", true}, {"gen-k", true},
          {"gen-pin", true}, {"gen-pout", true}, {"threads-list", true}, {"seed", true}, {"theta", true},
          {"gamma", true}, {"ensemble", true}, {"data", true}}},
    };
    return t;
}

// Parsed flags of one subcommand; typed getters validate on access.
class Options {
  public:
    Options(const std::vector<FlagSpec> &spec, const std::vector<std::string> &words) {
        std::map<std::string, bool> known;
        for (const FlagSpec &f : spec)
            known[f.name] = f.takes_value;
        for (std::size_t i = 0; i < words.size(); ++i) {
            const std::string &w = words[i];
            if (w.size() < 3 || w[0] != '-' || w[1] != '-')
                throw BadUsage("unexpected argument '" + w + "'");
            std::string key = w.substr(2);
            std::string value;
            const std::size_t eq = key.find('=');
            const bool inline_value = eq != std::string::npos;
            if (inline_value) {
                value = key.substr(eq + 1);
                key.resize(eq);
            }
            auto k = known.find(key);
            if (k == known.end())
                throw BadUsage("unknown option --" + key);
            if (!k->second) {
                if (inline_value)
                    throw BadUsage("flag --" + key + " takes no value");
                value = "1";
            } else if (!inline_value) {
                if (i + 1 == words.size())
                    throw BadUsage("--" + key + " requires a value");
                value = words[++i];
            }
            given_[key] = value;
        }
    }

    bool given(const std::string &key) const { return given_.find(key) != given_.end(); }
    std::string text(const std::string &key, const std::string &fallback = "") const {
        auto it = given_.find(key);
        return it == given_.end() ? fallback : it->second;
    }
    std::string required(const std::string &key) const {
        if (!given(key))
            throw BadUsage("--" + key + " is required");
        return text(key);
    }
    template <class T>
    T number(const std::string &key, T fallback) const {
        return given(key) ? convert<T>(key, text(key)) : fallback;
    }
    template <class T>
    T required_number(const std::string &key) const {
        return convert<T>(key, required(key));
    }

    // whole-token numeric conversion; unsigned values reject a sign
    template <class T>
    static T convert(const std::string &key, const std::string &s) {
        std::istringstream in(s);
        T v{};
        bool ok = !s.empty() && !(std::is_unsigned_v<T> && s[0] == '-');
        if (ok) {
            if constexpr (std::is_same_v<T, std::uint64_t>) {
                unsigned long long u = 0;
                ok = static_cast<bool>(in >> u);
                v = static_cast<T>(u);
            } else {
                ok = static_cast<bool>(in >> v);
            }
            ok = ok && in.peek() == std::char_traits<char>::eof();
        }
        if (!ok)
            throw BadUsage("--" + key + ": invalid value '" + s + "'");
        return v;
    }

  private:
    std::map<std::string, std::string> given_;
};

// ---------------------------------------------------------------------------
// detector registry: algorithm name -> one run on the device
// ---------------------------------------------------------------------------
struct RunSettings {
    int workers = 1;
    long long theta = -1;
    bool shuffle = false;
    double gamma = 1.0;
    count ensemble = 4;
};

using Detector = std::function<std::pair<Partition, RunReport>(const Graph &, const RunSettings &, std::uint64_t)>;

const Detector &detector(const std::string &algo) {
    static const std::map<std::string, Detector> registry = {
        {"plp",
         [](const Graph &g, const RunSettings &s, std::uint64_t seed) {
             PlpConfig c;
             c.theta = s.theta;
             c.randomize_order = s.shuffle;
             c.seed = seed;
             c.workers = s.workers;
             return run_plp(g, c);
         }},
        {"plm",
         [](const Graph &g, const RunSettings &s, std::uint64_t seed) {
             LouvainConfig c;
             c.gamma = s.gamma;
             c.seed = seed;
             c.workers = s.workers;
             return run_plm(g, c);
         }},
        {"plmr",
         [](const Graph &g, const RunSettings &s, std::uint64_t seed) {
             LouvainConfig c;
             c.gamma = s.gamma;
             c.seed = seed;
             c.workers = s.workers;
             return run_plmr(g, c);
         }},
        {"epp",
         [](const Graph &g, const RunSettings &s, std::uint64_t seed) {
             EnsembleConfig c;
             c.ensemble_size = s.ensemble;
             c.seed = seed;
             c.workers = s.workers;
             c.base_plp.theta = s.theta;
             c.final_louvain.gamma = s.gamma;
             return run_epp(g, c);
         }},
    };
    auto it = registry.find(algo);
    if (it == registry.end())
        throw input_error("unknown algorithm '" + algo + "'");
    return it->second;
}

Graph read_graph(const std::string &path, const std::string &format, bool merge) {
    if (format == "edges")
        return io::read_edge_list(path, merge);
    if (format != "metis")
        throw input_error("unknown graph format '" + format + "'");
    return io::read_metis(path);
}

RunSettings settings_from(const Options &o) {
    RunSettings s;
    s.workers = o.number<int>("threads", 1);
    s.theta = o.number<long long>("theta", -1);
    s.shuffle = o.given("shuffle");
    s.gamma = o.number<double>("gamma", 1.0);
    s.ensemble = o.number<count>("ensemble", 4);
    return s;
}

void print_pairs(const std::vector<std::pair<std::string, std::string>> &rows) {
    for (const auto &[k, v] : rows)
        std::cout << k << " " << v << "\n";
}

template <class T>
std::string fmt(const T &v) {
    std::ostringstream s;
    s.precision(15);
    s << v;
    return s.str();
}

std::ofstream open_for_writing(const std::string &path) {
    std::ofstream f(path);
    if (!f)
        throw input_error("cannot open " + path + " for writing");
    return f;
}

// ---------------------------------------------------------------------------
// subcommands
// ---------------------------------------------------------------------------
int detect(const Options &o) {
    const std::string algo = o.text("algo", "plm");
    const std::string input = o.required("input");
    const unsigned runs = o.number<unsigned>("runs", 1);
    if (runs == 0)
        throw BadUsage("--runs: value must be positive");
    const std::uint64_t seed0 = o.number<std::uint64_t>("seed", 1);
    const RunSettings s = settings_from(o);
    const Graph g = read_graph(input, o.text("format", "metis"), o.given("merge-duplicates"));
    const Detector &run = detector(algo);

    // reports in run order; the best partition (highest modularity, the
    // earliest run on ties) is kept compacted
    std::vector<RunReport> reps;
    Partition best;
    double best_q = -2.0;
    for (unsigned i = 0; i < runs; ++i) {
        auto [z, r] = run(g, s, seed0 + i);
        r.input = input;
        if (r.modularity > best_q) {
            best_q = r.modularity;
            best = z.compacted();
        }
        reps.push_back(std::move(r));
    }
    double sum_ms = 0.0, sum_q = 0.0, sum_cov = 0.0;
    for (const RunReport &r : reps) {
        sum_ms += r.total_ms;
        sum_q += r.modularity;
        sum_cov += r.coverage;
    }
    const double k = static_cast<double>(reps.size());
    print_pairs({{"algorithm", algo},
                 {"runs", fmt(runs)},
                 {"threads", fmt(s.workers)},
                 {"avg_time_ms", fmt(sum_ms / k)},
                 {"avg_modularity", fmt(sum_q / k)},
                 {"avg_coverage", fmt(sum_cov / k)},
                 {"best_modularity", fmt(best_q)},
                 {"communities", fmt(best.upper_bound())}});
    if (o.given("output"))
        io::write_partition(best, o.text("output"));
    if (o.given("community-graph"))
        io::write_community_graph(g, best, o.text("community-graph"));
    if (o.given("report")) {
        Json doc = Json::object();
        Json mean = Json::object();
        mean["time_ms"] = sum_ms / k;
        mean["modularity"] = sum_q / k;
        mean["coverage"] = sum_cov / k;
        doc["average"] = mean;
        doc["best_modularity"] = best_q;
        Json list = Json::array();
        for (const RunReport &r : reps)
            list.push_back(r.to_json());
        doc["runs"] = list;
        open_for_writing(o.text("report")) << doc.dump(2) << "\n";
    }
    return kOk;
}

int score(const Options &o) {
    const Graph g = read_graph(o.required("input"), o.text("format", "metis"), false);
    auto load_cover = [&](const std::string &path, const char *what) {
        Partition p = io::read_partition(path);
        if (p.size() != g.node_count())
            throw input_error(std::string(what) + " length " + std::to_string(p.size()) +
                              " does not match node count " + std::to_string(g.node_count()));
        return p;
    };
    const Partition z = load_cover(o.required("partition"), "partition");
    const QualityReport q = evaluate(g, z, o.number<double>("gamma", 1.0));
    std::vector<std::pair<std::string, std::string>> rows = {
        {"modularity", fmt(q.modularity)}, {"coverage", fmt(q.coverage)}, {"communities", fmt(q.community_count)}};
    if (o.given("reference"))
        rows.emplace_back("rand_index", fmt(graph_rand_index(g, z, load_cover(o.text("reference"), "reference"))));
    print_pairs(rows);
    return kOk;
}

PlantedPartitionSpec planted_spec(const Options &o, const std::string &prefix, bool all_required) {
    auto take = [&](const char *field, const char *fallback) {
        const std::string key = prefix + field;
        return all_required ? o.required(key) : o.text(key, fallback);
    };
    PlantedPartitionSpec s;
    s.n = Options::convert<count>(prefix + "n", take("n", ""));
    s.k = Options::convert<count>(prefix + "k", take("k", "1"));
    s.p_in = Options::convert<double>(prefix + "pin", take("pin", "0"));
    s.p_out = Options::convert<double>(prefix + "pout", take("pout", "0"));
    return s;
}

int generate(const Options &o) {
    PlantedPartitionSpec spec = planted_spec(o, "", true);
    spec.seed = o.number<std::uint64_t>("seed", 1);
    const std::string out = o.required("output");
    auto made = generate_planted(spec, o.number<int>("threads", 1));
    io::write_metis(made.first, out);
    if (o.given("ground-truth"))
        io::write_partition(made.second.compacted(), o.text("ground-truth"));
    print_pairs({{"nodes", fmt(made.first.node_count())},
                 {"edges", fmt(made.first.edge_count())},
                 {"blocks", fmt(spec.k)}});
    return kOk;
}

std::vector<int> worker_counts(const std::string &csv) {
    std::vector<int> out;
    std::stringstream in(csv);
    std::string item;
    while (std::getline(in, item, ','))
        out.push_back(Options::convert<int>("threads-list", item));
    if (csv.empty() || csv.back() == ',')
        out.push_back(Options::convert<int>("threads-list", ""));
    return out;
}

int bench(const Options &o) {
    const std::string mode = o.text("mode", "strong");
    const bool synthetic = o.given("gen-n");
    if (mode != "strong" && mode != "weak")
        throw input_error("unknown bench mode '" + mode + "'");
    if (mode == "weak" && !synthetic)
        throw input_error("weak scaling requires a generator spec (--gen-n ...)");
    if (!synthetic && !o.given("input"))
        throw input_error("bench needs --input or --gen-n");
    const std::vector<int> counts = worker_counts(o.text("threads-list", "1"));
    PlantedPartitionSpec base = synthetic ? planted_spec(o, "gen-", false) : PlantedPartitionSpec{};
    RunSettings s = settings_from(o);
    const Detector &run = detector(o.text("algo", "plm"));
    const std::uint64_t seed = o.number<std::uint64_t>("seed", 1);

    // strong: one graph for every worker count; weak: n grows with the count
    Graph shared;
    if (mode == "strong")
        shared = synthetic ? generate_planted(base, counts.back()).first
                           : read_graph(o.text("input"), o.text("format", "metis"), false);
    std::ofstream tsv;
    if (o.given("data")) {
        tsv = open_for_writing(o.text("data"));
        tsv << "threads\ttime_ms\tspeedup\tmodularity\tedges\n";
    }
    std::printf("%8s %12s %9s %12s %12s\n", "threads", "time_ms", "speedup", "modularity", "edges");
    double first_ms = 0.0;
    for (std::size_t i = 0; i < counts.size(); ++i) {
        const int w = counts[i];
        if (w < 1)
            throw input_error("thread counts must be >= 1");
        Graph scaled;
        if (mode == "weak") {
            PlantedPartitionSpec sp = base;
            sp.n *= static_cast<count>(w);
            scaled = generate_planted(sp, w).first;
        }
        const Graph &g = mode == "weak" ? scaled : shared;
        s.workers = w;
        const RunReport r = run(g, s, seed).second;
        if (i == 0)
            first_ms = r.total_ms;
        const double speedup = r.total_ms > 0 ? first_ms / r.total_ms : 1.0;
        const auto edges = static_cast<unsigned long long>(g.edge_count());
        std::printf("%8d %12.2f %9.3f %12.6f %12llu\n", w, r.total_ms, speedup, r.modularity, edges);
        if (tsv)
            tsv << w << "\t" << r.total_ms << "\t" << speedup << "\t" << r.modularity << "\t" << edges << "\n";
    }
    return kOk;
}

int usage(int status) {
    std::cerr << "usage: commdet_gpu {detect|score|generate|bench} [options]\n"
                 "  (the reference CLI's flags; see the header of tools/commdet_gpu.cpp)\n";
    return status;
}

}  // namespace

int main(int argc, char **argv) {
    std::cout.precision(15);
    const std::string first = argc > 1 ? argv[1] : "";
    if (first == "--help" || first == "-h")
        return usage(kOk);
    static const std::map<std::string, int (*)(const Options &)> handlers = {
        {"detect", detect}, {"score", score}, {"generate", generate}, {"bench", bench}};
    auto h = handlers.find(first);
    if (h == handlers.end())
        return usage(kBadInput);
    try {
        const Options o(command_table().at(first), std::vector<std::string>(argv + 2, argv + argc));
        return h->second(o);
    } catch (const BadUsage &e) {
        std::cerr << e.what() << "\n";
        return usage(kBadInput);
    } catch (const input_error &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kBadInput;
    } catch (const std::invalid_argument &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kBadInput;
    } catch (const std::exception &e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return kInternal;
    }
}
