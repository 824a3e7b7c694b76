// commdet_gpu -- the reference's command-line driver (P/tools/commdet.cpp,
// SURVEY.md §8(f) rank 2) over the B200 library: the same subcommands, flags,
// text output, JSON report fields and exit codes, so scripts that drive the
// reference binary can drive this one.  Everything runs through the drop-in
// C++ shim (include/commdet/gpu.hpp) and therefore on the device:
//
//   detect    --algo plp|plm|plmr|epp --input F [--format metis|edges]
//             [--merge-duplicates] [--threads N] [--theta T] [--shuffle]
//             [--gamma G] [--ensemble B] [--seed S] [--runs R] [--output P]
//             [--report J] [--community-graph C]           (commdet.cpp:81-131)
//   score     --input F [--format] --partition P [--reference Q] [--gamma G]
//   generate  --n N --k K --pin P --pout Q [--seed S] [--threads] --output F
//             [--ground-truth T]
//   bench     [--mode strong|weak] [--algo] [--input F | --gen-n N --gen-k K
//             --gen-pin P --gen-pout Q] [--threads-list 1,2,4] [--seed]
//             [--theta] [--gamma] [--ensemble] [--data TSV]  (commdet.cpp:193-248)
//
// `--threads` is accepted and echoed like the reference's worker count; the
// device path does not use it.  Exit codes: 0 ok, 2 usage / input error,
// 3 internal error (commdet.cpp:24-25).
#define COMMDET_GPU_DROP_IN
#include <commdet/gpu.hpp>

#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace {

using namespace commdet;

constexpr int kExitUsage = 2;
constexpr int kExitInternal = 3;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --name value | --name=value | --flag
class Args {
  public:
    Args(int argc, char **argv, int first, const std::set<std::string> &flags, const std::set<std::string> &opts) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0)
                throw UsageError("unexpected argument '" + a + "'");
            std::string name = a.substr(2), value;
            const auto eq = name.find('=');
            if (eq != std::string::npos) {
                value = name.substr(eq + 1);
                name = name.substr(0, eq);
            }
            if (flags.count(name)) {
                if (eq != std::string::npos)
                    throw UsageError("flag --" + name + " takes no value");
                vals_[name] = "1";
            } else if (opts.count(name)) {
                if (eq == std::string::npos) {
                    if (i + 1 >= argc)
                        throw UsageError("--" + name + " requires a value");
                    value = argv[++i];
                }
                vals_[name] = value;
            } else {
                throw UsageError("unknown option --" + name);
            }
        }
    }
    bool has(const std::string &k) const { return vals_.count(k) > 0; }
    std::string str(const std::string &k, const std::string &def = "") const {
        auto it = vals_.find(k);
        return it == vals_.end() ? def : it->second;
    }
    std::string req(const std::string &k) const {
        if (!has(k))
            throw UsageError("--" + k + " is required");
        return str(k);
    }
    template <class T>
    T num(const std::string &k, T def) const {
        if (!has(k))
            return def;
        return parse<T>(k, str(k));
    }
    template <class T>
    static T parse(const std::string &k, const std::string &v) {
        try {
            size_t pos = 0;
            T out;
            if constexpr (std::is_floating_point_v<T>)
                out = static_cast<T>(std::stod(v, &pos));
            else if constexpr (std::is_signed_v<T>)
                out = static_cast<T>(std::stoll(v, &pos));
            else {
                if (!v.empty() && v[0] == '-')
                    throw std::invalid_argument("negative");
                out = static_cast<T>(std::stoull(v, &pos));
            }
            if (pos != v.size())
                throw std::invalid_argument("trailing");
            return out;
        } catch (const std::exception &) {
            throw UsageError("--" + k + ": invalid value '" + v + "'");
        }
    }

  private:
    std::map<std::string, std::string> vals_;
};

Graph load_graph(const std::string &path, const std::string &format, bool merge_duplicates) {
    if (format == "metis")
        return io::read_metis(path);
    if (format == "edges")
        return io::read_edge_list(path, merge_duplicates);
    throw input_error("unknown graph format '" + format + "'");
}

struct DetectOptions {
    std::string algo = "plm";
    std::string input;
    std::string format = "metis";
    bool merge_duplicates = false;
    int threads = 1;
    long long theta = -1;
    bool shuffle = false;
    double gamma = 1.0;
    count ensemble = 4;
    std::uint64_t seed = 1;
    unsigned runs = 1;
    std::string output;
    std::string report_path;
    std::string community_graph;
};

std::pair<Partition, RunReport> run_algorithm(const Graph &g, const DetectOptions &opt, std::uint64_t seed) {
    if (opt.algo == "plp") {
        PlpConfig cfg;
        cfg.theta = opt.theta;
        cfg.randomize_order = opt.shuffle;
        cfg.seed = seed;
        cfg.workers = opt.threads;
        return run_plp(g, cfg);
    }
    LouvainConfig lc;
    lc.gamma = opt.gamma;
    lc.seed = seed;
    lc.workers = opt.threads;
    if (opt.algo == "plm")
        return run_plm(g, lc);
    if (opt.algo == "plmr")
        return run_plmr(g, lc);
    if (opt.algo == "epp") {
        EnsembleConfig ec;
        ec.ensemble_size = opt.ensemble;
        ec.seed = seed;
        ec.workers = opt.threads;
        ec.base_plp.theta = opt.theta;
        ec.final_louvain.gamma = opt.gamma;
        return run_epp(g, ec);
    }
    throw input_error("unknown algorithm '" + opt.algo + "'");
}

int cmd_detect(const DetectOptions &opt) {
    const Graph g = load_graph(opt.input, opt.format, opt.merge_duplicates);
    std::vector<RunReport> reports;
    Partition best;
    double best_mod = -2.0;
    for (unsigned r = 0; r < opt.runs; ++r) {
        auto [z, report] = run_algorithm(g, opt, opt.seed + r);
        report.input = opt.input;
        if (report.modularity > best_mod) {
            best_mod = report.modularity;
            best = z.compacted();
        }
        reports.push_back(std::move(report));
    }
    double avg_ms = 0.0, avg_mod = 0.0, avg_cov = 0.0;
    for (const auto &r : reports) {
        avg_ms += r.total_ms;
        avg_mod += r.modularity;
        avg_cov += r.coverage;
    }
    avg_ms /= reports.size();
    avg_mod /= reports.size();
    avg_cov /= reports.size();
    std::cout << "algorithm " << opt.algo << "\n"
              << "runs " << opt.runs << "\n"
              << "threads " << opt.threads << "\n"
              << "avg_time_ms " << avg_ms << "\n"
              << "avg_modularity " << avg_mod << "\n"
              << "avg_coverage " << avg_cov << "\n"
              << "best_modularity " << best_mod << "\n"
              << "communities " << best.upper_bound() << "\n";
    if (!opt.output.empty())
        io::write_partition(best, opt.output);
    if (!opt.community_graph.empty())
        io::write_community_graph(g, best, opt.community_graph);
    if (!opt.report_path.empty()) {
        Json j = Json::object();
        Json avg = Json::object();
        avg["time_ms"] = avg_ms;
        avg["modularity"] = avg_mod;
        avg["coverage"] = avg_cov;
        j["average"] = avg;
        j["best_modularity"] = best_mod;
        Json runs = Json::array();
        for (const auto &r : reports)
            runs.push_back(r.to_json());
        j["runs"] = runs;
        std::ofstream out(opt.report_path);
        if (!out)
            throw input_error("cannot open " + opt.report_path + " for writing");
        out << j.dump(2) << "\n";
    }
    return 0;
}

int cmd_score(const Args &a) {
    const Graph g = load_graph(a.req("input"), a.str("format", "metis"), false);
    const Partition z = io::read_partition(a.req("partition"));
    if (z.size() != g.node_count())
        throw input_error("partition length " + std::to_string(z.size()) + " does not match node count " +
                          std::to_string(g.node_count()));
    const QualityReport q = evaluate(g, z, a.num<double>("gamma", 1.0));
    std::cout << "modularity " << q.modularity << "\n"
              << "coverage " << q.coverage << "\n"
              << "communities " << q.community_count << "\n";
    if (a.has("reference")) {
        const Partition ref = io::read_partition(a.str("reference"));
        if (ref.size() != g.node_count())
            throw input_error("reference partition length does not match node count");
        std::cout << "rand_index " << graph_rand_index(g, z, ref) << "\n";
    }
    return 0;
}

PlantedPartitionSpec gen_spec(const Args &a, const std::string &pre, bool required) {
    PlantedPartitionSpec s;
    auto get = [&](const std::string &k) { return required ? a.req(pre + k) : a.str(pre + k); };
    s.n = Args::parse<count>(pre + "n", get("n"));
    s.k = Args::parse<count>(pre + "k", get("k"));
    s.p_in = Args::parse<double>(pre + "pin", get("pin"));
    s.p_out = Args::parse<double>(pre + "pout", get("pout"));
    return s;
}

int cmd_generate(const Args &a) {
    PlantedPartitionSpec spec = gen_spec(a, "", true);
    spec.seed = a.num<std::uint64_t>("seed", 1);
    auto [g, truth] = generate_planted(spec, a.num<int>("threads", 1));
    io::write_metis(g, a.req("output"));
    if (a.has("ground-truth"))
        io::write_partition(truth.compacted(), a.str("ground-truth"));
    std::cout << "nodes " << g.node_count() << "\n"
              << "edges " << g.edge_count() << "\n"
              << "blocks " << spec.k << "\n";
    return 0;
}

int cmd_bench(const Args &a) {
    const std::string mode = a.str("mode", "strong");
    const bool use_generator = a.has("gen-n");
    if (mode != "strong" && mode != "weak")
        throw input_error("unknown bench mode '" + mode + "'");
    if (mode == "weak" && !use_generator)
        throw input_error("weak scaling requires a generator spec (--gen-n ...)");
    if (!use_generator && !a.has("input"))
        throw input_error("bench needs --input or --gen-n");
    std::vector<int> threads_list;
    {
        const std::string tl = a.str("threads-list", "1");
        size_t p = 0;
        while (p <= tl.size()) {
            const size_t q = tl.find(',', p);
            const std::string t = tl.substr(p, q == std::string::npos ? std::string::npos : q - p);
            threads_list.push_back(Args::parse<int>("threads-list", t));
            if (q == std::string::npos)
                break;
            p = q + 1;
        }
    }
    PlantedPartitionSpec gen;
    if (use_generator) {
        gen.n = Args::parse<count>("gen-n", a.str("gen-n"));
        gen.k = Args::parse<count>("gen-k", a.str("gen-k", "1"));
        gen.p_in = Args::parse<double>("gen-pin", a.str("gen-pin", "0"));
        gen.p_out = Args::parse<double>("gen-pout", a.str("gen-pout", "0"));
    }
    const std::uint64_t seed = a.num<std::uint64_t>("seed", 1);
    Graph fixed;
    if (mode == "strong")
        fixed = use_generator ? generate_planted(gen, threads_list.back()).first
                              : load_graph(a.str("input"), a.str("format", "metis"), false);
    std::printf("%8s %12s %9s %12s %12s\n", "threads", "time_ms", "speedup", "modularity", "edges");
    std::ofstream data;
    if (a.has("data")) {
        data.open(a.str("data"));
        if (!data)
            throw input_error("cannot open " + a.str("data") + " for writing");
        data << "threads\ttime_ms\tspeedup\tmodularity\tedges\n";
    }
    double base_time = 0.0;
    for (std::size_t i = 0; i < threads_list.size(); ++i) {
        const int t = threads_list[i];
        if (t < 1)
            throw input_error("thread counts must be >= 1");
        Graph scaled;
        const Graph *g = &fixed;
        if (mode == "weak") {
            PlantedPartitionSpec s = gen;
            s.n *= static_cast<count>(t);
            scaled = generate_planted(s, t).first;
            g = &scaled;
        }
        DetectOptions run;
        run.algo = a.str("algo", "plm");
        run.threads = t;
        run.theta = a.num<long long>("theta", -1);
        run.gamma = a.num<double>("gamma", 1.0);
        run.ensemble = a.num<count>("ensemble", 4);
        auto [z, report] = run_algorithm(*g, run, seed);
        if (i == 0)
            base_time = report.total_ms;
        const double speedup = report.total_ms > 0 ? base_time / report.total_ms : 1.0;
        std::printf("%8d %12.2f %9.3f %12.6f %12llu\n", t, report.total_ms, speedup, report.modularity,
                    static_cast<unsigned long long>(g->edge_count()));
        if (data)
            data << t << "\t" << report.total_ms << "\t" << speedup << "\t" << report.modularity << "\t"
                 << g->edge_count() << "\n";
    }
    return 0;
}

void usage() {
    std::cerr << "usage: commdet_gpu {detect|score|generate|bench} [options]\n"
                 "  (flags of the reference CLI, P/tools/commdet.cpp; see the header of tools/commdet_gpu.cpp)\n";
}

}  // namespace

int main(int argc, char **argv) {
    std::cout.precision(15);
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        usage();
        return argc < 2 ? kExitUsage : 0;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "detect") {
            Args a(argc, argv, 2, {"merge-duplicates", "shuffle"},
                   {"algo", "input", "format", "threads", "theta", "gamma", "ensemble", "seed", "runs", "output",
                    "report", "community-graph"});
            DetectOptions o;
            o.algo = a.str("algo", "plm");
            o.input = a.req("input");
            o.format = a.str("format", "metis");
            o.merge_duplicates = a.has("merge-duplicates");
            o.threads = a.num<int>("threads", 1);
            o.theta = a.num<long long>("theta", -1);
            o.shuffle = a.has("shuffle");
            o.gamma = a.num<double>("gamma", 1.0);
            o.ensemble = a.num<count>("ensemble", 4);
            o.seed = a.num<std::uint64_t>("seed", 1);
            o.runs = a.num<unsigned>("runs", 1);
            if (o.runs < 1)
                throw UsageError("--runs: value must be positive");
            o.output = a.str("output");
            o.report_path = a.str("report");
            o.community_graph = a.str("community-graph");
            return cmd_detect(o);
        }
        if (cmd == "score")
            return cmd_score(Args(argc, argv, 2, {}, {"input", "format", "partition", "reference", "gamma"}));
        if (cmd == "generate")
            return cmd_generate(
                Args(argc, argv, 2, {}, {"n", "k", "pin", "pout", "seed", "threads", "output", "ground-truth"}));
        if (cmd == "bench")
            return cmd_bench(Args(argc, argv, 2, {},
                                  {"mode", "algo", "input", "format", "gen-n", "gen-k", "gen-pin", "gen-pout",
                                   "threads-list", "seed", "theta", "gamma", "ensemble", "data"}));
        usage();
        return kExitUsage;
    } catch (const UsageError &e) {
        std::cerr << e.what() << "\n";
        usage();
        return kExitUsage;
    } catch (const input_error &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const std::invalid_argument &e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    } catch (const std::exception &e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return kExitInternal;
    }
}
