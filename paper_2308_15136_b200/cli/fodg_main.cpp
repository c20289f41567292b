// `fodg` command line over the B200 engine: the reference CLI's subcommands
// (build / metrics / search / bench), flags and exit codes (0 ok, 2 usage,
// 3 format / other errors), on the drop-in library.  A small flag parser
// replaces the absent CLI11.
#include <algorithm>
#include <chrono>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "fodg/engine.hpp"
#include "fodg/graph_metrics.hpp"
#include "fodg/graph_opt.hpp"
#include "fodg/io.hpp"
#include "fodg/knn_build.hpp"

namespace {

constexpr int kOk = 0, kUsage = 2, kFormat = 3;

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --flag value pairs; a flag given several times keeps every value (--grid).
class Flags {
public:
    Flags(int argc, char** argv, int first) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw ParseError("unexpected argument: " + a);
            const auto eq = a.find('=');
            if (eq != std::string::npos) {
                vals_[a.substr(2, eq - 2)].push_back(a.substr(eq + 1));
            } else {
                if (i + 1 >= argc) throw ParseError(a + " needs a value");
                vals_[a.substr(2)].push_back(argv[++i]);
            }
        }
    }
    bool has(const std::string& k) const { return vals_.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") {
        seen_.insert(k);
        return has(k) ? vals_.at(k).back() : def;
    }
    std::string required(const std::string& k) {
        if (!has(k)) throw ParseError("--" + k + " is required");
        return str(k);
    }
    template <typename T>
    T num(const std::string& k, T def) {
        if (!has(k)) {
            seen_.insert(k);
            return def;
        }
        const std::string v = str(k);
        try {
            std::size_t pos = 0;
            const unsigned long long x = std::stoull(v, &pos);
            if (pos != v.size()) throw std::invalid_argument(v);
            return static_cast<T>(x);
        } catch (const std::exception&) {
            throw ParseError("--" + k + ": not a non-negative integer: " + v);
        }
    }
    std::vector<std::string> all(const std::string& k) {
        seen_.insert(k);
        return has(k) ? vals_.at(k) : std::vector<std::string>{};
    }
    void reject_unknown() const {
        for (const auto& [k, v] : vals_)
            if (!seen_.count(k)) throw ParseError("unknown flag --" + k);
    }

private:
    std::map<std::string, std::vector<std::string>> vals_;
    std::set<std::string> seen_;
};

std::vector<std::uint32_t> u32_list(const std::string& csv) {
    std::vector<std::uint32_t> out;
    std::stringstream ss(csv);
    std::string item;
    while (std::getline(ss, item, ','))
        if (!item.empty()) out.push_back(static_cast<std::uint32_t>(std::stoul(item)));
    if (out.empty()) throw fodg::UsageError("empty value list in grid spec");
    return out;
}

struct SearchOpts {
    fodg::SearchParams params;
    std::string exec = "auto";
    std::uint32_t teams = 4, b_t = 0, m_t = 512;
    unsigned threads = 0;
};

SearchOpts search_flags(Flags& f) {
    SearchOpts o;
    auto& p = o.params;
    p.k = f.num<std::uint32_t>("k", p.k);
    p.topm = f.num<std::uint32_t>("M", p.topm);
    p.width = f.num<std::uint32_t>("p", p.width);
    p.max_iterations = f.num<std::uint32_t>("i-max", p.max_iterations);
    p.min_iterations = f.num<std::uint32_t>("min-iterations", p.min_iterations);
    const std::string hash = f.str("hash", "standard");
    p.hash_bits = f.num<std::uint32_t>("hash-bits", p.hash_bits);
    p.reset_interval = f.num<std::uint32_t>("reset-interval", p.reset_interval);
    p.seed = f.num<std::uint64_t>("seed", p.seed);
    o.threads = f.num<unsigned>("threads", 0);
    o.exec = f.str("exec", "auto");
    o.teams = f.num<std::uint32_t>("team-count", 4);
    o.b_t = f.num<std::uint32_t>("b-t", 0);
    o.m_t = f.num<std::uint32_t>("m-t", 512);
    if (hash == "forgettable") p.hash_policy = fodg::HashPolicy::kForgettable;
    else if (hash != "standard") throw fodg::UsageError("--hash must be standard or forgettable");
    return o;
}

fodg::ExecutionMode exec_mode(const SearchOpts& o, std::uint64_t batch, std::uint32_t topm) {
    if (o.exec == "per-query") return fodg::ExecutionMode::kPerQueryWorker;
    if (o.exec == "shared") return fodg::ExecutionMode::kSharedQueryWorkers;
    return fodg::choose_mode(batch, topm, {o.b_t, o.m_t});
}

int cmd_build(Flags& f) {
    const std::string data = f.required("data"), out = f.required("out");
    const std::uint32_t d = f.num<std::uint32_t>("d", 32);
    std::uint32_t d_init = f.num<std::uint32_t>("d-init", 0);
    const std::string mode = f.str("mode", "rank"), builder = f.str("builder", "auto");
    const std::uint64_t seed = f.num<std::uint64_t>("seed", 0);
    const unsigned threads = f.num<unsigned>("threads", 0);
    f.reject_unknown();
    if (d == 0) throw fodg::UsageError("build: --d must be >= 1");
    if (!d_init) d_init = 2 * d;
    if (d_init < d) throw fodg::UsageError("build: --d-init must be >= --d");
    const fodg::Dataset ds = fodg::load_fvecs(data);
    if (mode != "rank" && mode != "distance") throw fodg::UsageError("build: --mode must be rank or distance");
    const auto rmode = mode == "distance" ? fodg::ReorderMode::kDistance : fodg::ReorderMode::kRank;
    if (builder != "exact" && builder != "nn-descent" && builder != "auto")
        throw fodg::UsageError("build: --builder must be exact, nn-descent, or auto");
    const bool exact = builder == "exact" || (builder == "auto" && ds.size() <= 4096);
    if (d_init >= ds.size()) throw fodg::UsageError("build: --d-init must be < N");
    const auto t0 = std::chrono::steady_clock::now();
    fodg::KnnGraph knn;
    if (exact) {
        knn = fodg::exact_knn_graph(ds, d_init, threads);
    } else {
        fodg::NNDescentParams np;
        np.seed = seed;
        np.num_threads = threads;
        knn = fodg::nn_descent(ds, d_init, np);
    }
    const double knn_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fodg::OptimizeOptions opts;
    opts.mode = rmode;
    opts.num_threads = threads;
    fodg::OptimizeStats st;
    const fodg::Graph g = fodg::optimize(knn, d, opts, rmode == fodg::ReorderMode::kDistance ? &ds : nullptr, &st);
    fodg::save_graph(g, out);
    std::cout << "builder=" << (exact ? "exact" : "nn-descent") << "\n"
              << "reorder_mode=" << mode << "\n"
              << "num_nodes=" << g.num_nodes << "\n"
              << "degree=" << g.degree << "\n"
              << "d_init=" << d_init << "\n"
              << "knn_build_seconds=" << knn_s << "\n"
              << st.report();
    return kOk;
}

int cmd_metrics(Flags& f) {
    const std::string gp = f.required("graph");
    const unsigned threads = f.num<unsigned>("threads", 0);
    f.reject_unknown();
    std::cout << fodg::measure_graph(fodg::load_graph(gp), threads).report();
    return kOk;
}

int cmd_search(Flags& f) {
    const std::string gp = f.required("graph"), dp = f.required("data"), qp = f.required("queries");
    SearchOpts o = search_flags(f);
    f.reject_unknown();
    const fodg::Graph g = fodg::load_graph(gp);
    const fodg::Dataset ds = fodg::load_fvecs(dp), qs = fodg::load_fvecs(qp);
    fodg::EngineOptions eo;
    eo.mode = exec_mode(o, qs.size(), o.params.topm);
    eo.team_count = o.teams;
    eo.num_threads = o.threads;
    const auto res = fodg::batch_search(g, ds, qs, o.params, eo);
    for (std::uint32_t q = 0; q < res.size(); ++q) {
        std::cout << "query " << q << ":";
        for (std::size_t i = 0; i < res[q].ids.size(); ++i) std::cout << ' ' << res[q].ids[i] << ':' << res[q].dists[i];
        std::cout << "\n";
    }
    return kOk;
}

int cmd_bench(Flags& f) {
    const std::string gp = f.required("graph"), dp = f.required("data"), qp = f.required("queries"),
                      tp = f.required("truth");
    SearchOpts o = search_flags(f);
    const auto grid_entries = f.all("grid");
    const std::string out_path = f.str("out", ""), name = f.str("name", "dataset");
    f.reject_unknown();
    const fodg::Graph g = fodg::load_graph(gp);
    const fodg::Dataset ds = fodg::load_fvecs(dp), qs = fodg::load_fvecs(qp);
    const fodg::IdMatrix tm = fodg::load_ivecs(tp);
    std::vector<std::vector<std::uint32_t>> truth(tm.rows);
    for (std::uint32_t i = 0; i < tm.rows; ++i)
        for (const std::int32_t id : tm.row(i)) {
            if (id < 0) throw fodg::FormatError("negative id in ground truth");
            truth[i].push_back(static_cast<std::uint32_t>(id));
        }
    std::vector<std::uint32_t> ms{64}, ps{1};
    for (const auto& e : grid_entries) {
        const auto eq = e.find('=');
        if (eq == std::string::npos) throw fodg::UsageError("grid entry must look like M=16,32,64: " + e);
        const std::string key = e.substr(0, eq);
        if (key == "M") ms = u32_list(e.substr(eq + 1));
        else if (key == "p") ps = u32_list(e.substr(eq + 1));
        else throw fodg::UsageError("unknown grid key (expected M or p): " + key);
    }
    std::vector<fodg::SearchParams> grid;
    for (const auto m : ms)
        for (const auto p : ps) {
            fodg::SearchParams sp = o.params;
            sp.topm = m;
            sp.width = p;
            grid.push_back(sp);
        }
    fodg::EngineOptions eo;
    eo.mode = exec_mode(o, qs.size(), *std::max_element(ms.begin(), ms.end()));
    eo.team_count = o.teams;
    eo.num_threads = o.threads;
    const auto recs = fodg::run_benchmark(g, ds, qs, truth, grid, eo, name);
    std::ostringstream csv;
    csv << fodg::bench_csv_header() << "\n";
    for (const auto& r : recs) csv << fodg::bench_csv_row(r) << "\n";
    if (out_path.empty()) {
        std::cout << csv.str();
    } else {
        std::ofstream out(out_path, std::ios::trunc);
        if (!out) throw fodg::FormatError("cannot open for writing: " + out_path);
        out << csv.str();
    }
    return kOk;
}

void usage(std::ostream& os) {
    os << "usage: fodg <build|metrics|search|bench> [--flag value ...]\n"
          "  build   --data D.fvecs --out G [--d 32 --d-init 0 --mode rank|distance "
          "--builder exact|nn-descent|auto --seed 0 --threads 0]\n"
          "  metrics --graph G [--threads 0]\n"
          "  search  --graph G --data D --queries Q [--k --M --p --i-max --min-iterations --hash "
          "--hash-bits --reset-interval --seed --threads --exec auto|per-query|shared --team-count "
          "--b-t --m-t]\n"
          "  bench   (search flags) --truth T.ivecs [--grid M=16,32 --grid p=1,2 --out CSV --name N]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage(std::cerr);
        return kUsage;
    }
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
        usage(std::cout);
        return kOk;
    }
    std::map<std::string, std::function<int(Flags&)>> cmds{
        {"build", cmd_build}, {"metrics", cmd_metrics}, {"search", cmd_search}, {"bench", cmd_bench}};
    auto it = cmds.find(cmd);
    if (it == cmds.end()) {
        std::cerr << "fodg: unknown subcommand " << cmd << "\n";
        usage(std::cerr);
        return kUsage;
    }
    try {
        Flags f(argc, argv, 2);
        return it->second(f);
    } catch (const ParseError& e) {
        std::cerr << "fodg: " << e.what() << "\n";
        return kUsage;
    } catch (const fodg::UsageError& e) {
        std::cerr << "fodg: usage error: " << e.what() << "\n";
        return kUsage;
    } catch (const fodg::FormatError& e) {
        std::cerr << "fodg: " << e.what() << "\n";
        return kFormat;
    } catch (const std::exception& e) {
        std::cerr << "fodg: error: " << e.what() << "\n";
        return kFormat;
    }
}
