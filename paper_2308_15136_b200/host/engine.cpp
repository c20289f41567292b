// fodg drop-in: batch search and the benchmark contract (engine.cpp:82-180).
// One device launch per batch; seeds, modes and validation as the reference.
#include <algorithm>
#include <chrono>
#include <iomanip>
#include <sstream>

#include "abi.hpp"
#include "fodg/engine.hpp"

namespace fodg {

const char* mode_name(ExecutionMode mode) {
    return mode == ExecutionMode::kPerQueryWorker ? "per_query" : "shared";
}

// b_T = 0 resolves to the device's parallel workers (SMs).
ExecutionMode choose_mode(std::uint64_t batch_size, std::uint32_t topm, const ModeThresholds& th) {
    const std::uint64_t bt = th.batch_threshold ? th.batch_threshold : b200::device_sm_count();
    return (batch_size < bt || topm > th.topm_threshold) ? ExecutionMode::kSharedQueryWorkers
                                                          : ExecutionMode::kPerQueryWorker;
}

namespace {

cagra_search_params to_abi(const SearchParams& s) {
    cagra_search_params p;
    cagra_search_params_default(&p);
    p.k = s.k;
    p.topm = s.topm;
    p.width = s.width;
    p.max_iterations = s.max_iterations;
    p.min_iterations = s.min_iterations;
    p.hash_policy = s.hash_policy == HashPolicy::kForgettable ? CAGRA_HASH_FORGETTABLE : CAGRA_HASH_STANDARD;
    p.hash_bits = s.hash_bits;
    p.reset_interval = s.reset_interval;
    p.seed = s.seed;
    return p;
}

}  // namespace

std::vector<SearchResult> batch_search(const Graph& graph, const Dataset& ds, const Dataset& queries,
                                       const SearchParams& params, const EngineOptions& options) {
    // engine.cpp:98-102, same order
    if (queries.size() == 0) return {};
    if (queries.dim() != ds.dim()) throw UsageError("batch_search: query dimension mismatch");
    params.validate();
    if (options.mode == ExecutionMode::kSharedQueryWorkers && options.team_count < 2)
        throw UsageError("batch_search: shared mode requires team_count >= 2");
    if (graph.num_nodes != ds.size()) throw UsageError("search: graph/dataset size mismatch");
    const cagra_search_params p = to_abi(params);
    cagra_engine_opts o;
    cagra_engine_opts_default(&o);
    o.mode = options.mode == ExecutionMode::kSharedQueryWorkers ? CAGRA_MODE_SHARED : CAGRA_MODE_PER_QUERY;
    o.team_count = options.team_count;
    o.num_threads = options.num_threads;
    o.seed_mode = 0;  // mix_seed(seed ^ (0x0bad + qi)), engine.cpp:108
    o.exact_distances = b200::fast_distances() ? 0u : 1u;
    const std::uint32_t nq = queries.size(), k = params.k;
    std::vector<std::uint32_t> ids(static_cast<std::size_t>(nq) * k), counts(nq);
    std::vector<float> dists(ids.size());
    std::vector<cagra_search_stats> st(nq);
    // CAGRA_DEVICES=0,1,...: the batch is split over replicas on those GPUs
    // (results identical to one device: every query keeps its global seed)
    b200::with_index(graph, ds, [&](cagra_index* ix, cagra_mindex* mx) {
        if (mx)
            b200::check(cagra_msearch(mx, queries.raw(), nq, queries.dim(), &p, &o, ids.data(),
                                      dists.data(), counts.data(), st.data()));
        else
            b200::check(cagra_search(ix, queries.raw(), nq, queries.dim(), &p, &o, ids.data(),
                                     dists.data(), counts.data(), st.data()));
    });
    std::vector<SearchResult> out(nq);
    for (std::uint32_t q = 0; q < nq; ++q) {
        auto& r = out[q];
        const std::size_t b = static_cast<std::size_t>(q) * k;
        r.ids.assign(ids.begin() + b, ids.begin() + b + counts[q]);
        r.dists.assign(dists.begin() + b, dists.begin() + b + counts[q]);
        r.stats.iterations = st[q].iterations;
        r.stats.distance_evals = st[q].distance_evals;
        r.stats.hash_resets = st[q].hash_resets;
        r.stats.converged = st[q].converged != 0;
    }
    return out;
}

std::string bench_csv_header() { return "dataset,mode,M,p,d,k,iterations,recall,qps"; }

std::string bench_csv_row(const BenchRecord& r) {
    std::ostringstream os;
    os << r.dataset << ',' << mode_name(r.mode) << ',' << r.params.topm << ',' << r.params.width << ','
       << r.graph_degree << ',' << r.params.k << ',' << std::fixed << std::setprecision(2)
       << r.mean_iterations << ',' << std::setprecision(6) << r.recall << ',' << std::setprecision(1)
       << r.qps;
    return os.str();
}

std::vector<BenchRecord> run_benchmark(const Graph& graph, const Dataset& ds, const Dataset& queries,
                                       const std::vector<std::vector<std::uint32_t>>& truth,
                                       const std::vector<SearchParams>& param_grid,
                                       const EngineOptions& options, const std::string& dataset_name) {
    if (queries.size() == 0) throw UsageError("run_benchmark: no queries");
    if (truth.size() < queries.size()) throw UsageError("run_benchmark: missing ground truth rows");
    for (const auto& p : param_grid) {
        p.validate();
        for (std::uint32_t q = 0; q < queries.size(); ++q)
            if (truth[q].size() < p.k) throw UsageError("run_benchmark: ground truth shorter than k");
    }
    std::vector<BenchRecord> records;
    for (const auto& p : param_grid) {
        batch_search(graph, ds, queries, p, options);  // untimed warm-up (also uploads the index)
        const auto t0 = std::chrono::steady_clock::now();
        const auto results = batch_search(graph, ds, queries, p, options);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        double rsum = 0.0, isum = 0.0;
        for (std::uint32_t q = 0; q < queries.size(); ++q) {
            std::size_t hits = 0;
            for (const std::uint32_t id : results[q].ids)
                for (std::uint32_t j = 0; j < p.k; ++j)
                    if (truth[q][j] == id) {
                        ++hits;
                        break;
                    }
            rsum += static_cast<double>(hits) / p.k;
            isum += results[q].stats.iterations;
        }
        BenchRecord rec;
        rec.dataset = dataset_name;
        rec.mode = options.mode;
        rec.params = p;
        rec.graph_degree = graph.degree;
        rec.mean_iterations = isum / queries.size();
        rec.recall = rsum / queries.size();
        rec.qps = queries.size() / std::max(el, 1e-12);
        records.push_back(rec);
    }
    return records;
}

}  // namespace fodg
