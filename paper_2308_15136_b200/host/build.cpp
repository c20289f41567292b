// fodg drop-in: kNN graph build and graph optimization, on the device.
#include <algorithm>
#include <chrono>
#include <sstream>
#include <unordered_set>

#include "abi.hpp"
#include "fodg/graph_opt.hpp"
#include "fodg/knn_build.hpp"

namespace fodg {

KnnGraph exact_knn_graph(const Dataset& ds, std::uint32_t k, unsigned /*num_threads*/) {
    if (k == 0 || k >= ds.size()) throw UsageError("exact_knn_graph: require 1 <= k < N");
    KnnGraph g;
    g.num_nodes = ds.size();
    g.degree = k;
    g.ids.resize(static_cast<std::size_t>(g.num_nodes) * k);
    g.dists.resize(g.ids.size());
    const std::vector<int> devs = b200::devices();
    if (devs.size() > 1)  // CAGRA_DEVICES: rows spread over the set (row-sharded K1)
        b200::check(cagra_exact_knn_graph_multi(ds.raw(), ds.size(), ds.dim(), k, devs.data(),
                                                static_cast<std::uint32_t>(devs.size()),
                                                g.ids.data(), g.dists.data()));
    else
        b200::check(cagra_exact_knn_graph(ds.raw(), ds.size(), ds.dim(), k, devs[0],
                                          g.ids.data(), g.dists.data()));
    return g;
}

// nn_descent (knn_build.cpp:96-231) on the device (csrc/nn_descent.cu):
// same validation, deterministic for a fixed seed, thread count ignored.
KnnGraph nn_descent(const Dataset& ds, std::uint32_t k, const NNDescentParams& params) {
    if (k == 0 || k >= ds.size()) throw UsageError("nn_descent: require 1 <= k < N");
    if (params.sample_rate <= 0.0 || params.sample_rate > 1.0)
        throw UsageError("nn_descent: sample_rate must be in (0, 1]");
    if (params.termination_delta <= 0.0 || params.termination_delta >= 1.0)
        throw UsageError("nn_descent: termination_delta must be in (0, 1)");
    KnnGraph g;
    g.num_nodes = ds.size();
    g.degree = k;
    g.ids.resize(static_cast<std::size_t>(g.num_nodes) * k);
    g.dists.resize(g.ids.size());
    std::uint32_t conv = 0;
    b200::check(cagra_nn_descent(ds.raw(), ds.size(), ds.dim(), k, params.sample_rate,
                                 params.termination_delta, params.max_rounds, params.seed,
                                 b200::device(), g.ids.data(), g.dists.data(), &conv, nullptr));
    g.converged = conv != 0;
    return g;
}

void sort_neighbor_lists(KnnGraph& g) {
    if (g.dists.size() != g.ids.size()) throw UsageError("sort_neighbor_lists: rows have no distances");
    std::vector<std::pair<float, std::uint32_t>> row(g.degree);
    for (std::uint32_t v = 0; v < g.num_nodes; ++v) {
        const std::size_t b = static_cast<std::size_t>(v) * g.degree;
        for (std::uint32_t j = 0; j < g.degree; ++j) row[j] = {g.dists[b + j], g.ids[b + j]};
        std::sort(row.begin(), row.end());
        for (std::uint32_t j = 0; j < g.degree; ++j) {
            g.dists[b + j] = row[j].first;
            g.ids[b + j] = row[j].second;
        }
    }
}

double knn_graph_recall(const KnnGraph& g, const KnnGraph& exact) {
    if (g.num_nodes != exact.num_nodes || g.degree != exact.degree)
        throw UsageError("knn_graph_recall: shape mismatch");
    double sum = 0.0;
    for (std::uint32_t v = 0; v < g.num_nodes; ++v) {
        const auto t = exact.row_ids(v);
        const std::unordered_set<std::uint32_t> truth(t.begin(), t.end());
        std::size_t hits = 0;
        for (const std::uint32_t id : g.row_ids(v)) hits += truth.count(id);
        sum += static_cast<double>(hits) / g.degree;
    }
    return sum / g.num_nodes;
}

std::string OptimizeStats::report() const {
    std::ostringstream os;
    os << "stage_detour_count_seconds=" << count_seconds << "\n"
       << "stage_reorder_seconds=" << reorder_seconds << "\n"
       << "stage_reverse_seconds=" << reverse_seconds << "\n"
       << "stage_merge_seconds=" << merge_seconds << "\n"
       << "optimize_total_seconds=" << total_seconds << "\n";
    return os.str();
}

namespace {
void require_dists(const KnnGraph& g) {
    if (g.dists.size() != g.ids.size()) throw UsageError("graph_opt: input rows have no distances");
}
}  // namespace

std::vector<std::uint32_t> count_detourable_routes(const KnnGraph& g, ReorderMode mode,
                                                   const Dataset* ds, unsigned /*num_threads*/) {
    require_dists(g);
    std::vector<std::uint32_t> counts(static_cast<std::size_t>(g.num_nodes) * g.degree);
    if (mode == ReorderMode::kRank) {
        b200::check(cagra_count_detourable_routes(g.ids.data(), g.dists.data(), g.num_nodes,
                                                  g.degree, b200::device(), counts.data()));
    } else {
        b200::check(cagra_count_detourable_routes_distance(
            g.ids.data(), g.dists.data(), g.num_nodes, g.degree, ds ? ds->raw() : nullptr,
            ds ? ds->size() : 0, ds ? ds->dim() : 0, b200::device(), counts.data()));
    }
    return counts;
}

Graph reorder_and_prune(const KnnGraph& g, const std::vector<std::uint32_t>& counts, std::uint32_t d,
                        unsigned /*num_threads*/) {
    if (d == 0 || d > g.degree) throw UsageError("reorder_and_prune: require 1 <= d <= input degree");
    if (counts.size() != g.ids.size()) throw UsageError("reorder_and_prune: counts size mismatch");
    Graph out;
    out.num_nodes = g.num_nodes;
    out.degree = d;
    out.ids.resize(static_cast<std::size_t>(g.num_nodes) * d);
    b200::check(cagra_reorder_and_prune(g.ids.data(), counts.data(), g.num_nodes, g.degree, d,
                                        b200::device(), out.ids.data()));
    return out;
}

Graph truncate_graph(const KnnGraph& g, std::uint32_t d) {
    if (d == 0 || d > g.degree) throw UsageError("truncate_graph: require 1 <= d <= input degree");
    Graph out;
    out.num_nodes = g.num_nodes;
    out.degree = d;
    out.ids.reserve(static_cast<std::size_t>(g.num_nodes) * d);
    for (std::uint32_t v = 0; v < g.num_nodes; ++v) {
        const auto r = g.row_ids(v);
        out.ids.insert(out.ids.end(), r.begin(), r.begin() + d);
    }
    return out;
}

ReverseGraph build_reverse_graph(const Graph& pruned, std::uint32_t cap) {
    ReverseGraph rg;
    rg.num_nodes = pruned.num_nodes;
    rg.rows.resize(pruned.num_nodes);
    const std::uint32_t c = std::max<std::uint32_t>(std::min(cap, pruned.num_nodes), 1);
    std::vector<std::uint32_t> cnt(pruned.num_nodes), ids(static_cast<std::size_t>(pruned.num_nodes) * c);
    b200::check(cagra_build_reverse_graph(pruned.ids.data(), pruned.num_nodes, pruned.degree, cap,
                                          b200::device(), cnt.data(), ids.data()));
    for (std::uint32_t y = 0; y < pruned.num_nodes; ++y)
        rg.rows[y].assign(ids.begin() + static_cast<std::size_t>(y) * c,
                          ids.begin() + static_cast<std::size_t>(y) * c + cnt[y]);
    return rg;
}

Graph merge_graphs(const Graph& pruned, const ReverseGraph& rev, std::uint32_t d) {
    if (pruned.degree != d) throw UsageError("merge_graphs: pruned degree must equal d");
    if (rev.num_nodes != pruned.num_nodes || rev.rows.size() != pruned.num_nodes)
        throw UsageError("merge_graphs: size mismatch");
    std::uint32_t cap = 1;
    for (const auto& r : rev.rows) cap = std::max<std::uint32_t>(cap, static_cast<std::uint32_t>(r.size()));
    std::vector<std::uint32_t> cnt(pruned.num_nodes), ids(static_cast<std::size_t>(pruned.num_nodes) * cap,
                                                          kInvalidId);
    for (std::uint32_t y = 0; y < pruned.num_nodes; ++y) {
        cnt[y] = static_cast<std::uint32_t>(rev.rows[y].size());
        std::copy(rev.rows[y].begin(), rev.rows[y].end(), ids.begin() + static_cast<std::size_t>(y) * cap);
    }
    Graph out;
    out.num_nodes = pruned.num_nodes;
    out.degree = d;
    out.ids.resize(static_cast<std::size_t>(pruned.num_nodes) * d);
    b200::check(cagra_merge_graphs(pruned.ids.data(), cnt.data(), ids.data(), pruned.num_nodes, d,
                                   cap, b200::device(), out.ids.data()));
    return out;
}

Graph optimize(const KnnGraph& g, std::uint32_t d, const OptimizeOptions& opts, const Dataset* ds,
               OptimizeStats* stats) {
    if (d == 0 || d > g.degree) throw UsageError("optimize: require 1 <= d <= input degree");
    if (opts.reorder) require_dists(g);
    Graph out;
    out.num_nodes = g.num_nodes;
    out.degree = d;
    out.ids.resize(static_cast<std::size_t>(g.num_nodes) * d);
    if (opts.mode == ReorderMode::kRank || !opts.reorder) {
        cagra_opt_stats st{};
        b200::check(cagra_optimize(g.ids.data(), g.dists.empty() ? nullptr : g.dists.data(),
                                   g.num_nodes, g.degree, d,
                                   opts.reorder ? 1u : 0u, opts.add_reverse ? 1u : 0u,
                                   b200::device(), out.ids.data(), &st));
        if (stats) {
            stats->count_seconds = st.count_seconds;
            stats->reorder_seconds = st.reorder_seconds;
            stats->reverse_seconds = st.reverse_seconds;
            stats->merge_seconds = st.merge_seconds;
            stats->total_seconds = st.total_seconds;
        }
        return out;
    }
    // distance mode (comparison variant): device stages one by one
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    auto counts = count_detourable_routes(g, ReorderMode::kDistance, ds, opts.num_threads);
    const auto t1 = clock::now();
    Graph pruned = reorder_and_prune(g, counts, d, opts.num_threads);
    const auto t2 = clock::now();
    Graph result = pruned;
    auto t3 = t2, t4 = t2;
    if (opts.add_reverse) {
        ReverseGraph rev = build_reverse_graph(pruned, d);
        t3 = clock::now();
        result = merge_graphs(pruned, rev, d);
        t4 = clock::now();
    }
    if (stats) {
        auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        stats->count_seconds = s(t0, t1);
        stats->reorder_seconds = s(t1, t2);
        stats->reverse_seconds = s(t2, t3);
        stats->merge_seconds = s(t3, t4);
        stats->total_seconds = s(t0, t4);
    }
    return result;
}

}  // namespace fodg
