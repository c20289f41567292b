// fodg drop-in: Dataset / distance / validate_graph / exact top-k / recall.
#include <cmath>
#include <unordered_set>

#include "abi.hpp"
#include "fodg/dataset.hpp"
#include "fodg/graph.hpp"
#include "fodg/topk.hpp"

namespace fodg {

// dataset.cpp:7-18 validation, same order and messages.
Dataset::Dataset(std::uint32_t dim, std::vector<float> data) : dim_(dim), data_(std::move(data)) {
    if (dim_ == 0) throw UsageError("dataset dimension must be >= 1");
    if (data_.empty() || data_.size() % dim_ != 0)
        throw UsageError("dataset size is not a multiple of the dimension");
    const std::size_t rows = data_.size() / dim_;
    if (rows > kMaxNodes) throw UsageError("dataset exceeds 2^31 - 1 vectors (index MSB is reserved)");
    for (const float v : data_)
        if (!std::isfinite(v)) throw UsageError("dataset contains non-finite components");
    n_rows_ = static_cast<std::uint32_t>(rows);
}

float distance(std::span<const float> a, std::span<const float> b) {
    if (a.size() != b.size()) throw UsageError("distance: dimension mismatch");
    return squared_l2(a, b);
}

void validate_graph(const Graph& g) {
    if (g.num_nodes == 0 || g.degree == 0) throw FormatError("graph: empty");
    if (g.ids.size() != static_cast<std::size_t>(g.num_nodes) * g.degree)
        throw FormatError("graph: payload size mismatch");
    std::vector<std::uint32_t> seen;
    for (std::uint32_t v = 0; v < g.num_nodes; ++v) {
        const auto r = g.row(v);
        for (std::uint32_t j = 0; j < g.degree; ++j) {
            const std::uint32_t id = r[j];
            if (has_parent_flag(id)) throw FormatError("graph: id with MSB set");
            if (id >= g.num_nodes) throw FormatError("graph: id out of range");
            if (id == v) throw FormatError("graph: self loop");
            for (std::uint32_t i = 0; i < j; ++i)
                if (r[i] == id) throw FormatError("graph: duplicate id in row");
        }
    }
}

NeighborList exact_topk(const Dataset& ds, std::span<const float> q, std::uint32_t k) {
    if (q.size() != ds.dim()) throw UsageError("exact_topk: query dimension mismatch");
    if (k == 0 || k > ds.size()) throw UsageError("exact_topk: k out of range [1, N]");
    NeighborList out;
    out.ids.resize(k);
    out.dists.resize(k);
    b200::check(cagra_exact_topk(ds.raw(), ds.size(), ds.dim(), q.data(), 1, k, b200::device(),
                                 out.ids.data(), out.dists.data()));
    return out;
}

double recall(std::span<const std::uint32_t> result_ids, std::span<const std::uint32_t> truth_ids) {
    if (truth_ids.empty()) throw UsageError("recall: empty ground truth");
    if (result_ids.size() != truth_ids.size())
        throw UsageError("recall: result and truth lengths differ");
    const std::unordered_set<std::uint32_t> truth(truth_ids.begin(), truth_ids.end());
    if (truth.size() != truth_ids.size()) throw UsageError("recall: duplicate ids in truth");
    std::unordered_set<std::uint32_t> seen;
    std::size_t hits = 0;
    for (const std::uint32_t id : result_ids) {
        if (!seen.insert(id).second) throw UsageError("recall: duplicate ids in result");
        hits += truth.count(id);
    }
    return static_cast<double>(hits) / static_cast<double>(truth_ids.size());
}

}  // namespace fodg
