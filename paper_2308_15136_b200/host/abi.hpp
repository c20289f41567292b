// Bridge from the fodg:: drop-in to the C ABI (include/cagra/capi.h):
// status codes -> the reference's exception types, device selection, and the
// cache of device-resident indexes that stands in for the reference's
// per-call `const Graph&, const Dataset&` (re-uploading the index on every
// batch_search would dominate).
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "cagra/capi.h"
#include "fodg/dataset.hpp"
#include "fodg/graph.hpp"

namespace fodg::b200 {

/// Throws UsageError / FormatError / std::logic_error / std::runtime_error
/// for a non-zero cagra status (message from cagra_last_error()).
void check(int rc);

/// CUDA device used by the drop-in (env CAGRA_DEVICE, default 0).
int device();

/// Devices the drop-in spreads batch_search / exact_knn_graph over
/// (env CAGRA_DEVICES=0,1,..., default {device()}).
std::vector<int> devices();

/// Fast in-loop distances (team reductions; reported distances still the
/// sequential chain, ids and recall as the reference's within the parity bar)
/// — the default; CAGRA_FAST_DISTANCES=0 selects the reference-order chain
/// everywhere (ids, distances and counters bit for bit).
bool fast_distances();

/// The device index for (graph, ds), created on first use and reused while
/// the host buffers are unchanged.
cagra_index* index_for(const Graph& graph, const Dataset& ds);

/// Runs `search(ix, mx)` on the cached device copy of (graph, ds) for the
/// current device set (one of ix / mx is set).  A cached copy found by
/// address and shape is searched at once while the full-content hash of the
/// host buffers is computed on host threads in parallel; if the contents
/// changed, the copy is re-uploaded and the search re-run — so in-place edits
/// are always seen, and the check costs no latency when the search takes
/// longer than the hash (large batches).
void with_index(const Graph& graph, const Dataset& ds,
                const std::function<void(cagra_index*, cagra_mindex*)>& search);

/// The replicated device-set index (CAGRA_DEVICES with more than one entry)
/// for (graph, ds), cached under the same rule as index_for.
cagra_mindex* mindex_for(const Graph& graph, const Dataset& ds);

/// SM count of device() (the default b_T of choose_mode).
unsigned device_sm_count();

}  // namespace fodg::b200
