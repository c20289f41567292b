// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Neutral C wrapper over the UNMODIFIED reference library, compiled from the
// sources under /root/reference/proj/core/src with -Dfodg=fodg_ref into
// oracle/_ref/libfodg_ref.so (recipe: oracle/Makefile).  It lets the tests pin
// the C restatement (oracle/fodg_oracle.c) and the GPU engine against the
// reference itself, and lets bench.py time the reference CPU path
// (cpu_baseline kind "reference" and `bench.py --impl reference`).
//
// The entry points mirror oracle/fodg_oracle.h with a `ref_` prefix.
#include <cstdint>
#include <cstring>
#include <limits>
#include <span>
#include <stdexcept>
#include <vector>

#include "fodg/engine.hpp"
#include "fodg/graph_metrics.hpp"
#include "fodg/graph_opt.hpp"
#include "fodg/knn_build.hpp"
#include "fodg/search.hpp"
#include "fodg/topk.hpp"
#include "test_util.hpp"  // reference fixture generator (tests/test_util.hpp:11-18)

using namespace fodg_ref;

namespace {

struct Params {
  uint32_t k, topm, width, max_iterations, min_iterations, hash_policy, hash_bits,
      reset_interval;
  uint64_t seed;
};
struct Stats {
  uint32_t iterations, hash_resets;
  uint64_t distance_evals;
  uint32_t converged, pad;
};

SearchParams to_ref(const Params* p) {
  SearchParams s;
  s.k = p->k;
  s.topm = p->topm;
  s.width = p->width;
  s.max_iterations = p->max_iterations;
  s.min_iterations = p->min_iterations;
  s.hash_policy = p->hash_policy ? HashPolicy::kForgettable : HashPolicy::kStandard;
  s.hash_bits = p->hash_bits;
  s.reset_interval = p->reset_interval;
  s.seed = p->seed;
  return s;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError&) {
    return 2;
  } catch (const FormatError&) {
    return 3;
  } catch (const std::logic_error&) {
    return 6;
  } catch (...) {
    return 7;
  }
}

Dataset make_ds(const float* data, uint64_t rows, uint32_t dim) {
  return Dataset(dim, std::vector<float>(data, data + rows * dim));
}

struct RefIndex {
  Dataset ds;
  Graph g;
};

}  // namespace

extern "C" {

int ref_exact_knn_graph(const float* data, uint32_t n, uint32_t dim, uint32_t k, uint32_t* ids,
                        float* dists, int threads) {
  return guard([&] {
    Dataset ds = make_ds(data, n, dim);
    KnnGraph g = exact_knn_graph(ds, k, threads > 0 ? threads : 0);
    std::memcpy(ids, g.ids.data(), g.ids.size() * 4);
    std::memcpy(dists, g.dists.data(), g.dists.size() * 4);
  });
}

int ref_exact_topk_batch(const float* data, uint32_t n, uint32_t dim, const float* qs,
                         uint32_t nq, uint32_t k, uint32_t* ids, float* dists, int threads) {
  return guard([&] {
    Dataset ds = make_ds(data, n, dim);
    parallel_for(nq, threads > 0 ? threads : 0, [&](std::size_t qi) {
      NeighborList nl = exact_topk(ds, std::span<const float>(qs + qi * dim, dim), k);
      std::memcpy(ids + qi * k, nl.ids.data(), k * 4);
      std::memcpy(dists + qi * k, nl.dists.data(), k * 4);
    });
  });
}

static KnnGraph make_knn(const uint32_t* ids, const float* dists, uint32_t n, uint32_t deg) {
  KnnGraph g;
  g.num_nodes = n;
  g.degree = deg;
  g.ids.assign(ids, ids + (size_t)n * deg);
  g.dists.assign(dists, dists + (size_t)n * deg);
  return g;
}

int ref_count_detourable_routes(const uint32_t* ids, const float* dists, uint32_t n,
                                uint32_t deg, uint32_t* counts) {
  return guard([&] {
    auto c = count_detourable_routes(make_knn(ids, dists, n, deg), ReorderMode::kRank);
    std::memcpy(counts, c.data(), c.size() * 4);
  });
}

int ref_optimize(const uint32_t* ids, const float* dists, uint32_t n, uint32_t deg, uint32_t d,
                 uint32_t reorder, uint32_t add_reverse, uint32_t* out, double* seconds) {
  return guard([&] {
    OptimizeOptions o;
    o.reorder = reorder != 0;
    o.add_reverse = add_reverse != 0;
    OptimizeStats st;
    Graph g = optimize(make_knn(ids, dists, n, deg), d, o, nullptr, &st);
    std::memcpy(out, g.ids.data(), g.ids.size() * 4);
    if (seconds) {
      seconds[0] = st.count_seconds;
      seconds[1] = st.reorder_seconds;
      seconds[2] = st.reverse_seconds;
      seconds[3] = st.merge_seconds;
      seconds[4] = st.total_seconds;
    }
  });
}

int ref_build_reverse_graph(const uint32_t* pruned, uint32_t n, uint32_t d, uint32_t cap,
                            uint32_t* rev_counts, uint32_t* rev_ids) {
  return guard([&] {
    Graph g;
    g.num_nodes = n;
    g.degree = d;
    g.ids.assign(pruned, pruned + (size_t)n * d);
    ReverseGraph rg = build_reverse_graph(g, cap);
    for (uint32_t y = 0; y < n; ++y) {
      rev_counts[y] = (uint32_t)rg.rows[y].size();
      for (size_t j = 0; j < rg.rows[y].size(); ++j) rev_ids[(size_t)y * cap + j] = rg.rows[y][j];
    }
  });
}

// strong_cc_count / avg_2hop_count (graph_metrics.hpp:22-26), num_threads 0
int ref_graph_metrics(const uint32_t* graph, uint32_t n, uint32_t d, uint64_t* scc,
                      double* avg_2hop) {
  return guard([&] {
    Graph g;
    g.num_nodes = n;
    g.degree = d;
    g.ids.assign(graph, graph + (size_t)n * d);
    *scc = strong_cc_count(g);
    *avg_2hop = avg_2hop_count(g, 0);
  });
}

void* ref_index_create(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                       uint32_t degree) {
  auto* h = new RefIndex{make_ds(data, n, dim), Graph{}};
  h->g.num_nodes = n;
  h->g.degree = degree;
  h->g.ids.assign(graph, graph + (size_t)n * degree);
  return h;
}

void ref_index_destroy(void* h) { delete static_cast<RefIndex*>(h); }

// batch_search through the reference's public API (engine.hpp:38-40).
// Outputs [nq][k], padded 0xffffffff / +inf.
int ref_index_batch_search(void* hv, const float* queries, uint32_t nq, uint32_t dim,
                           const Params* p, uint32_t mode, uint32_t team_count,
                           uint32_t threads, uint32_t* ids, float* dists, uint32_t* counts,
                           Stats* stats) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    Dataset qs = make_ds(queries, nq, dim);
    EngineOptions eo;
    eo.mode = mode ? ExecutionMode::kSharedQueryWorkers : ExecutionMode::kPerQueryWorker;
    eo.team_count = team_count;
    eo.num_threads = threads;
    auto res = batch_search(h->g, h->ds, qs, to_ref(p), eo);
    for (uint32_t qi = 0; qi < nq; ++qi) {
      const auto& r = res[qi];
      counts[qi] = (uint32_t)r.ids.size();
      for (uint32_t j = 0; j < p->k; ++j) {
        ids[(size_t)qi * p->k + j] = j < r.ids.size() ? r.ids[j] : 0xffffffffu;
        dists[(size_t)qi * p->k + j] =
            j < r.ids.size() ? r.dists[j] : std::numeric_limits<float>::infinity();
      }
      if (stats) {
        stats[qi].iterations = r.stats.iterations;
        stats[qi].hash_resets = r.stats.hash_resets;
        stats[qi].distance_evals = r.stats.distance_evals;
        stats[qi].converged = r.stats.converged;
        stats[qi].pad = 0;
      }
    }
  });
}

// search_one (search.hpp:156-157) with params.seed as given.
int ref_index_search_one(void* hv, const float* query, const Params* p, uint32_t* ids,
                         float* dists, uint32_t* count, Stats* st) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    auto r = search_one(h->g, h->ds, std::span<const float>(query, h->ds.dim()), to_ref(p));
    *count = (uint32_t)r.ids.size();
    for (uint32_t j = 0; j < p->k; ++j) {
      ids[j] = j < r.ids.size() ? r.ids[j] : 0xffffffffu;
      dists[j] = j < r.ids.size() ? r.dists[j] : std::numeric_limits<float>::infinity();
    }
    if (st) {
      st->iterations = r.stats.iterations;
      st->hash_resets = r.stats.hash_resets;
      st->distance_evals = r.stats.distance_evals;
      st->converged = r.stats.converged;
      st->pad = 0;
    }
  });
}

// run_benchmark (engine.hpp:59-64): one grid point, warm-up + timed pass
// measured by the reference itself (engine.cpp:150-177).
int ref_index_run_benchmark(void* hv, const float* queries, uint32_t nq, uint32_t dim,
                            const uint32_t* truth, uint32_t truth_k, const Params* p,
                            uint32_t mode, uint32_t team_count, uint32_t threads,
                            double* recall, double* qps, double* mean_iterations) {
  auto* h = static_cast<RefIndex*>(hv);
  return guard([&] {
    Dataset qs = make_ds(queries, nq, dim);
    std::vector<std::vector<uint32_t>> t(nq);
    for (uint32_t qi = 0; qi < nq; ++qi)
      t[qi].assign(truth + (size_t)qi * truth_k, truth + (size_t)(qi + 1) * truth_k);
    EngineOptions eo;
    eo.mode = mode ? ExecutionMode::kSharedQueryWorkers : ExecutionMode::kPerQueryWorker;
    eo.team_count = team_count;
    eo.num_threads = threads;
    auto recs = run_benchmark(h->g, h->ds, qs, t, {to_ref(p)}, eo, "bench");
    *recall = recs[0].recall;
    *qps = recs[0].qps;
    *mean_iterations = recs[0].mean_iterations;
  });
}

uint64_t ref_mix_seed(uint64_t x) { return mix_seed(x); }

// The reference's own fixture generator, testutil::make_uniform_dataset.
int ref_uniform_dataset(uint64_t seed, uint32_t rows, uint32_t dim, float* out) {
  return guard([&] {
    Dataset ds = testutil::make_uniform_dataset(rows, dim, seed);
    std::memcpy(out, ds.raw(), (size_t)rows * dim * 4);
  });
}

unsigned ref_hardware_threads() { return resolve_thread_count(0); }

}  // extern "C"
