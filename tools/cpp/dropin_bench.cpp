// The C++ drop-in measured the way a reference user calls it: fodg:: API
// (include/fodg), host std::vector buffers, no CUDA in the caller.
//   dropin_bench [n] [batch] [batch1_queries]
// Prints one JSON object per measurement:
//   * build: exact_knn_graph(ds, 128) + optimize(knn, 64) through the drop-in;
//   * batch: batch_search of `batch` queries, per-query mode, M=896 p=16, in
//     the default reference-order distances and with CAGRA_FAST_DISTANCES=1,
//     standard and forgettable visited policies, with the index cache's
//     full-content check (default) and CAGRA_INDEX_CACHE=identity;
//   * batch 1: sequential single-query batch_search calls, shared mode
//     (choose_mode's pick for batch 1), M=10, 96 teams.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <set>
#include <vector>

#include "cagra/capi.h"
#include "fodg/engine.hpp"
#include "fodg/graph_opt.hpp"
#include "fodg/knn_build.hpp"
#include "fodg/topk.hpp"

using clk = std::chrono::steady_clock;

static fodg::Dataset uniform(uint32_t n, uint32_t dim, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> u(0.0f, 1.0f);
  std::vector<float> v((size_t)n * dim);
  for (auto& x : v) x = u(rng);
  return fodg::Dataset(dim, std::move(v));
}

static double secs(clk::time_point a) {
  return std::chrono::duration<double>(clk::now() - a).count();
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? std::atoi(argv[1]) : 1000000, dim = 96;
  const uint32_t nq = argc > 2 ? std::atoi(argv[2]) : 10000;
  const uint32_t nb = argc > 3 ? std::atoi(argv[3]) : 300;
  fodg::Dataset ds = uniform(n, dim, 424242), qs = uniform(nq, dim, 424243);
  auto t = clk::now();
  fodg::KnnGraph knn = fodg::exact_knn_graph(ds, 128);
  const double knn_s = secs(t);
  t = clk::now();
  fodg::Graph g = fodg::optimize(knn, 64, fodg::OptimizeOptions{});
  const double opt_s = secs(t);
  std::printf("{\"what\": \"build via drop-in\", \"exact_knn_graph_s\": %.3f, \"optimize_s\": %.3f}\n",
              knn_s, opt_s);
  // ground truth: one batched exact top-10 through the C ABI (the drop-in's
  // exact_topk is per query)
  std::vector<uint32_t> gi((size_t)nq * 10);
  std::vector<float> gd((size_t)nq * 10);
  if (cagra_exact_topk(ds.raw(), n, dim, qs.raw(), nq, 10, 0, gi.data(), gd.data()) != CAGRA_OK)
    return 1;
  std::vector<std::set<uint32_t>> truth(nq);
  for (uint32_t q = 0; q < nq; ++q) truth[q] = std::set<uint32_t>(gi.begin() + q * 10, gi.begin() + q * 10 + 10);
  auto recall = [&](const std::vector<fodg::SearchResult>& res, uint32_t off) {
    double h = 0;
    for (size_t i = 0; i < res.size(); ++i)
      for (uint32_t id : res[i].ids) h += truth[off + i].count(id);
    return h / (10.0 * res.size());
  };
  for (int cache = 0; cache < 2; ++cache) {
    if (cache) setenv("CAGRA_INDEX_CACHE", "identity", 1);
    for (int fast = 0; fast < 2; ++fast) {
      setenv("CAGRA_FAST_DISTANCES", fast ? "1" : "0", 1);
      for (int pol = 0; pol < 2; ++pol) {
        fodg::SearchParams p;
        p.k = 10;
        p.topm = 896;
        p.width = 16;
        p.hash_policy = pol ? fodg::HashPolicy::kForgettable : fodg::HashPolicy::kStandard;
        p.hash_bits = 12;
        p.seed = 11;
        fodg::EngineOptions o;
        o.mode = fodg::ExecutionMode::kPerQueryWorker;
        fodg::batch_search(g, ds, qs, p, o);  // warm-up (uploads the index once)
        t = clk::now();
        auto res = fodg::batch_search(g, ds, qs, p, o);
        const double el = secs(t);
        std::printf("{\"what\": \"batch_search %u queries\", \"distances\": \"%s\", \"hash\": \"%s\", "
                    "\"index_cache\": \"%s\", \"qps\": %.0f, \"recall@10\": %.4f}\n",
                    nq, fast ? "fast" : "reference-order", pol ? "forgettable" : "standard",
                    cache ? "identity" : "content-hash", nq / el, recall(res, 0));
      }
    }
    // batch 1: shared mode (choose_mode picks it for one query), fast distances
    setenv("CAGRA_FAST_DISTANCES", "1", 1);
    fodg::SearchParams p1;
    p1.k = 10;
    p1.topm = 10;
    p1.width = 1;
    p1.seed = 11;
    fodg::EngineOptions o1;
    o1.mode = fodg::ExecutionMode::kSharedQueryWorkers;
    o1.team_count = 96;
    std::vector<fodg::SearchResult> out;
    for (uint32_t i = 0; i < nb; ++i) {
      fodg::Dataset one(dim, std::vector<float>(qs.row(i).begin(), qs.row(i).end()));
      if (i == 3) t = clk::now();
      auto r = fodg::batch_search(g, ds, one, p1, o1);
      if (i >= 3) out.push_back(r[0]);
    }
    const double el = secs(t);
    double h = 0;
    for (size_t i = 0; i < out.size(); ++i)
      for (uint32_t id : out[i].ids) h += truth[3 + i].count(id);
    std::printf("{\"what\": \"batch 1 (sequential batch_search of one query)\", \"index_cache\": "
                "\"%s\", \"qps\": %.1f, \"latency_us\": %.1f, \"recall@10\": %.4f}\n",
                cache ? "identity" : "content-hash", out.size() / el, el / out.size() * 1e6,
                h / (10.0 * out.size()));
  }
  return 0;
}
