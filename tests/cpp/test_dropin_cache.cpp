// The drop-in's device-index cache (host/abi.cpp) must never serve a stale
// copy: an in-place edit of a searched Dataset or Graph is seen by the next
// batch_search / search_one (the reference reads its arguments afresh on every
// call), with the full-content check on by default; with
// CAGRA_INDEX_CACHE=identity the caller promises to call
// fodg::b200::invalidate_index_cache() after such an edit.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "fodg/b200.hpp"
#include "fodg/engine.hpp"
#include "fodg/graph_opt.hpp"
#include "fodg/knn_build.hpp"

static int fails = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

static fodg::Dataset uniform(uint32_t n, uint32_t dim, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> u(0.0f, 1.0f);
  std::vector<float> v((size_t)n * dim);
  for (auto& x : v) x = u(rng);
  return fodg::Dataset(dim, std::move(v));
}

static std::vector<uint32_t> ids_of(const std::vector<fodg::SearchResult>& r) {
  std::vector<uint32_t> out;
  for (const auto& x : r) out.insert(out.end(), x.ids.begin(), x.ids.end());
  return out;
}

int main() {
  const uint32_t n = 4000, dim = 16;
  fodg::Dataset ds = uniform(n, dim, 1), qs = uniform(50, dim, 2);
  fodg::Graph g = fodg::optimize(fodg::exact_knn_graph(ds, 32), 16, fodg::OptimizeOptions{});
  fodg::SearchParams p;
  p.k = 10;
  p.topm = 64;
  p.width = 2;
  p.seed = 3;
  fodg::EngineOptions o;
  for (int identity = 0; identity < 2; ++identity) {
    if (identity) setenv("CAGRA_INDEX_CACHE", "identity", 1);
    auto before = ids_of(fodg::batch_search(g, ds, qs, p, o));
    // move every query's first result far away, in place (same buffer)
    std::vector<float> far(dim, 1000.0f);
    std::vector<uint32_t> moved;
    for (uint32_t q = 0; q < 50; ++q) moved.push_back(before[q * 10]);
    fodg::Dataset edited = ds;  // reference copy with the same edit, fresh buffer
    for (uint32_t id : moved) {
      float* row = const_cast<float*>(ds.row(id).data());
      for (uint32_t d = 0; d < dim; ++d) row[d] = far[d];
      float* row2 = const_cast<float*>(edited.row(id).data());
      for (uint32_t d = 0; d < dim; ++d) row2[d] = far[d];
    }
    if (identity) fodg::b200::invalidate_index_cache();
    auto after = ids_of(fodg::batch_search(g, ds, qs, p, o));
    auto fresh = ids_of(fodg::batch_search(g, edited, qs, p, o));
    EXPECT(after == fresh);
    EXPECT(after != before);
    for (uint32_t q = 0; q < 50; ++q) EXPECT(after[q * 10] != before[q * 10]);
    // a graph edit in place: search_one sees it too
    auto r1 = fodg::search_one(g, ds, qs.row(0), p);
    std::vector<uint32_t> row0(g.ids.begin(), g.ids.begin() + 16);
    for (uint32_t v = 0; v < n; ++v)
      for (uint32_t j = 0; j < 16; ++j) g.ids[(size_t)v * 16 + j] = g.ids[(size_t)v * 16 + (15 - j)];
    if (identity) fodg::b200::invalidate_index_cache();
    auto r2 = fodg::search_one(g, ds, qs.row(0), p);
    fodg::Graph g2 = g;
    auto r3 = fodg::search_one(g2, ds, qs.row(0), p);
    EXPECT(r2.ids == r3.ids);
    EXPECT(r2.stats.distance_evals == r3.stats.distance_evals);
    (void)r1;
    (void)row0;
    ds = uniform(n, dim, 1);
    g = fodg::optimize(fodg::exact_knn_graph(ds, 32), 16, fodg::OptimizeOptions{});
  }
  std::printf("[dropin-cache] %s (%d failures)\n", fails ? "FAIL" : "ok", fails);
  return fails ? 1 : 0;
}
