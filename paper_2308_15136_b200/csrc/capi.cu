// The C-ABI boundary (include/cagra/capi.h): validation in the reference's
// order, device memory management, status-code error mapping.  No CPU
// compute path exists behind any entry point: without a CUDA device every
// compute call fails with CAGRA_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "cagra/capi.h"
#include "common.cuh"
#include "host_util.hpp"
#include "kernels.hpp"

namespace cagra {

std::string& last_error_slot() {
  thread_local std::string err;
  return err;
}

// ---- optimize pipeline on device (graph_opt.cpp:211-246) ----
void optimize_device(const uint32_t* d_knn, const float* d_dists, uint32_t n, uint32_t deg,
                     uint32_t d, bool reorder, bool add_reverse, uint32_t* d_out,
                     cudaStream_t s, OptOut* times) {
  if (d == 0 || d > deg) throw UsageErr("optimize: require 1 <= d <= input degree");
  DBuf flag(sizeof(int));
  int hflag = 0;
  CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  launch_check_ids(d_knn, (uint64_t)n * deg, n, flag.as<int>(), s);
  // rank-mode reordering requires distance-sorted rows (graph_opt.cpp:19-31);
  // plain truncation (reorder = false) does not read distances
  if (reorder) launch_check_sorted(d_knn, d_dists, n, deg, flag.as<int>(), s);
  read_flag(flag.as<int>(), &hflag, s);
  if (hflag & 2) throw UsageErr("optimize: neighbour id out of range");
  if (hflag & 1) throw UsageErr("graph_opt: input rows must be distance-sorted");
  Event e0, e1, e2, e3, e4;
  // every scratch buffer is allocated before the first event, so the stage
  // times are device time, not host allocation time
  DBuf pruned(sizeof(uint32_t) * (size_t)n * d);
  DBuf scratch(add_reverse ? reverse_scratch_bytes(n, d) : 0);
  DBuf rc(add_reverse ? sizeof(uint32_t) * n : 0), ri(add_reverse ? sizeof(uint32_t) * (size_t)n * d : 0);
  CAGRA_CUDA_TRY(cudaEventRecord(e0.e, s));
  if (reorder) {
    launch_detour_reorder(d_knn, n, deg, d, nullptr, pruned.as<uint32_t>(), s);
  } else {
    CAGRA_CUDA_TRY(cudaMemcpy2DAsync(pruned.p, sizeof(uint32_t) * d, d_knn, sizeof(uint32_t) * deg,
                                     sizeof(uint32_t) * d, n, cudaMemcpyDeviceToDevice, s));
  }
  CAGRA_CUDA_TRY(cudaEventRecord(e1.e, s));
  if (add_reverse) {
    launch_reverse(pruned.as<uint32_t>(), n, d, d, scratch.p, rc.as<uint32_t>(), ri.as<uint32_t>(),
                   s);
    CAGRA_CUDA_TRY(cudaEventRecord(e2.e, s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    launch_merge(pruned.as<uint32_t>(), rc.as<uint32_t>(), ri.as<uint32_t>(), n, d, d, d_out,
                 flag.as<int>(), s);
    CAGRA_CUDA_TRY(cudaEventRecord(e3.e, s));
    read_flag(flag.as<int>(), &hflag, s);
    if (hflag & 4) throw UsageErr("merge_graphs: fewer than d distinct candidates");
  } else {
    CAGRA_CUDA_TRY(cudaMemcpyAsync(d_out, pruned.p, sizeof(uint32_t) * (size_t)n * d,
                                   cudaMemcpyDeviceToDevice, s));
    CAGRA_CUDA_TRY(cudaEventRecord(e2.e, s));
    CAGRA_CUDA_TRY(cudaEventRecord(e3.e, s));
  }
  CAGRA_CUDA_TRY(cudaEventRecord(e4.e, s));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  if (times) {
    cudaEventElapsedTime(&times->ms[0], e0.e, e1.e);  // count + reorder (fused)
    times->ms[1] = 0;
    cudaEventElapsedTime(&times->ms[2], e1.e, e2.e);
    cudaEventElapsedTime(&times->ms[3], e2.e, e3.e);
    cudaEventElapsedTime(&times->ms[4], e0.e, e4.e);
  }
}

}  // namespace cagra

using namespace cagra;

// ============================================================ the index ====
struct cagra_index {
  int device = 0;
  int sm_count = 148;
  uint32_t n = 0, dim = 0, ld = 0, degree = 0;
  DBuf data, graph;
  Stream* stream = nullptr;
  std::mutex mu;
  // persistent visited-table arena (generation tagged)
  DBuf tables, gens;
  size_t table_elems = 0;
  uint32_t table_hcap = 0, table_grid = 0;
  // per-call scratch
  DBuf init_ids, work, q, ids, dists, counts, stats, team_out, team_stats;
  uint32_t last_launches = 0;
  uint32_t mc_tag = 0;        // generation of the multi-CTA per-query tables
  SearchPlan plan;            // cached plan for (plan_cfg, plan_nq)
  SearchConfig plan_cfg{};
  uint32_t plan_nq = 0;
  bool plan_valid = false;
  int mc_layout = 0;          // tables laid out: 0 per CTA, 1 per query (generic
                              // multi-CTA), 2 per query x 2 regions (batch-1 kernel),
                              // 3 per-CTA visited bitmaps (standard policy)
  DBuf b1_ctr;                // batch-1 kernel: teams finished per query (zeroed)
  // Completion of the last search issued on this index, on whatever stream
  // it ran.  Every search first makes its stream wait on it and records it
  // again at the end, so calls on different streams (cagra_search on the
  // private stream, cagra_search_dev on caller streams) never overlap on the
  // per-index scratch, and a scratch buffer is only reallocated once the
  // work that used it has finished (grow()).
  cudaEvent_t done = nullptr;
  ~cagra_index() {
    if (done) cudaEventDestroy(done);
    delete stream;
  }
};

namespace {

// A host pointer the device can dereference directly (pinned memory mapped
// into the unified address space: the same address on both sides).
bool host_mapped(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// Grows a per-index scratch buffer after the index's previous search is done.
void grow(cagra_index* ix, DBuf& b, size_t bytes) {
  if (bytes <= b.bytes) return;
  CAGRA_CUDA_TRY(cudaEventSynchronize(ix->done));
  b.alloc(bytes);
}

// Orders this call's work on `s` after every earlier search on the index.
void begin_on(cagra_index* ix, cudaStream_t s) {
  CAGRA_CUDA_TRY(cudaStreamWaitEvent(s, ix->done, 0));
}
void end_on(cagra_index* ix, cudaStream_t s) { CAGRA_CUDA_TRY(cudaEventRecord(ix->done, s)); }

void validate_params(const cagra_search_params* p) {
  // SearchParams::validate (search.cpp:39-50), same order
  if (p->k == 0) throw UsageErr("search: k must be >= 1");
  if (p->k > p->topm) throw UsageErr("search: require k <= M");
  if (p->width == 0) throw UsageErr("search: p must be >= 1");
  uint32_t it = p->max_iterations;
  if (!it) {
    it = (2 * p->topm + p->width - 1) / p->width;
    it = it < 16 ? 16 : (it > 256 ? 256 : it);
  }
  if (p->min_iterations > it) throw UsageErr("search: min_iterations exceeds max_iterations");
  if (p->hash_policy == CAGRA_HASH_FORGETTABLE) {
    if (p->hash_bits < 4 || p->hash_bits > 24)
      throw UsageErr("search: forgettable hash_bits out of range");
    if (p->reset_interval == 0) throw UsageErr("search: reset_interval must be >= 1");
  }
}

SearchConfig to_config(const cagra_search_params* p, const cagra_engine_opts* o) {
  SearchConfig c{};  // zeroed padding: the plan cache compares configs bytewise
  c.k = p->k;
  c.topm = p->topm;
  c.width = p->width;
  c.max_iter = p->max_iterations;
  c.min_iter = p->min_iterations;
  c.hash_policy = p->hash_policy;
  c.hash_bits = p->hash_bits;
  c.reset_interval = p->reset_interval;
  c.seed = p->seed;
  c.mode = o->mode;
  c.team_count = o->team_count;
  c.seed_mode = o->seed_mode;
  c.exact = o->exact_distances;
  c.team_size = o->team_size;
  c.query_offset = o->query_offset;
  c.multi_cta = o->multi_cta;
  return c;
}

constexpr size_t kTableBudget = 8ull << 30;

// kTableBudget, or CAGRA_TABLE_BUDGET_MB (tests exercise the chunked paths)
size_t table_budget() {
  const char* e = std::getenv("CAGRA_TABLE_BUDGET_MB");
  return e && *e ? (size_t)std::strtoull(e, nullptr, 10) << 20 : kTableBudget;
}

// Runs a search on device-resident queries (rows of ix->ld floats).
void run_search(cagra_index* ix, const float* d_queries, uint32_t nq,
                const cagra_search_params* params, const cagra_engine_opts* opts,
                uint32_t* d_ids, float* d_dists, uint32_t* d_counts, void* d_stats,
                cudaStream_t s) {
  DeviceIndexView v{ix->data.as<float>(), ix->graph.as<uint32_t>(), ix->n, ix->dim, ix->ld,
                    ix->degree};
  SearchConfig c = to_config(params, opts);
  if (c.mode == 1 && !c.exact && c.multi_cta == 2 && nq > 1) {
    // forced multi-CTA on a large batch: chunks whose per-query visited
    // regions fit the table budget (query_offset keeps the seeds global)
    const uint64_t maxq =
        std::max<uint64_t>(1, table_budget() / mc_table_bytes_per_query(c, ix->degree));
    if (nq > maxq) {
      const size_t k = params->k;
      cagra_engine_opts o = *opts;
      for (uint64_t off = 0; off < nq; off += maxq) {
        const uint32_t m = (uint32_t)std::min<uint64_t>(maxq, nq - off);
        o.query_offset = opts->query_offset + off;
        run_search(ix, d_queries + off * ix->ld, m, params, &o, d_ids + off * k,
                   d_dists + off * k, d_counts ? d_counts + off : nullptr,
                   d_stats ? static_cast<cagra_search_stats*>(d_stats) + off : nullptr, s);
      }
      return;
    }
  }
  // the plan (kernel variant, grid, smem, table sizes) depends only on the
  // configuration and the batch size: reuse it across repeated calls
  // (batch-1 loops) instead of re-querying attributes and occupancy
  if (!ix->plan_valid || ix->plan_nq != nq ||
      std::memcmp(&ix->plan_cfg, &c, sizeof(SearchConfig)) != 0) {
    ix->plan = plan_search(v, c, nq, ix->sm_count, table_budget());
    ix->plan_cfg = c;
    ix->plan_nq = nq;
    ix->plan_valid = true;
  }
  const SearchPlan& pl = ix->plan;
  grow(ix, ix->init_ids, sizeof(uint32_t) * std::max<size_t>(pl.init_elems, 1));
  grow(ix, ix->work, sizeof(uint32_t));
  if (pl.mc) {
    grow(ix, ix->team_out, sizeof(unsigned long long) * std::max<size_t>(pl.team_elems, 1));
    grow(ix, ix->team_stats, sizeof(cagra_search_stats) * (size_t)nq * pl.teams);
    // per-query regions tagged by a call generation; a new layout starts clean
    const int kind = pl.b1 ? 2 : 1;
    // (the fused kernel's regions are nq * hcap words: a new nq is a new layout,
    // since each call clears the other region at the current layout)
    if (ix->mc_layout != kind || pl.hcap != ix->table_hcap || pl.table_elems > ix->table_elems ||
        (pl.b1 && pl.grid != ix->table_grid) || ix->mc_tag == 0xffffffffu) {
      if (pl.table_elems > ix->table_elems) {
        grow(ix, ix->tables, sizeof(unsigned long long) * pl.table_elems);
        ix->table_elems = pl.table_elems;
      }
      CAGRA_CUDA_TRY(cudaMemsetAsync(ix->tables.p, 0, ix->tables.bytes, s));
      ix->mc_tag = 0;
      ix->table_hcap = pl.hcap;
      ix->table_grid = pl.b1 ? pl.grid : 0;  // per-CTA generations no longer match
      grow(ix, ix->gens, sizeof(uint32_t) * std::max<uint32_t>(pl.grid, 1));
      CAGRA_CUDA_TRY(cudaMemsetAsync(ix->gens.p, 0, ix->gens.bytes, s));
      ix->mc_layout = kind;
    }
    if (pl.b1 && ix->b1_ctr.bytes < sizeof(uint32_t) * nq) {
      grow(ix, ix->b1_ctr, sizeof(uint32_t) * nq);
      CAGRA_CUDA_TRY(cudaMemsetAsync(ix->b1_ctr.p, 0, ix->b1_ctr.bytes, s));
    }
    ix->mc_tag++;
    grow(ix, ix->gens, sizeof(uint32_t) * pl.grid);
  } else if (pl.bitmap) {
    // per-CTA bitmaps, cleared by the kernel at every query: no tags to keep
    if (pl.table_elems > ix->table_elems) {
      grow(ix, ix->tables, sizeof(unsigned long long) * pl.table_elems);
      ix->table_elems = pl.table_elems;
    }
    grow(ix, ix->gens, sizeof(uint32_t) * std::max<uint32_t>(pl.grid, 1));
    ix->mc_layout = 3;
  } else if (pl.table_elems) {
    bool relayout = ix->mc_layout != 0 || pl.hcap != ix->table_hcap || pl.grid > ix->table_grid ||
                    pl.table_elems > ix->table_elems;
    if (relayout) {
      // a changed layout would alias old tags into other slots: start clean
      if (pl.table_elems > ix->table_elems) {
        grow(ix, ix->tables, sizeof(unsigned long long) * pl.table_elems);
        ix->table_elems = pl.table_elems;
      }
      grow(ix, ix->gens, sizeof(uint32_t) * std::max<uint32_t>(pl.grid, ix->table_grid));
      CAGRA_CUDA_TRY(cudaMemsetAsync(ix->tables.p, 0, ix->tables.bytes, s));
      CAGRA_CUDA_TRY(cudaMemsetAsync(ix->gens.p, 0, ix->gens.bytes, s));
      ix->table_hcap = pl.hcap;
      ix->table_grid = std::max(pl.grid, ix->table_grid);
      ix->mc_layout = 0;
    }
  } else {
    grow(ix, ix->gens, sizeof(uint32_t) * pl.grid);
  }
  ix->last_launches = launch_search(v, c, pl, d_queries, nq, d_ids, d_dists, d_counts, d_stats,
                                    ix->init_ids.as<uint32_t>(), ix->work.as<uint32_t>(),
                                    ix->tables.as<unsigned long long>(), ix->gens.as<uint32_t>(),
                                    ix->team_out.as<unsigned long long>(), ix->team_stats.p,
                                    ix->mc_tag, s, ix->b1_ctr.as<uint32_t>());
}

}  // namespace

extern "C" {

const char* cagra_last_error(void) { return last_error_slot().c_str(); }

const char* cagra_version(void) { return "cagra-b200 0.1 (sm_100a)"; }

int cagra_device_count(int* out) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  cudaGetLastError();
  *out = c;
  return CAGRA_OK;
}

void cagra_search_params_default(cagra_search_params* p) {
  p->k = 10;
  p->topm = 64;
  p->width = 1;
  p->max_iterations = 0;
  p->min_iterations = 1;
  p->hash_policy = CAGRA_HASH_STANDARD;
  p->hash_bits = 11;
  p->reset_interval = 1;
  p->seed = 0;
}

void cagra_engine_opts_default(cagra_engine_opts* o) {
  o->multi_cta = 0;
  o->_pad = 0;
  o->mode = CAGRA_MODE_PER_QUERY;
  o->team_count = 4;
  o->num_threads = 0;
  o->seed_mode = 0;
  o->query_offset = 0;
  o->exact_distances = 0;
  o->team_size = 0;
}

uint64_t cagra_mix_seed(uint64_t x) { return mix_seed(x); }

int cagra_uniform_dataset(uint64_t seed, uint64_t count, float* out) {
  // tests/test_util.hpp:11-18 (libstdc++ mt19937_64 + uniform_real_distribution)
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> dist(0.0f, 1.0f);
    for (uint64_t i = 0; i < count; ++i) out[i] = dist(rng);
  });
}

int cagra_exact_knn_graph(const float* data, uint32_t n, uint32_t dim, uint32_t k, int device,
                          uint32_t* ids_out, float* dists_out) {
  return guarded([&] {
    if (k == 0 || k >= n) throw UsageErr("exact_knn_graph: require 1 <= k < N");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    uint32_t ld = row_stride(dim);
    DBuf dd(sizeof(float) * (size_t)n * ld),
        di(sizeof(uint32_t) * (size_t)n * k), ds(sizeof(float) * (size_t)n * k);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    launch_exact_topk(dd.as<float>(), n, ld, dd.as<float>(), n, ld, dim, k, true,
                      di.as<uint32_t>(), ds.as<float>(), st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, di.p, sizeof(uint32_t) * (size_t)n * k,
                                   cudaMemcpyDeviceToHost, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, ds.p, sizeof(float) * (size_t)n * k,
                                   cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_nn_descent(const float* data, uint32_t n, uint32_t dim, uint32_t k, double sample_rate,
                     double termination_delta, uint32_t max_rounds, uint64_t seed, int device,
                     uint32_t* ids_out, float* dists_out, uint32_t* converged_out,
                     uint32_t* rounds_out) {
  return guarded([&] {
    // knn_build.cpp:97-102, same order
    if (k == 0 || k >= n) throw UsageErr("nn_descent: require 1 <= k < N");
    if (!(sample_rate > 0.0 && sample_rate <= 1.0))
      throw UsageErr("nn_descent: sample_rate must be in (0, 1]");
    if (!(termination_delta > 0.0 && termination_delta < 1.0))
      throw UsageErr("nn_descent: termination_delta must be in (0, 1)");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    const uint32_t ld = row_stride(dim);
    DBuf dd(sizeof(float) * (size_t)n * ld), di(sizeof(uint32_t) * (size_t)n * k),
        ds(sizeof(float) * (size_t)n * k);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    const NnDescentInfo info =
        launch_nn_descent(dd.as<float>(), n, ld, dim, k, sample_rate, termination_delta,
                          max_rounds, seed, di.as<uint32_t>(), ds.as<float>(), st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, di.p, sizeof(uint32_t) * (size_t)n * k,
                                   cudaMemcpyDeviceToHost, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, ds.p, sizeof(float) * (size_t)n * k,
                                   cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (converged_out) *converged_out = info.converged ? 1u : 0u;
    if (rounds_out) *rounds_out = info.rounds;
  });
}

int cagra_exact_knn_rows(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                         uint32_t row_begin, uint32_t row_end, int device, uint32_t* ids_out,
                         float* dists_out) {
  return guarded([&] {
    if (k == 0 || k >= n) throw UsageErr("exact_knn_graph: require 1 <= k < N");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    if (row_begin > row_end || row_end > n) throw UsageErr("kNN rows: range outside [0, N]");
    const uint32_t cnt = row_end - row_begin;
    if (cnt == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    uint32_t ld = row_stride(dim);
    DBuf dd(sizeof(float) * (size_t)n * ld), di(sizeof(uint32_t) * (size_t)cnt * k),
        ds(sizeof(float) * (size_t)cnt * k);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    launch_exact_topk(dd.as<float>(), n, ld, dd.as<float>() + (size_t)row_begin * ld, cnt, ld,
                      dim, k, true, di.as<uint32_t>(), ds.as<float>(), st.s, row_begin);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, di.p, sizeof(uint32_t) * (size_t)cnt * k,
                                   cudaMemcpyDeviceToHost, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, ds.p, sizeof(float) * (size_t)cnt * k,
                                   cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_exact_topk(const float* data, uint32_t n, uint32_t dim, const float* queries,
                     uint32_t nq, uint32_t k, int device, uint32_t* ids_out, float* dists_out) {
  return guarded([&] {
    if (k == 0 || k > n) throw UsageErr("exact_topk: k out of range [1, N]");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    if (nq == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    uint32_t ld = row_stride(dim);
    DBuf dd(sizeof(float) * (size_t)n * ld), dq(sizeof(float) * (size_t)nq * ld),
        di(sizeof(uint32_t) * (size_t)nq * k),
        ds(sizeof(float) * (size_t)nq * k);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    upload_rows(dq.as<float>(), queries, nq, dim, ld, st.s);
    launch_exact_topk(dd.as<float>(), n, ld, dq.as<float>(), nq, ld, dim, k, false,
                      di.as<uint32_t>(), ds.as<float>(), st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, di.p, sizeof(uint32_t) * (size_t)nq * k,
                                   cudaMemcpyDeviceToHost, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, ds.p, sizeof(float) * (size_t)nq * k,
                                   cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_knn_last_filter(uint32_t* split_terms, uint32_t* gemm_k) {
  if (split_terms) *split_terms = g_knn_tc_stats.split_terms;
  if (gemm_k) *gemm_k = g_knn_tc_stats.gemm_k;
  return CAGRA_OK;
}

int cagra_trim_scratch(int device) {
  return guarded([&] { knn_trim_scratch(device); });
}

int cagra_knn_last_stats(uint64_t* rows, uint64_t* fallback_rows, uint64_t* reranked,
                         uint64_t* retried_rows) {
  if (retried_rows) *retried_rows = g_knn_tc_stats.retried_rows;
  if (rows) *rows = g_knn_tc_stats.rows;
  if (fallback_rows) *fallback_rows = g_knn_tc_stats.fallback_rows;
  if (reranked) *reranked = g_knn_tc_stats.reranked;
  return CAGRA_OK;
}

int cagra_count_detourable_routes(const uint32_t* knn_ids, const float* knn_dists, uint32_t n,
                                  uint32_t deg, int device, uint32_t* counts_out) {
  return guarded([&] {
    if (n == 0 || deg == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    size_t e = (size_t)n * deg;
    DBuf di(4 * e), dd(4 * e), dc(4 * e), flag(sizeof(int));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(di.p, knn_ids, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dd.p, knn_dists, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st.s));
    launch_check_sorted(di.as<uint32_t>(), dd.as<float>(), n, deg, flag.as<int>(), st.s);
    launch_check_ids(di.as<uint32_t>(), e, n, flag.as<int>(), st.s);
    int h = 0;
    read_flag(flag.as<int>(), &h, st.s);
    if (h & 1) throw UsageErr("graph_opt: input rows must be distance-sorted");
    if (h & 2) throw UsageErr("count_detourable_routes: neighbour id out of range");
    launch_detour_reorder(di.as<uint32_t>(), n, deg, 0, dc.as<uint32_t>(), nullptr, st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(counts_out, dc.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_count_detourable_routes_distance(const uint32_t* knn_ids, const float* knn_dists,
                                           uint32_t n, uint32_t deg, const float* data,
                                           uint32_t ds_n, uint32_t dim, int device,
                                           uint32_t* counts_out) {
  return guarded([&] {
    if (n == 0 || deg == 0) return;
    // graph_opt.cpp:45-51: sortedness first, then the dataset checks
    if (!knn_dists) throw UsageErr("graph_opt: input rows have no distances");
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    size_t e = (size_t)n * deg;
    DBuf di(4 * e), dd(4 * e), dc(4 * e), flag(sizeof(int));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(di.p, knn_ids, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dd.p, knn_dists, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st.s));
    launch_check_sorted(di.as<uint32_t>(), dd.as<float>(), n, deg, flag.as<int>(), st.s);
    launch_check_ids(di.as<uint32_t>(), e, n, flag.as<int>(), st.s);
    int h = 0;
    read_flag(flag.as<int>(), &h, st.s);
    if (h & 1) throw UsageErr("graph_opt: input rows must be distance-sorted");
    if (!data) throw UsageErr("count_detourable_routes: distance mode requires the dataset");
    if (ds_n != n) throw UsageErr("count_detourable_routes: dataset/graph size mismatch");
    if (h & 2) throw UsageErr("graph_opt: neighbour id out of range");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    const uint32_t ld = row_stride(dim);
    DBuf dx(sizeof(float) * (size_t)n * ld);
    upload_rows(dx.as<float>(), data, n, dim, ld, st.s);
    launch_detour_distance(di.as<uint32_t>(), n, deg, dx.as<float>(), ld, dim, dc.as<uint32_t>(),
                           st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(counts_out, dc.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_reorder_and_prune(const uint32_t* knn_ids, const uint32_t* counts, uint32_t n,
                            uint32_t deg, uint32_t d, int device, uint32_t* pruned_out) {
  return guarded([&] {
    if (d == 0 || d > deg) throw UsageErr("reorder_and_prune: require 1 <= d <= input degree");
    if (n == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    size_t e = (size_t)n * deg;
    DBuf di(4 * e), dc(4 * e), dp(4ull * n * d);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(di.p, knn_ids, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dc.p, counts, 4 * e, cudaMemcpyHostToDevice, st.s));
    launch_reorder_from_counts(di.as<uint32_t>(), dc.as<uint32_t>(), n, deg, d,
                               dp.as<uint32_t>(), st.s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(pruned_out, dp.p, 4ull * n * d, cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_build_reverse_graph(const uint32_t* pruned, uint32_t n, uint32_t d, uint32_t cap,
                              int device, uint32_t* rev_counts_out, uint32_t* rev_ids_out) {
  return guarded([&] {
    if (n == 0 || d == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    size_t e = (size_t)n * d;
    cap = std::min(cap, n);  // no row holds more than n sources: larger caps mean "no cap"
    DBuf dp(4 * e), flag(sizeof(int)), sc(reverse_scratch_bytes(n, d)), rc(4ull * n),
        ri(4ull * n * std::max(cap, 1u));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dp.p, pruned, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st.s));
    launch_check_ids(dp.as<uint32_t>(), e, n, flag.as<int>(), st.s);
    int h = 0;
    read_flag(flag.as<int>(), &h, st.s);
    if (h) throw UsageErr("build_reverse_graph: neighbour id out of range");
    CAGRA_CUDA_TRY(cudaMemsetAsync(ri.p, 0xff, ri.bytes, st.s));
    if (cap > 0)
      launch_reverse(dp.as<uint32_t>(), n, d, cap, sc.p, rc.as<uint32_t>(), ri.as<uint32_t>(), st.s);
    else
      CAGRA_CUDA_TRY(cudaMemsetAsync(rc.p, 0, 4ull * n, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(rev_counts_out, rc.p, 4ull * n, cudaMemcpyDeviceToHost, st.s));
    if (cap > 0)
      CAGRA_CUDA_TRY(
          cudaMemcpyAsync(rev_ids_out, ri.p, 4ull * n * cap, cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_graph_metrics(const uint32_t* graph, uint32_t n, uint32_t degree, int device,
                        uint64_t* strong_cc, uint64_t* two_hop) {
  return guarded([&] {
    if (strong_cc) *strong_cc = 0;
    if (two_hop) *two_hop = 0;
    if (n == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    const size_t e = (size_t)n * degree;
    DBuf dg(4 * e), flag(sizeof(int));
    if (e) CAGRA_CUDA_TRY(cudaMemcpyAsync(dg.p, graph, 4 * e, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st.s));
    if (e) launch_check_ids(dg.as<uint32_t>(), e, n, flag.as<int>(), st.s);
    int h = 0;
    read_flag(flag.as<int>(), &h, st.s);
    if (h & 2) throw UsageErr("graph_metrics: neighbour id out of range");
    if (strong_cc) *strong_cc = scc_count(dg.as<uint32_t>(), n, degree, st.s);
    if (two_hop) *two_hop = two_hop_total(dg.as<uint32_t>(), n, degree, sm_count_of(dev), st.s);
  });
}

int cagra_merge_graphs(const uint32_t* pruned, const uint32_t* rev_counts,
                       const uint32_t* rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
                       int device, uint32_t* graph_out) {
  return guarded([&] {
    if (n == 0 || d == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    DBuf dp(4ull * n * d), rc(4ull * n), ri(4ull * n * std::max(rev_cap, 1u)),
        out(4ull * n * d), flag(sizeof(int));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dp.p, pruned, 4ull * n * d, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(rc.p, rev_counts, 4ull * n, cudaMemcpyHostToDevice, st.s));
    if (rev_cap)
      CAGRA_CUDA_TRY(
          cudaMemcpyAsync(ri.p, rev_ids, 4ull * n * rev_cap, cudaMemcpyHostToDevice, st.s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st.s));
    launch_merge(dp.as<uint32_t>(), rc.as<uint32_t>(), ri.as<uint32_t>(), n, d, rev_cap,
                 out.as<uint32_t>(), flag.as<int>(), st.s);
    int h = 0;
    read_flag(flag.as<int>(), &h, st.s);
    if (h & 4) throw UsageErr("merge_graphs: fewer than d distinct candidates");
    CAGRA_CUDA_TRY(cudaMemcpyAsync(graph_out, out.p, 4ull * n * d, cudaMemcpyDeviceToHost, st.s));
    st.sync();
  });
}

int cagra_optimize(const uint32_t* knn_ids, const float* knn_dists, uint32_t n, uint32_t deg,
                   uint32_t d, uint32_t reorder, uint32_t add_reverse, int device,
                   uint32_t* graph_out, cagra_opt_stats* stats) {
  return guarded([&] {
    if (d == 0 || d > deg) throw UsageErr("optimize: require 1 <= d <= input degree");
    if (n == 0) return;
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    size_t e = (size_t)n * deg;
    DBuf di(4 * e), dd(4 * e), out(4ull * n * d);
    if (reorder && !knn_dists) throw UsageErr("graph_opt: input rows have no distances");
    CAGRA_CUDA_TRY(cudaMemcpyAsync(di.p, knn_ids, 4 * e, cudaMemcpyHostToDevice, st.s));
    if (knn_dists)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(dd.p, knn_dists, 4 * e, cudaMemcpyHostToDevice, st.s));
    OptOut t;
    optimize_device(di.as<uint32_t>(), dd.as<float>(), n, deg, d, reorder != 0, add_reverse != 0,
                    out.as<uint32_t>(), st.s, &t);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(graph_out, out.p, 4ull * n * d, cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (stats) {
      stats->count_seconds = t.ms[0] * 1e-3;
      stats->reorder_seconds = t.ms[1] * 1e-3;
      stats->reverse_seconds = t.ms[2] * 1e-3;
      stats->merge_seconds = t.ms[3] * 1e-3;
      stats->total_seconds = t.ms[4] * 1e-3;
    }
  });
}

int cagra_build_graph(const float* data, uint32_t n, uint32_t dim, uint32_t d_init, uint32_t d,
                      int device, uint32_t* graph_out, uint32_t* knn_ids_out,
                      float* knn_dists_out, double* seconds_out) {
  return guarded([&] {
    if (d_init == 0 || d_init >= n) throw UsageErr("exact_knn_graph: require 1 <= k < N");
    if (d == 0 || d > d_init) throw UsageErr("optimize: require 1 <= d <= input degree");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    Stream st;
    uint32_t ld = row_stride(dim);
    size_t e = (size_t)n * d_init;
    DBuf dd(sizeof(float) * (size_t)n * ld), di(4 * e), ds(4 * e), out(4ull * n * d);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    Event a, b;
    CAGRA_CUDA_TRY(cudaEventRecord(a.e, st.s));
    {
      launch_exact_topk(dd.as<float>(), n, ld, dd.as<float>(), n, ld, dim, d_init, true,
                        di.as<uint32_t>(), ds.as<float>(), st.s);
      CAGRA_CUDA_TRY(cudaEventRecord(b.e, st.s));
      st.sync();
    }
    OptOut t;
    optimize_device(di.as<uint32_t>(), ds.as<float>(), n, d_init, d, true, true,
                    out.as<uint32_t>(), st.s, &t);
    float knn_ms = 0;
    cudaEventElapsedTime(&knn_ms, a.e, b.e);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(graph_out, out.p, 4ull * n * d, cudaMemcpyDeviceToHost, st.s));
    if (knn_ids_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(knn_ids_out, di.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    if (knn_dists_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(knn_dists_out, ds.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (seconds_out) {
      seconds_out[0] = knn_ms * 1e-3;
      seconds_out[1] = t.ms[4] * 1e-3;
    }
  });
}

static void create_index(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                         uint32_t degree, int device, bool from_device, cagra_index** out) {
  if (n == 0 || dim == 0) throw UsageErr("index: empty dataset");
  if (degree == 0) throw FormatErr("graph: empty");
  if ((uint64_t)n > kMaxNodes) throw UsageErr("dataset exceeds 2^31 - 1 vectors");
  int dev = resolve_device(device);
  DeviceScope scope(dev);
  auto* ix = new cagra_index();
  try {
    ix->device = dev;
    ix->sm_count = sm_count_of(dev);
    ix->n = n;
    ix->dim = dim;
    ix->ld = row_stride(dim);
    ix->degree = degree;
    ix->stream = new Stream();
    CAGRA_CUDA_TRY(cudaEventCreateWithFlags(&ix->done, cudaEventDisableTiming));
    cudaStream_t s = ix->stream->s;
    ix->data.alloc(sizeof(float) * (size_t)n * ix->ld);
    ix->graph.alloc(sizeof(uint32_t) * (size_t)n * degree);
    upload_rows(ix->data.as<float>(), data, n, dim, ix->ld, s, from_device);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ix->graph.p, graph, sizeof(uint32_t) * (size_t)n * degree,
                                   from_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                   s));
    DBuf flag(sizeof(int));
    CAGRA_CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    launch_check_ids(ix->graph.as<uint32_t>(), (uint64_t)n * degree, n, flag.as<int>(), s);
    int h = 0;
    read_flag(flag.as<int>(), &h, s);
    if (h) throw UsageErr("search: graph/dataset size mismatch (neighbour id out of range)");
    end_on(ix, s);
  } catch (...) {
    delete ix;
    throw;
  }
  *out = ix;
}

int cagra_index_create(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                       uint32_t degree, int device, cagra_index** out) {
  return guarded([&] { create_index(data, n, dim, graph, degree, device, false, out); });
}

int cagra_index_create_dev(const float* d_data, uint32_t n, uint32_t dim,
                           const uint32_t* d_graph, uint32_t degree, int device,
                           cagra_index** out) {
  return guarded([&] { create_index(d_data, n, dim, d_graph, degree, device, true, out); });
}

int cagra_index_destroy(cagra_index* index) {
  return guarded([&] {
    if (!index) return;
    DeviceScope scope(index->device);
    delete index;
  });
}

int cagra_index_info(const cagra_index* index, uint32_t* n, uint32_t* dim, uint32_t* degree,
                     int* device) {
  return guarded([&] {
    if (!index) throw UsageErr("null index");
    if (n) *n = index->n;
    if (dim) *dim = index->dim;
    if (degree) *degree = index->degree;
    if (device) *device = index->device;
  });
}

uint32_t cagra_index_row_stride(const cagra_index* index) { return index ? index->ld : 0; }

int cagra_search(cagra_index* ix, const float* queries, uint32_t nq, uint32_t dim,
                 const cagra_search_params* params, const cagra_engine_opts* opts,
                 uint32_t* ids_out, float* dists_out, uint32_t* counts_out,
                 cagra_search_stats* stats_out) {
  return guarded([&] {
    if (!ix) throw UsageErr("null index");
    // batch_search validation order, engine.cpp:98-102
    if (nq == 0) return;
    if (dim != ix->dim) throw UsageErr("batch_search: query dimension mismatch");
    validate_params(params);
    cagra_engine_opts def;
    cagra_engine_opts_default(&def);
    const cagra_engine_opts* o = opts ? opts : &def;
    if (o->mode == CAGRA_MODE_SHARED && o->team_count < 2)
      throw UsageErr("batch_search: shared mode requires team_count >= 2");
    std::lock_guard<std::mutex> lock(ix->mu);
    DeviceScope scope(ix->device);
    cudaStream_t s = ix->stream->s;
    const uint32_t k = params->k;
    begin_on(ix, s);
    // Small batches whose host buffers are device-accessible (pinned,
    // cudaHostAlloc'd: mapped under UVA) skip the staging copies: the kernels
    // read the query rows once per CTA and write the k results once, straight
    // over PCIe/C2C (the batch-1 latency path: one launch, no memcpy).
    if (nq <= 64 && dim == ix->ld && host_mapped(queries) && host_mapped(ids_out) &&
        host_mapped(dists_out) && (!counts_out || host_mapped(counts_out)) &&
        (!stats_out || host_mapped(stats_out))) {
      uint32_t* counts = counts_out;
      if (!counts) {
        grow(ix, ix->counts, sizeof(uint32_t) * nq);
        counts = ix->counts.as<uint32_t>();
      }
      run_search(ix, queries, nq, params, o, ids_out, dists_out, counts, stats_out, s);
      end_on(ix, s);
      CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
      return;
    }
    grow(ix, ix->q, sizeof(float) * (size_t)nq * ix->ld);
    grow(ix, ix->ids, sizeof(uint32_t) * (size_t)nq * k);
    grow(ix, ix->dists, sizeof(float) * (size_t)nq * k);
    grow(ix, ix->counts, sizeof(uint32_t) * nq);
    grow(ix, ix->stats, sizeof(cagra_search_stats) * nq);
    upload_rows(ix->q.as<float>(), queries, nq, dim, ix->ld, s);
    run_search(ix, ix->q.as<float>(), nq, params, o, ix->ids.as<uint32_t>(),
               ix->dists.as<float>(), ix->counts.as<uint32_t>(), ix->stats.p, s);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, ix->ids.p, sizeof(uint32_t) * (size_t)nq * k,
                                   cudaMemcpyDeviceToHost, s));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, ix->dists.p, sizeof(float) * (size_t)nq * k,
                                   cudaMemcpyDeviceToHost, s));
    if (counts_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(counts_out, ix->counts.p, sizeof(uint32_t) * nq,
                                     cudaMemcpyDeviceToHost, s));
    if (stats_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(stats_out, ix->stats.p, sizeof(cagra_search_stats) * nq,
                                     cudaMemcpyDeviceToHost, s));
    end_on(ix, s);
    CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  });
}

int cagra_search_dev(cagra_index* ix, const float* d_queries, uint32_t nq,
                     const cagra_search_params* params, const cagra_engine_opts* opts,
                     uint32_t* d_ids_out, float* d_dists_out, uint32_t* d_counts_out,
                     cagra_search_stats* d_stats_out, void* stream) {
  return guarded([&] {
    if (!ix) throw UsageErr("null index");
    if (nq == 0) return;
    validate_params(params);
    cagra_engine_opts def;
    cagra_engine_opts_default(&def);
    const cagra_engine_opts* o = opts ? opts : &def;
    if (o->mode == CAGRA_MODE_SHARED && o->team_count < 2)
      throw UsageErr("batch_search: shared mode requires team_count >= 2");
    std::lock_guard<std::mutex> lock(ix->mu);
    DeviceScope scope(ix->device);
    // NULL = the caller's legacy default stream (CUDA's usual convention)
    cudaStream_t s = stream ? reinterpret_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    begin_on(ix, s);
    uint32_t* counts = d_counts_out;
    if (!counts) {
      grow(ix, ix->counts, sizeof(uint32_t) * nq);
      counts = ix->counts.as<uint32_t>();
    }
    run_search(ix, d_queries, nq, params, o, d_ids_out, d_dists_out, counts, d_stats_out, s);
    end_on(ix, s);
  });
}

uint32_t cagra_last_launch_count(const cagra_index* index) {
  return index ? index->last_launches : 0;
}

int cagra_merge_shard_topk_dev(const uint32_t* d_shard_ids, const float* d_shard_dists,
                               uint32_t shards, uint32_t nq, uint32_t k,
                               const uint64_t* shard_offsets, uint32_t* d_ids_out,
                               float* d_dists_out, int device, void* stream) {
  return guarded([&] {
    if (shards == 0 || k == 0) throw UsageErr("shard merge: empty input");
    int dev = resolve_device(device);
    DeviceScope scope(dev);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DBuf off(sizeof(uint64_t) * shards);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(off.p, shard_offsets, sizeof(uint64_t) * shards,
                                   cudaMemcpyHostToDevice, s));
    launch_shard_merge(d_shard_ids, d_shard_dists, shards, nq, k, off.as<uint64_t>(), d_ids_out,
                       d_dists_out, s);
    CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
