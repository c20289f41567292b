// Internal launcher declarations shared by the kernel files and capi.cu.
// Everything here takes DEVICE pointers and is asynchronous on `stream`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace cagra {

// ---- knn_exact.cu / knn_tc.cu -----------------------------------------------
// Exact top-K by (dist, id) for nq query rows against n data rows (row
// strides ld / qld floats).  exclude_self drops data index == the query's own
// index (the kNN graph, knn_build.cpp:52-60): query row qi is data row
// self_base + qi (row-sharded builds pass d_queries = d_data + self_base * ld).
// Dispatcher: the tensor-core path (knn_tc.cu) when eligible, else SIMT.
void launch_exact_topk(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                       uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K, bool exclude_self,
                       uint32_t* d_ids, float* d_dists, cudaStream_t stream,
                       uint32_t self_base = 0);
// SIMT register-tiled sequential-chain kernel.  d_topk_scratch: nq*K u64.
void launch_exact_topk_simt(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                            uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K,
                            bool exclude_self, const uint32_t* d_self_ids,
                            uint64_t* d_topk_scratch, uint32_t* d_ids, float* d_dists,
                            cudaStream_t stream);
// tcgen05 path (fp16 single-term or bf16x3 split GEMM filter + exact re-rank); synchronous.
bool knn_tc_eligible(uint32_t dim, uint32_t K);
void launch_knn_tc(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                   uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K, bool exclude_self,
                   uint32_t self_base, uint32_t* d_ids, float* d_dists, cudaStream_t stream);
struct KnnTcStats {
  uint64_t rows = 0, fallback_rows = 0, reranked = 0, retried_rows = 0;
  uint32_t split_terms = 0;  // filter split of the last call: 1 fp16, 3 bf16x3
  uint32_t gemm_k = 0;       // K of the filter GEMM (16-wide MMA steps actually issued)
};
extern KnnTcStats g_knn_tc_stats;
// Frees the kNN build's cached scratch on `device` (all devices when < 0).
void knn_trim_scratch(int device);

// ---- nn_descent.cu -------------------------------------------------------------
struct NnDescentInfo {
  uint32_t rounds = 0;
  bool converged = false;
  unsigned long long last_inserted = 0;
};
// nn_descent (knn_build.cpp:96-231) on device: rows [n][k] sorted by (dist, id)
// with sequential-chain distances; synchronous on `s`.
NnDescentInfo launch_nn_descent(const float* d_data, uint32_t n, uint32_t ld, uint32_t dim,
                                uint32_t k, double sample_rate, double termination_delta,
                                uint32_t max_rounds, uint64_t seed, uint32_t* d_ids,
                                float* d_dists, cudaStream_t s);

// ---- metrics.cu ---------------------------------------------------------------
// Distinct <=2-hop neighbours summed over all nodes (avg_2hop_count * n) and
// the strongly connected component count; synchronous on `stream`.
uint64_t two_hop_total(const uint32_t* d_graph, uint32_t n, uint32_t d, int sm_count,
                       cudaStream_t stream);
uint64_t scc_count(const uint32_t* d_graph, uint32_t n, uint32_t d, cudaStream_t stream);

// ---- graph_opt.cu -----------------------------------------------------------
struct OptTimes {
  float count_ms = 0, reorder_ms = 0, reverse_ms = 0, merge_ms = 0, total_ms = 0;
};

// Validation passes (flags are device ints, set non-zero on violation).
void launch_check_sorted(const uint32_t* d_ids, const float* d_dists, uint32_t n, uint32_t deg,
                         int* d_flag, cudaStream_t stream);
void launch_check_ids(const uint32_t* d_ids, uint64_t count, uint32_t n, int* d_flag,
                      cudaStream_t stream);

// K2: rank-mode detour counting fused with the stable (count, rank) reorder.
// counts_out (n*deg) and/or pruned_out (n*d) may be null.
void launch_detour_reorder(const uint32_t* d_knn, uint32_t n, uint32_t deg, uint32_t d,
                           uint32_t* d_counts_out, uint32_t* d_pruned_out,
                           cudaStream_t stream);
// distance-mode detour counts (graph_opt.cpp:66-71, 87-93); data rows of ld floats.
void launch_detour_distance(const uint32_t* d_knn, uint32_t n, uint32_t deg, const float* d_data,
                            uint32_t ld, uint32_t dim, uint32_t* d_counts_out,
                            cudaStream_t stream);
// reorder only, from given counts (reorder_and_prune)
void launch_reorder_from_counts(const uint32_t* d_knn, const uint32_t* d_counts, uint32_t n,
                                uint32_t deg, uint32_t d, uint32_t* d_pruned_out,
                                cudaStream_t stream);
// K3: reverse graph in [n][cap] form + counts.
struct ReverseScratch {
  uint32_t* indeg = nullptr;       // n
  unsigned long long* start = nullptr;  // n+1
  uint32_t* fill = nullptr;        // n
  uint64_t* keys = nullptr;        // n*d
  unsigned long long* block_sums = nullptr;
};
size_t reverse_scratch_bytes(uint32_t n, uint32_t d);
void launch_reverse(const uint32_t* d_pruned, uint32_t n, uint32_t d, uint32_t cap,
                    void* d_scratch, uint32_t* d_rev_counts, uint32_t* d_rev_ids,
                    cudaStream_t stream);
// K4: interleave merge. d_flag set when a row lacks d distinct candidates.
void launch_merge(const uint32_t* d_pruned, const uint32_t* d_rev_counts,
                  const uint32_t* d_rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
                  uint32_t* d_out, int* d_flag, cudaStream_t stream);

// ---- search.cu ----------------------------------------------------------------
struct SearchConfig {
  uint32_t k, topm, width, max_iter, min_iter, hash_policy, hash_bits, reset_interval;
  uint64_t seed;
  uint32_t mode, team_count, seed_mode, exact, team_size;
  uint64_t query_offset;
  uint32_t multi_cta;  // 0 auto, 1 single-CTA lockstep teams, 2 one CTA per team
};

struct DeviceIndexView {
  const float* data;   // n x ld
  const uint32_t* graph;  // n x degree
  uint32_t n, dim, ld, degree;
};

struct SearchPlan {
  uint32_t grid = 0, hcap = 0, teams = 1, C = 0, max_iter = 0, min_iter = 0;
  bool smem_table = false;
  size_t smem = 0;
  size_t table_elems = 0;  // u64 slots of HBM visited tables (grid * hcap)
  size_t init_elems = 0;   // u32 init sample ids
  bool mc = false;         // shared mode with one CTA per (query, team)
  bool b1 = false;         // mc via the fused small-team kernel (search_b1.cu)
  bool b1_direct = false;  // its visited bitmap indexed by node id (hcap words >= n bits)
  bool bitmap = false;     // standard policy: exact visited bitmap per resident CTA
  bool inplace = false;    // per-query kernel: one top-M buffer (update_topm in place)
  uint32_t bm_words = 0;   // u32 words per CTA bitmap
  size_t team_elems = 0;   // u64 team top-M keys (nq * teams * M) in mc mode
  const void* fn = nullptr;
};
// Validates device limits and picks the kernel variant / grid.
// bytes of one query's multi-CTA visited region (shared by its teams)
uint64_t mc_table_bytes_per_query(const SearchConfig& c, uint32_t degree);
SearchPlan plan_search(const DeviceIndexView& ix, const SearchConfig& c, uint32_t nq,
                       int sm_count, size_t table_budget_bytes);
// Launches init-sample + search kernels; returns the number of kernels.
// d_tables / d_gens persist across calls (zeroed when first allocated).
uint32_t launch_search(const DeviceIndexView& ix, const SearchConfig& c, const SearchPlan& pl,
                       const float* d_queries, uint32_t nq, uint32_t* d_ids, float* d_dists,
                       uint32_t* d_counts, void* d_stats, uint32_t* d_init_ids,
                       uint32_t* d_work, unsigned long long* d_tables, uint32_t* d_gens,
                       unsigned long long* d_team_out, void* d_team_stats, uint32_t mc_tag,
                       cudaStream_t stream, uint32_t* d_b1_ctr = nullptr);

// ---- search_b1.cu: multi-CTA shared mode, one 128-thread CTA per team ------
// with the team merge in the query's last CTA (one launch per batch)
bool team_b1_eligible(uint32_t M, uint32_t k, uint32_t T, uint32_t degree, uint32_t ld);
void launch_team_b1(const float* data, const uint32_t* graph, uint32_t n, uint32_t ld,
                    uint32_t dim, uint32_t degree, const float* queries, uint32_t nq, uint32_t T,
                    uint32_t M, uint32_t k, uint32_t max_iter, uint32_t min_iter, uint64_t seed,
                    uint64_t query_offset, uint32_t seed_mode, uint32_t* tab, uint32_t hcap,
                    uint32_t tag, uint32_t direct, unsigned long long* team_out, void* team_stats,
                    uint32_t* done_ctr, uint32_t* out_ids, float* out_dists,
                    uint32_t* out_counts, void* stats, cudaStream_t stream);

// ---- merge.cu (K8) --------------------------------------------------------------
void launch_shard_merge(const uint32_t* d_shard_ids, const float* d_shard_dists,
                        uint32_t shards, uint32_t nq, uint32_t k, const uint64_t* d_offsets,
                        uint32_t* d_ids, float* d_dists, cudaStream_t stream);

}  // namespace cagra
