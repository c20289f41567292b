/*
 * cagra/capi.h — the C-ABI boundary of the B200-native CAGRA engine.
 *
 * This is the only seam between host code (the C++ drop-in `fodg::` shim in
 * paper_2308_15136_b200/host/, the Python mirror in paper_2308_15136_b200/fodg.py,
 * a cgo/JNI/ctypes binding) and the sm_100a kernels.  Signatures use plain
 * pointers, sizes and POD structs; no C++ or torch types cross it.
 *
 * Every entry point replaces one reference interface (namespace fodg in
 * /root/reference/proj/core/include/fodg/); the replaced declaration is cited
 * beside each function.  Semantics (argument meaning, validation order, error
 * class) follow the reference:
 *   CAGRA_ERR_USAGE  <-> fodg::UsageError  (common.hpp:13-15)
 *   CAGRA_ERR_FORMAT <-> fodg::FormatError (common.hpp:18-20)
 *   CAGRA_ERR_LOGIC  <-> std::logic_error  (search.cpp:180)
 * and the message is available from cagra_last_error() (thread-local).
 *
 * Memory conventions: unless a function name ends in `_dev`, every pointer is
 * a HOST pointer; inputs are borrowed for the call, outputs are caller
 * allocated.  Calls are synchronous on return.  `_dev` variants take device
 * pointers and a cudaStream_t (as void*) and are asynchronous on that stream.
 *
 * Id layout (common.hpp:22-30): low 31 bits = node id, MSB = parent flag,
 * 0xffffffff = dummy / padding.
 */
#ifndef CAGRA_CAPI_H_
#define CAGRA_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
enum {
  CAGRA_OK = 0,
  CAGRA_ERR_USAGE = 2,    /* fodg::UsageError */
  CAGRA_ERR_FORMAT = 3,   /* fodg::FormatError */
  CAGRA_ERR_CUDA = 4,     /* CUDA runtime failure (no device, OOM, launch) */
  CAGRA_ERR_NCCL = 5,     /* collective failure */
  CAGRA_ERR_LOGIC = 6     /* std::logic_error: internal invariant broken */
};

/* Thread-local message of the last failing call on this thread. */
const char* cagra_last_error(void);
/* Library version string and the compiled target ("sm_100a"). */
const char* cagra_version(void);
/* Number of visible CUDA devices (0 when none); returns CAGRA_OK. */
int cagra_device_count(int* out);

/* ---- enums mirrored from the reference ----------------------------------- */
/* HashPolicy (search.hpp:12) */
enum { CAGRA_HASH_STANDARD = 0, CAGRA_HASH_FORGETTABLE = 1 };
/* ExecutionMode (engine.hpp:15) */
enum { CAGRA_MODE_PER_QUERY = 0, CAGRA_MODE_SHARED = 1 };
/* ReorderMode (graph_opt.hpp:16); only rank mode is implemented on device. */
enum { CAGRA_REORDER_RANK = 0, CAGRA_REORDER_DISTANCE = 1 };

/* ---- POD mirrors of the reference parameter/stat structs ----------------- */
/* SearchParams (search.hpp:14-27), field for field. */
typedef struct cagra_search_params {
  uint32_t k;
  uint32_t topm;           /* M */
  uint32_t width;          /* p */
  uint32_t max_iterations; /* 0 = clamp(ceil(2M/p), 16, 256) */
  uint32_t min_iterations;
  uint32_t hash_policy;    /* CAGRA_HASH_* */
  uint32_t hash_bits;
  uint32_t reset_interval;
  uint64_t seed;
} cagra_search_params;

/* Fills the reference defaults (search.hpp:15-23). */
void cagra_search_params_default(cagra_search_params* p);

/* EngineOptions (engine.hpp:27-31) plus the device-side knobs that have no
 * reference counterpart.  `num_threads` is accepted and ignored (the grid
 * replaces parallel_for). */
typedef struct cagra_engine_opts {
  uint32_t mode;          /* CAGRA_MODE_* */
  uint32_t team_count;    /* shared mode traversals per query */
  uint32_t num_threads;   /* ignored on device (results never depend on it) */
  uint32_t seed_mode;     /* 0: batch_search seeds mix_seed(seed ^ (0x0bad+qi))
                             (engine.cpp:108); 1: params.seed as given for every
                             query (search_one, search.cpp:163) */
  uint64_t query_offset;  /* global index of query 0 (query-sharded runs keep
                             the single-GPU seeds) */
  uint32_t exact_distances; /* 1: in-loop distances use the sequential fp32
                               chain of squared_l2 (dataset.hpp:33-43), bit-equal
                               to the CPU; 0: warp-team reduction (faster),
                               final k re-scored with the sequential chain */
  uint32_t team_size;     /* lanes per distance in fast mode: 0=auto,4,8,16,32 */
  uint32_t multi_cta;     /* shared mode: 0 auto (one CTA per team when the batch
                             is smaller than the SM count and exact_distances=0),
                             1 single-CTA lockstep teams (the reference's team
                             order, engine.cpp:63-72), 2 one CTA per team */
  uint32_t _pad;
} cagra_engine_opts;

void cagra_engine_opts_default(cagra_engine_opts* o);

/* SearchStats (search.hpp:96-101). */
typedef struct cagra_search_stats {
  uint32_t iterations;
  uint32_t hash_resets;
  uint64_t distance_evals;
  uint32_t converged;
  uint32_t _pad;
} cagra_search_stats;

/* OptimizeStats (graph_opt.hpp:33-41) — device-timed stage seconds. */
typedef struct cagra_opt_stats {
  double count_seconds;
  double reorder_seconds;
  double reverse_seconds;
  double merge_seconds;
  double total_seconds;
} cagra_opt_stats;

/* ---- synthetic inputs ---------------------------------------------------- */
/* The reference fixture generator (tests/test_util.hpp:11-18): mt19937_64(seed)
 * feeding std::uniform_real_distribution<float>(0,1), row-major.  Host code;
 * bit-identical to libstdc++. */
int cagra_uniform_dataset(uint64_t seed, uint64_t count, float* out);
/* splitmix64 finaliser, common.hpp:34-39. */
uint64_t cagra_mix_seed(uint64_t x);

/* ---- kNN build and ground truth ------------------------------------------ */
/* exact_knn_graph (knn_build.hpp:40): per node the k nearest other nodes,
 * rows sorted by (dist, id), dists bit-equal to the sequential fp32 chain.
 * Validation: 1 <= k < n else USAGE. */
int cagra_exact_knn_graph(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                          int device, uint32_t* ids_out, float* dists_out);

/* Rows [row_begin, row_end) of exact_knn_graph(data, k) (knn_build.cpp:40-63:
 * the parallel_for over rows at :49, one contiguous range) — bit-identical to
 * those rows of the full graph.  Outputs (row_end - row_begin) x k.  The unit
 * of a row-sharded multi-GPU / multi-process kNN build. */
int cagra_exact_knn_rows(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                         uint32_t row_begin, uint32_t row_end, int device, uint32_t* ids_out,
                         float* dists_out);

/* nn_descent (knn_build.hpp:42; knn_build.cpp:96-231) on the device: random
 * initial rows, rounds of neighbour-of-neighbour joins over sampled new/old
 * entries until fewer than termination_delta * N * k row insertions or
 * max_rounds.  Deterministic for a fixed seed.  Rows sorted by (dist, id),
 * distances the sequential fp32 chain.  k <= 256. */
int cagra_nn_descent(const float* data, uint32_t n, uint32_t dim, uint32_t k, double sample_rate,
                     double termination_delta, uint32_t max_rounds, uint64_t seed, int device,
                     uint32_t* ids_out, float* dists_out, uint32_t* converged_out,
                     uint32_t* rounds_out);

/* exact_topk (topk.hpp:20) for a batch of queries: k nearest by (dist, id). */
int cagra_exact_topk(const float* data, uint32_t n, uint32_t dim, const float* queries,
                     uint32_t nq, uint32_t k, int device, uint32_t* ids_out,
                     float* dists_out);

/* Counters of the last tensor-core kNN / top-k call in this process: rows
 * processed, rows re-done by the exact SIMT kernel because their candidate
 * band overflowed, candidates re-ranked with the sequential chain, rows whose
 * sample-pass threshold did not bracket their band (re-done by the
 * single-pass list mode).  Any pointer may be NULL. */
int cagra_knn_last_stats(uint64_t* rows, uint64_t* fallback_rows, uint64_t* reranked,
                         uint64_t* retried_rows);

/* Filter of the last tensor-core kNN / top-k call: split_terms 1 = fp16
 * single term, 3 = bf16x3; gemm_k = K of the filter GEMM (MMA work per
 * (query, point) pair = 2 gemm_k flops).  Either pointer may be NULL. */
int cagra_knn_last_filter(uint32_t* split_terms, uint32_t* gemm_k);

/* The kNN build keeps its large scratch (16-bit operand rows, candidate
 * buffers) cached per device between calls; this releases it (device < 0: all
 * devices).  No reference counterpart (the reference allocates per call). */
int cagra_trim_scratch(int device);

/* ---- graph quality metrics ----------------------------------------------- */
/* strong_cc_count (graph_metrics.hpp:22) and the integer total behind
 * avg_2hop_count (graph_metrics.hpp:26; mean = two_hop_total / n), on the
 * device.  graph: n x degree host ids (< n, else USAGE).  Either output may be
 * NULL to skip that metric. */
int cagra_graph_metrics(const uint32_t* graph, uint32_t n, uint32_t degree, int device,
                        uint64_t* strong_cc, uint64_t* two_hop_total);

/* ---- graph optimization (rank mode) -------------------------------------- */
/* count_detourable_routes (graph_opt.hpp:47-49), rank mode.  Rejects rows not
 * sorted by (dist, id) with USAGE (graph_opt.cpp:19-31). */
int cagra_count_detourable_routes(const uint32_t* knn_ids, const float* knn_dists,
                                  uint32_t n, uint32_t deg, int device,
                                  uint32_t* counts_out);
/* count_detourable_routes (graph_opt.hpp:47-49), distance mode — the paper's
 * comparison variant: every leg recomputed from the vectors (graph_opt.cpp:
 * 66-71, 87-93).  data: ds_n x dim host rows (NULL -> USAGE, as the
 * reference's "distance mode requires the dataset"). */
int cagra_count_detourable_routes_distance(const uint32_t* knn_ids, const float* knn_dists,
                                           uint32_t n, uint32_t deg, const float* data,
                                           uint32_t ds_n, uint32_t dim, int device,
                                           uint32_t* counts_out);
/* reorder_and_prune (graph_opt.hpp:53-54). */
int cagra_reorder_and_prune(const uint32_t* knn_ids, const uint32_t* counts, uint32_t n,
                            uint32_t deg, uint32_t d, int device, uint32_t* pruned_out);
/* build_reverse_graph (graph_opt.hpp:59): row y holds at most `cap` sources
 * ordered by (rank, source).  With c = min(cap, n) (a cap above n means no
 * cap): rev_counts_out[n], rev_ids_out[n*c] (row y at y*c, first
 * rev_counts_out[y] valid). */
int cagra_build_reverse_graph(const uint32_t* pruned, uint32_t n, uint32_t d, uint32_t cap,
                              int device, uint32_t* rev_counts_out, uint32_t* rev_ids_out);
/* merge_graphs (graph_opt.hpp:63) on the CSR reverse form above. */
int cagra_merge_graphs(const uint32_t* pruned, const uint32_t* rev_counts,
                       const uint32_t* rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
                       int device, uint32_t* graph_out);
/* optimize (graph_opt.hpp:67-68) with OptimizeOptions{kRank, reorder, add_reverse}.
 * knn_dists may be NULL when reorder = 0 (plain truncation). */
int cagra_optimize(const uint32_t* knn_ids, const float* knn_dists, uint32_t n,
                   uint32_t deg, uint32_t d, uint32_t reorder, uint32_t add_reverse,
                   int device, uint32_t* graph_out, cagra_opt_stats* stats);

/* Whole build on device, no host round trip between stages:
 * exact_knn_graph(ds, d_init) -> optimize(knn, d)  (tools/main.cpp:95, 111).
 * knn_ids_out / knn_dists_out may be NULL.  seconds_out[0] = kNN seconds,
 * seconds_out[1] = optimize seconds (device events); may be NULL. */
int cagra_build_graph(const float* data, uint32_t n, uint32_t dim, uint32_t d_init,
                      uint32_t d, int device, uint32_t* graph_out, uint32_t* knn_ids_out,
                      float* knn_dists_out, double* seconds_out);

/* ---- search -------------------------------------------------------------- */
typedef struct cagra_index cagra_index;

/* Upload (dataset, graph) once; the device-resident index replaces the
 * per-call `const Graph&, const Dataset&` of batch_search (engine.hpp:38-40).
 * Validates graph.num_nodes == ds.size() (search.cpp:165) and ids < n. */
int cagra_index_create(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                       uint32_t degree, int device, cagra_index** out);
/* Same, from device pointers already resident on `device` (copied). */
int cagra_index_create_dev(const float* d_data, uint32_t n, uint32_t dim,
                           const uint32_t* d_graph, uint32_t degree, int device,
                           cagra_index** out);
int cagra_index_destroy(cagra_index* index);
int cagra_index_info(const cagra_index* index, uint32_t* n, uint32_t* dim,
                     uint32_t* degree, int* device);
/* Row stride (floats) of device-resident rows: dim rounded up to 4.  Queries
 * passed to cagra_search_dev use this stride. */
uint32_t cagra_index_row_stride(const cagra_index* index);

/* batch_search (engine.hpp:38-40).  Outputs: ids_out[nq*k] / dists_out[nq*k]
 * (rows shorter than k padded with 0xffffffff / +inf), counts_out[nq] = number
 * of valid results, stats_out[nq] (may be NULL).  Validation order follows
 * engine.cpp:98-102 and search.cpp:39-50. */
int cagra_search(cagra_index* index, const float* queries, uint32_t nq, uint32_t dim,
                 const cagra_search_params* params, const cagra_engine_opts* opts,
                 uint32_t* ids_out, float* dists_out, uint32_t* counts_out,
                 cagra_search_stats* stats_out);

/* Device-pointer variant, asynchronous on `stream` (a cudaStream_t); used by
 * the benchmark and the multi-GPU paths (inputs already in HBM). */
int cagra_search_dev(cagra_index* index, const float* d_queries, uint32_t nq,
                     const cagra_search_params* params, const cagra_engine_opts* opts,
                     uint32_t* d_ids_out, float* d_dists_out, uint32_t* d_counts_out,
                     cagra_search_stats* d_stats_out, void* stream);

/* Number of kernels the last search call on this index launched. */
uint32_t cagra_last_launch_count(const cagra_index* index);

/* ---- multi-GPU in one process ---------------------------- */
/* The reference has no distributed code: batch_search is a parallel_for over
 * queries (engine.cpp:95-120) and exact_knn_graph one over rows
 * (knn_build.cpp:49).  These spread the same work over a device set; results
 * equal the one-device calls (replicated search and the row-sharded build
 * bit for bit).  `devices` may repeat a device. */
enum { CAGRA_SHARD_REPLICATE = 0, CAGRA_SHARD_DATASET = 1 };

/* cagra_build_graph with the exact kNN rows computed on every device of the
 * set (contiguous row ranges, peer-copied to devices[0], optimize there). */
int cagra_build_graph_multi(const float* data, uint32_t n, uint32_t dim, uint32_t d_init,
                            uint32_t d, const int* devices, uint32_t ndev, uint32_t* graph_out,
                            uint32_t* knn_ids_out, float* knn_dists_out, double* seconds_out);

/* exact_knn_graph (knn_build.hpp:40) with the rows spread over the device set. */
int cagra_exact_knn_graph_multi(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                                const int* devices, uint32_t ndev, uint32_t* ids_out,
                                float* dists_out);

typedef struct cagra_mindex cagra_mindex;
/* CAGRA_SHARD_REPLICATE: a replica of (data, graph) per device; graph NULL =
 * built with cagra_build_graph_multi (d_init = 2 degree).
 * CAGRA_SHARD_DATASET: device g holds ids [g n/G, (g+1) n/G) with its own
 * graph of `degree` built there (graph must be NULL). */
int cagra_mindex_create(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                        uint32_t degree, const int* devices, uint32_t ndev, uint32_t shard_mode,
                        cagra_mindex** out);
int cagra_mindex_destroy(cagra_mindex* index);
int cagra_mindex_info(const cagra_mindex* index, uint32_t* n, uint32_t* dim, uint32_t* degree,
                      uint32_t* parts, uint32_t* shard_mode);
/* batch_search over the set (host buffers, synchronous).  Replicated: the
 * batch is split into contiguous slices, one per device, each query keeping
 * its global seed.  Dataset-sharded: every device searches every query, the
 * per-shard top-k lists are stored into devices[0]'s gather buffer (peer
 * stores over NVLink) and merged by K8; stats sum evaluations / resets over
 * the shards, iterations are the maximum. */
int cagra_msearch(cagra_mindex* index, const float* queries, uint32_t nq, uint32_t dim,
                  const cagra_search_params* params, const cagra_engine_opts* opts,
                  uint32_t* ids_out, float* dists_out, uint32_t* counts_out,
                  cagra_search_stats* stats_out);

/* ---- dataset-sharded merge (K8) ------------------------------------------ */
/* Merge G per-shard top-k lists into one top-k per query by (dist, id).
 * Inputs (device): shard_ids/shard_dists laid out [G][nq][k], ids LOCAL to the
 * shard; shard_offsets[G] (host) are added to form global ids.  Outputs
 * [nq][k] (device), padded 0xffffffff/+inf.  Asynchronous on `stream`. */
int cagra_merge_shard_topk_dev(const uint32_t* d_shard_ids, const float* d_shard_dists,
                               uint32_t shards, uint32_t nq, uint32_t k,
                               const uint64_t* shard_offsets, uint32_t* d_ids_out,
                               float* d_dists_out, int device, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CAGRA_CAPI_H_ */
