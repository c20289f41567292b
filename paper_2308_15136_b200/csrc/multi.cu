// Multi-GPU layer of the C ABI, in one process (the reference
// has no distributed code — its batch_search is a parallel_for over queries,
// engine.cpp:95-120).  Built over the single-device entry points:
//
//  * row-sharded kNN build (cagra_build_graph_multi): every device holds the
//    whole dataset and computes the exact kNN rows of its contiguous row range
//    (the K1 launcher's self_base), the rows are copied peer-to-peer into the
//    first device's (n x d_init) buffers, and the rank optimize runs there —
//    the parallel_for over rows of knn_build.cpp:49 spread over GPUs; the
//    graph is bit-identical to a one-device build.
//  * cagra_mindex, CAGRA_SHARD_REPLICATE: every device holds a replica;
//    cagra_msearch splits the batch into contiguous slices, one per device,
//    with query_offset so every query keeps its single-GPU seed
//    (mix_seed(seed ^ (0x0bad + global qi)), engine.cpp:108).
//  * cagra_mindex, CAGRA_SHARD_DATASET: device g holds the id range
//    [g n/G, (g+1) n/G) with its own graph; every device searches every query
//    and its search kernel stores the shard's top-k straight into the first
//    device's [G][nq][k] gather buffer over NVLink (peer access; a peer copy
//    when the pair has none), then K8 merges by (dist, global id) there
//    (merge_team_results order, engine.cpp:24-34).
// Device lists may repeat a device (several parts on one GPU): that is how
// the multi-GPU paths are exercised on a one-GPU box.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "cagra/capi.h"
#include "host_util.hpp"

namespace cagra {
namespace {

// Runs f(g) for g in [0, G) on one host thread each (every thread selects its
// own device); rethrows the first failure.
template <class F>
void for_each_part(size_t G, F&& f) {
  if (G == 1) {
    f(size_t{0});
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(G);
  for (size_t g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        f(g);
      } catch (...) {
        err[g] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// contiguous, balanced [start, end) ranges (first n % G one longer)
std::vector<std::pair<uint64_t, uint64_t>> split_ranges(uint64_t n, size_t G) {
  std::vector<std::pair<uint64_t, uint64_t>> out(G);
  const uint64_t base = n / G, extra = n % G;
  uint64_t s = 0;
  for (size_t g = 0; g < G; ++g) {
    const uint64_t e = s + base + (g < extra ? 1 : 0);
    out[g] = {s, e};
    s = e;
  }
  return out;
}

std::vector<int> resolve_devices(const int* devices, uint32_t ndev) {
  if (!devices || ndev == 0) throw UsageErr("device set: empty");
  std::vector<int> out(ndev);
  for (uint32_t g = 0; g < ndev; ++g) out[g] = resolve_device(devices[g]);
  return out;
}

// lets `from` store into / copy from `to`'s memory directly when the pair
// supports it (always true for the same device)
bool enable_peer(int from, int to) {
  if (from == to) return true;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, from, to) != cudaSuccess || !can) return false;
  DeviceScope scope(from);
  const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return true;
  }
  return e == cudaSuccess;
}

// Row-sharded exact kNN on `devs` -> (ids, dists) rows on devs[0] (device
// buffers owned by the caller); returns the wall seconds of the parallel phase.
double knn_rows_multi(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                      const std::vector<int>& devs, uint32_t* root_ids, float* root_dists) {
  const size_t G = devs.size();
  const uint32_t ld = row_stride(dim);
  const auto rows = split_ranges(n, G);
  const int root = devs[0];
  std::vector<char> peer(G);
  for (size_t g = 0; g < G; ++g) peer[g] = enable_peer(devs[g], root);
  const auto t0 = std::chrono::steady_clock::now();
  for_each_part(G, [&](size_t g) {
    const uint64_t r0 = rows[g].first, cnt = rows[g].second - rows[g].first;
    if (!cnt) return;
    DeviceScope scope(devs[g]);
    Stream st;
    DBuf dd(sizeof(float) * (size_t)n * ld);
    upload_rows(dd.as<float>(), data, n, dim, ld, st.s);
    uint32_t* ids = root_ids + r0 * k;
    float* dists = root_dists + r0 * k;
    DBuf li, lds;
    if (!peer[g]) {  // no peer stores: compute locally, then one peer copy
      li.alloc(sizeof(uint32_t) * cnt * k);
      lds.alloc(sizeof(float) * cnt * k);
      ids = li.as<uint32_t>();
      dists = lds.as<float>();
    }
    launch_exact_topk(dd.as<float>(), n, ld, dd.as<float>() + r0 * ld, (uint32_t)cnt, ld, dim,
                      k, true, ids, dists, st.s, (uint32_t)r0);
    if (!peer[g]) {
      CAGRA_CUDA_TRY(cudaMemcpyPeerAsync(root_ids + r0 * k, root, li.p, devs[g],
                                         sizeof(uint32_t) * cnt * k, st.s));
      CAGRA_CUDA_TRY(cudaMemcpyPeerAsync(root_dists + r0 * k, root, lds.p, devs[g],
                                         sizeof(float) * cnt * k, st.s));
    }
    st.sync();
  });
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace
}  // namespace cagra

using namespace cagra;

// ============================================================ the index ====
struct cagra_mindex {
  uint32_t mode = CAGRA_SHARD_REPLICATE;
  uint32_t n = 0, dim = 0, degree = 0, ld = 0;
  std::vector<int> devs;
  std::vector<cagra_index*> parts;
  std::vector<uint64_t> offsets;   // first global id of each part (dataset mode)
  std::vector<char> peer;          // part g can store into devs[0]'s memory
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;
  // per part (on its device): queries, ids, dists, counts, stats
  std::vector<DBuf> q, ids, dists, counts, stats;
  // first device: [G][nq][k] gather, merged output, shard offsets
  DBuf gi, gd, oi, od, offs;
  std::mutex mu;
  ~cagra_mindex() {
    for (size_t g = 0; g < parts.size(); ++g) {
      DeviceScope scope(devs[g]);
      if (parts[g]) cagra_index_destroy(parts[g]);
      if (g < streams.size() && streams[g]) cudaStreamDestroy(streams[g]);
      if (g < events.size() && events[g]) cudaEventDestroy(events[g]);
      // buffers are freed on their own device
      if (g < q.size()) {
        q[g].release();
        ids[g].release();
        dists[g].release();
        counts[g].release();
        stats[g].release();
      }
    }
    if (!devs.empty()) {
      DeviceScope scope(devs[0]);
      gi.release();
      gd.release();
      oi.release();
      od.release();
      offs.release();
    }
  }
};

namespace {

void grow_on(int dev, DBuf& b, size_t bytes) {
  if (bytes <= b.bytes) return;
  DeviceScope scope(dev);
  CAGRA_CUDA_TRY(cudaDeviceSynchronize());
  b.alloc(bytes);
}

}  // namespace

extern "C" {

int cagra_build_graph_multi(const float* data, uint32_t n, uint32_t dim, uint32_t d_init,
                            uint32_t d, const int* devices, uint32_t ndev, uint32_t* graph_out,
                            uint32_t* knn_ids_out, float* knn_dists_out, double* seconds_out) {
  return guarded([&] {
    if (d_init == 0 || d_init >= n) throw UsageErr("exact_knn_graph: require 1 <= k < N");
    if (d == 0 || d > d_init) throw UsageErr("optimize: require 1 <= d <= input degree");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    const std::vector<int> devs = resolve_devices(devices, ndev);
    DeviceScope scope(devs[0]);
    const size_t e = (size_t)n * d_init;
    DBuf di(4 * e), ds(4 * e), out(4ull * n * d);
    const double knn_s = knn_rows_multi(data, n, dim, d_init, devs, di.as<uint32_t>(),
                                        ds.as<float>());
    Stream st;
    OptOut t;
    optimize_device(di.as<uint32_t>(), ds.as<float>(), n, d_init, d, true, true,
                    out.as<uint32_t>(), st.s, &t);
    CAGRA_CUDA_TRY(cudaMemcpyAsync(graph_out, out.p, 4ull * n * d, cudaMemcpyDeviceToHost, st.s));
    if (knn_ids_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(knn_ids_out, di.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    if (knn_dists_out)
      CAGRA_CUDA_TRY(cudaMemcpyAsync(knn_dists_out, ds.p, 4 * e, cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (seconds_out) {
      seconds_out[0] = knn_s;
      seconds_out[1] = t.ms[4] * 1e-3;
    }
  });
}

int cagra_exact_knn_graph_multi(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                                const int* devices, uint32_t ndev, uint32_t* ids_out,
                                float* dists_out) {
  return guarded([&] {
    if (k == 0 || k >= n) throw UsageErr("exact_knn_graph: require 1 <= k < N");
    if (dim == 0) throw UsageErr("dataset dimension must be >= 1");
    const std::vector<int> devs = resolve_devices(devices, ndev);
    DeviceScope scope(devs[0]);
    const size_t e = (size_t)n * k;
    DBuf di(4 * e), ds(4 * e);
    knn_rows_multi(data, n, dim, k, devs, di.as<uint32_t>(), ds.as<float>());
    CAGRA_CUDA_TRY(cudaMemcpy(ids_out, di.p, 4 * e, cudaMemcpyDeviceToHost));
    CAGRA_CUDA_TRY(cudaMemcpy(dists_out, ds.p, 4 * e, cudaMemcpyDeviceToHost));
  });
}

int cagra_mindex_create(const float* data, uint32_t n, uint32_t dim, const uint32_t* graph,
                        uint32_t degree, const int* devices, uint32_t ndev, uint32_t shard_mode,
                        cagra_mindex** out) {
  return guarded([&] {
    if (!out) throw UsageErr("null output handle");
    if (n == 0 || dim == 0) throw UsageErr("index: empty dataset");
    if (degree == 0) throw FormatErr("graph: empty");
    if (shard_mode != CAGRA_SHARD_REPLICATE && shard_mode != CAGRA_SHARD_DATASET)
      throw UsageErr("device set: unknown shard mode");
    auto* mx = new cagra_mindex();
    try {
      mx->mode = shard_mode;
      mx->devs = resolve_devices(devices, ndev);
      const size_t G = mx->devs.size();
      mx->n = n;
      mx->dim = dim;
      mx->degree = degree;
      mx->ld = row_stride(dim);
      mx->parts.assign(G, nullptr);
      mx->q.resize(G);
      mx->ids.resize(G);
      mx->dists.resize(G);
      mx->counts.resize(G);
      mx->stats.resize(G);
      mx->streams.assign(G, nullptr);
      mx->events.assign(G, nullptr);
      mx->peer.assign(G, 0);
      mx->offsets.assign(G, 0);
      for (size_t g = 0; g < G; ++g) {
        mx->peer[g] = enable_peer(mx->devs[g], mx->devs[0]);
        DeviceScope scope(mx->devs[g]);
        CAGRA_CUDA_TRY(cudaStreamCreateWithFlags(&mx->streams[g], cudaStreamNonBlocking));
        CAGRA_CUDA_TRY(cudaEventCreateWithFlags(&mx->events[g], cudaEventDisableTiming));
      }
      if (shard_mode == CAGRA_SHARD_REPLICATE) {
        std::vector<uint32_t> built;
        if (!graph) {  // row-sharded build over the same devices
          built.resize((size_t)n * degree);
          const int rc = cagra_build_graph_multi(data, n, dim, 2 * degree, degree, devices, ndev,
                                                 built.data(), nullptr, nullptr, nullptr);
          if (rc != CAGRA_OK) throw CudaErr(last_error_slot());
          graph = built.data();
        }
        for_each_part(G, [&](size_t g) {
          const int rc = cagra_index_create(data, n, dim, graph, degree, mx->devs[g],
                                            &mx->parts[g]);
          if (rc == CAGRA_ERR_USAGE) throw UsageErr(last_error_slot());
          if (rc != CAGRA_OK) throw CudaErr(last_error_slot());
        });
      } else {
        if (graph) throw UsageErr("dataset-sharded index: shard graphs are built per device "
                                  "(pass graph = NULL)");
        const auto rows = split_ranges(n, G);
        for (size_t g = 0; g < G; ++g) {
          mx->offsets[g] = rows[g].first;
          if (rows[g].second - rows[g].first <= 2ull * degree)
            throw UsageErr("dataset-sharded index: shard smaller than the kNN degree");
        }
        for_each_part(G, [&](size_t g) {
          const uint32_t a = (uint32_t)rows[g].first, cnt = (uint32_t)(rows[g].second - a);
          std::vector<uint32_t> sg((size_t)cnt * degree);
          int rc = cagra_build_graph(data + (size_t)a * dim, cnt, dim, 2 * degree, degree,
                                     mx->devs[g], sg.data(), nullptr, nullptr, nullptr);
          if (rc == CAGRA_OK)
            rc = cagra_index_create(data + (size_t)a * dim, cnt, dim, sg.data(), degree,
                                    mx->devs[g], &mx->parts[g]);
          if (rc == CAGRA_ERR_USAGE) throw UsageErr(last_error_slot());
          if (rc != CAGRA_OK) throw CudaErr(last_error_slot());
        });
      }
    } catch (...) {
      delete mx;
      throw;
    }
    *out = mx;
  });
}

int cagra_mindex_destroy(cagra_mindex* index) {
  return guarded([&] { delete index; });
}

int cagra_mindex_info(const cagra_mindex* index, uint32_t* n, uint32_t* dim, uint32_t* degree,
                      uint32_t* parts, uint32_t* shard_mode) {
  return guarded([&] {
    if (!index) throw UsageErr("null index");
    if (n) *n = index->n;
    if (dim) *dim = index->dim;
    if (degree) *degree = index->degree;
    if (parts) *parts = (uint32_t)index->parts.size();
    if (shard_mode) *shard_mode = index->mode;
  });
}

int cagra_msearch(cagra_mindex* mx, const float* queries, uint32_t nq, uint32_t dim,
                  const cagra_search_params* params, const cagra_engine_opts* opts,
                  uint32_t* ids_out, float* dists_out, uint32_t* counts_out,
                  cagra_search_stats* stats_out) {
  return guarded([&] {
    if (!mx) throw UsageErr("null index");
    // batch_search validation order, engine.cpp:98-102
    if (nq == 0) return;
    if (dim != mx->dim) throw UsageErr("batch_search: query dimension mismatch");
    cagra_engine_opts def;
    cagra_engine_opts_default(&def);
    const cagra_engine_opts* o = opts ? opts : &def;
    std::lock_guard<std::mutex> lock(mx->mu);
    const size_t G = mx->parts.size();
    const uint32_t k = params->k, ld = mx->ld;
    // the single-device search validates params / modes with the reference's
    // errors; a failing part rethrows here with its message
    auto search_part = [&](size_t g, const float* dq, uint32_t cnt, const cagra_engine_opts* po,
                           uint32_t* d_ids, float* d_dists) {
      const int rc = cagra_search_dev(mx->parts[g], dq, cnt, params, po, d_ids, d_dists,
                                      mx->counts[g].as<uint32_t>(),
                                      mx->stats[g].as<cagra_search_stats>(), mx->streams[g]);
      if (rc == CAGRA_ERR_USAGE) throw UsageErr(last_error_slot());
      if (rc == CAGRA_ERR_LOGIC) throw LogicErr(last_error_slot());
      if (rc != CAGRA_OK) throw CudaErr(last_error_slot());
    };
    if (mx->mode == CAGRA_SHARD_REPLICATE) {
      const auto sl = split_ranges(nq, G);
      // launches are asynchronous: one host thread drives every device
      for (size_t g = 0; g < G; ++g) {
        const uint32_t off = (uint32_t)sl[g].first, cnt = (uint32_t)(sl[g].second - off);
        if (!cnt) continue;
        const int dev = mx->devs[g];
        grow_on(dev, mx->q[g], sizeof(float) * (size_t)cnt * ld);
        grow_on(dev, mx->ids[g], sizeof(uint32_t) * (size_t)cnt * k);
        grow_on(dev, mx->dists[g], sizeof(float) * (size_t)cnt * k);
        grow_on(dev, mx->counts[g], sizeof(uint32_t) * cnt);
        grow_on(dev, mx->stats[g], sizeof(cagra_search_stats) * cnt);
        DeviceScope scope(dev);
        cudaStream_t s = mx->streams[g];
        upload_rows(mx->q[g].as<float>(), queries + (size_t)off * dim, cnt, dim, ld, s);
        cagra_engine_opts po = *o;
        po.query_offset = o->query_offset + off;  // global query index -> 1-GPU seeds
        search_part(g, mx->q[g].as<float>(), cnt, &po, mx->ids[g].as<uint32_t>(),
                    mx->dists[g].as<float>());
        CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out + (size_t)off * k, mx->ids[g].p,
                                       sizeof(uint32_t) * (size_t)cnt * k,
                                       cudaMemcpyDeviceToHost, s));
        CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out + (size_t)off * k, mx->dists[g].p,
                                       sizeof(float) * (size_t)cnt * k, cudaMemcpyDeviceToHost,
                                       s));
        if (counts_out)
          CAGRA_CUDA_TRY(cudaMemcpyAsync(counts_out + off, mx->counts[g].p,
                                         sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost, s));
        if (stats_out)
          CAGRA_CUDA_TRY(cudaMemcpyAsync(stats_out + off, mx->stats[g].p,
                                         sizeof(cagra_search_stats) * cnt,
                                         cudaMemcpyDeviceToHost, s));
      }
      for (size_t g = 0; g < G; ++g) {
        DeviceScope scope(mx->devs[g]);
        CAGRA_CUDA_TRY(cudaStreamSynchronize(mx->streams[g]));
      }
      return;
    }
    // ---- dataset-sharded: every part searches every query
    const int root = mx->devs[0];
    const size_t slab = (size_t)nq * k;
    grow_on(root, mx->gi, sizeof(uint32_t) * slab * G);
    grow_on(root, mx->gd, sizeof(float) * slab * G);
    grow_on(root, mx->oi, sizeof(uint32_t) * slab);
    grow_on(root, mx->od, sizeof(float) * slab);
    grow_on(root, mx->offs, sizeof(uint64_t) * G);
    std::vector<cagra_search_stats> part_stats(stats_out ? (size_t)nq * G : 0);
    for (size_t g = 0; g < G; ++g) {
      const int dev = mx->devs[g];
      grow_on(dev, mx->q[g], sizeof(float) * (size_t)nq * ld);
      grow_on(dev, mx->counts[g], sizeof(uint32_t) * nq);
      grow_on(dev, mx->stats[g], sizeof(cagra_search_stats) * nq);
      if (!mx->peer[g]) {
        grow_on(dev, mx->ids[g], sizeof(uint32_t) * slab);
        grow_on(dev, mx->dists[g], sizeof(float) * slab);
      }
    }
    for (size_t g = 0; g < G; ++g) {
      const int dev = mx->devs[g];
      DeviceScope scope(dev);
      cudaStream_t s = mx->streams[g];
      upload_rows(mx->q[g].as<float>(), queries, nq, dim, ld, s);
      uint32_t* gi = mx->gi.as<uint32_t>() + g * slab;
      float* gd = mx->gd.as<float>() + g * slab;
      if (mx->peer[g]) {
        // the search kernel's epilogue stores straight into the first
        // device's gather slab (NVLink peer stores)
        search_part(g, mx->q[g].as<float>(), nq, o, gi, gd);
      } else {
        search_part(g, mx->q[g].as<float>(), nq, o, mx->ids[g].as<uint32_t>(),
                    mx->dists[g].as<float>());
        CAGRA_CUDA_TRY(cudaMemcpyPeerAsync(gi, root, mx->ids[g].p, dev, sizeof(uint32_t) * slab,
                                           s));
        CAGRA_CUDA_TRY(cudaMemcpyPeerAsync(gd, root, mx->dists[g].p, dev, sizeof(float) * slab,
                                           s));
      }
      if (stats_out)
        CAGRA_CUDA_TRY(cudaMemcpyAsync(part_stats.data() + g * nq, mx->stats[g].p,
                                       sizeof(cagra_search_stats) * nq, cudaMemcpyDeviceToHost,
                                       s));
      CAGRA_CUDA_TRY(cudaEventRecord(mx->events[g], s));
    }
    {
      DeviceScope scope(root);
      cudaStream_t s = mx->streams[0];
      for (size_t g = 1; g < G; ++g) CAGRA_CUDA_TRY(cudaStreamWaitEvent(s, mx->events[g], 0));
      CAGRA_CUDA_TRY(cudaMemcpyAsync(mx->offs.p, mx->offsets.data(), sizeof(uint64_t) * G,
                                     cudaMemcpyHostToDevice, s));
      launch_shard_merge(mx->gi.as<uint32_t>(), mx->gd.as<float>(), (uint32_t)G, nq, k,
                         mx->offs.as<uint64_t>(), mx->oi.as<uint32_t>(), mx->od.as<float>(), s);
      CAGRA_CUDA_TRY(cudaMemcpyAsync(ids_out, mx->oi.p, sizeof(uint32_t) * slab,
                                     cudaMemcpyDeviceToHost, s));
      CAGRA_CUDA_TRY(cudaMemcpyAsync(dists_out, mx->od.p, sizeof(float) * slab,
                                     cudaMemcpyDeviceToHost, s));
    }
    for (size_t g = 0; g < G; ++g) {
      DeviceScope scope(mx->devs[g]);
      CAGRA_CUDA_TRY(cudaStreamSynchronize(mx->streams[g]));
    }
    if (counts_out)
      for (uint32_t qi = 0; qi < nq; ++qi) {
        uint32_t c = 0;
        while (c < k && ids_out[(size_t)qi * k + c] != 0xffffffffu) ++c;
        counts_out[qi] = c;
      }
    if (stats_out)
      // one traversal per shard: evaluations and resets add up, iterations
      // are the longest shard's, converged only if every shard converged
      for (uint32_t qi = 0; qi < nq; ++qi) {
        cagra_search_stats a{};
        a.converged = 1;
        for (size_t g = 0; g < G; ++g) {
          const cagra_search_stats& b = part_stats[g * nq + qi];
          a.iterations = std::max(a.iterations, b.iterations);
          a.hash_resets += b.hash_resets;
          a.distance_evals += b.distance_evals;
          a.converged &= b.converged;
        }
        stats_out[qi] = a;
      }
  });
}

}  // extern "C"
