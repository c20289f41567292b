// Batch-1 latency through the C ABI from C++ (no Python in the loop):
// builds the 1M x 96 index on the device, then times sequential single-query
// cagra_search calls with pinned host buffers.
//   b1_latency [n] [queries] [team_topm] [teams]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#include "cagra/capi.h"

static void ok(int rc) {
  if (rc != CAGRA_OK) {
    std::fprintf(stderr, "cagra error %d: %s\n", rc, cagra_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? std::atoi(argv[1]) : 1000000, dim = 96, d = 64;
  const uint32_t nq = argc > 2 ? std::atoi(argv[2]) : 1000;
  const uint32_t topm = argc > 3 ? std::atoi(argv[3]) : 16, teams = argc > 4 ? std::atoi(argv[4]) : 64;
  std::vector<float> data((size_t)n * dim), qs((size_t)nq * dim);
  ok(cagra_uniform_dataset(424242, data.size(), data.data()));
  ok(cagra_uniform_dataset(424243, qs.size(), qs.data()));
  std::vector<uint32_t> graph((size_t)n * d);
  ok(cagra_build_graph(data.data(), n, dim, 2 * d, d, 0, graph.data(), nullptr, nullptr, nullptr));
  std::vector<uint32_t> gt((size_t)nq * 10);
  std::vector<float> gtd((size_t)nq * 10);
  ok(cagra_exact_topk(data.data(), n, dim, qs.data(), nq, 10, 0, gt.data(), gtd.data()));
  cagra_index* ix = nullptr;
  ok(cagra_index_create(data.data(), n, dim, graph.data(), d, 0, &ix));
  float* hq = nullptr;
  uint32_t* hid = nullptr;
  float* hd = nullptr;
  cudaMallocHost(&hq, sizeof(float) * qs.size());
  cudaMallocHost(&hid, 40);
  cudaMallocHost(&hd, 40);
  std::copy(qs.begin(), qs.end(), hq);
  cagra_search_params p;
  cagra_search_params_default(&p);
  p.k = 10;
  p.topm = topm;
  p.width = 1;
  p.seed = 11;
  cagra_engine_opts o;
  cagra_engine_opts_default(&o);
  o.mode = CAGRA_MODE_SHARED;
  o.team_count = teams;
  for (uint32_t i = 0; i < 5; ++i) ok(cagra_search(ix, hq + (size_t)i * dim, 1, dim, &p, &o, hid, hd, nullptr, nullptr));
  double hits = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t i = 0; i < nq; ++i) {
    ok(cagra_search(ix, hq + (size_t)i * dim, 1, dim, &p, &o, hid, hd, nullptr, nullptr));
    std::set<uint32_t> t(gt.begin() + i * 10, gt.begin() + i * 10 + 10);
    for (int j = 0; j < 10; ++j) hits += t.count(hid[j]);
  }
  const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"batch1_qps\": %.1f, \"latency_us\": %.1f, \"recall@10\": %.4f, \"queries\": %u, "
              "\"team_topm\": %u, \"teams\": %u, \"launches\": %u}\n",
              nq / el, el / nq * 1e6, hits / (10.0 * nq), nq, topm, teams, cagra_last_launch_count(ix));
  // device-resident query / results: kernel-only time per call (events)
  float* dq = nullptr;
  uint32_t* di = nullptr;
  float* dd = nullptr;
  const uint32_t ld = cagra_index_row_stride(ix);
  cudaMalloc(&dq, sizeof(float) * ld * nq);
  cudaMalloc(&di, 40);
  cudaMalloc(&dd, 40);
  cudaMemset(dq, 0, sizeof(float) * ld * nq);
  cudaMemcpy2D(dq, ld * 4, hq, dim * 4, dim * 4, nq, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double dev_ms = 0;
  const auto t1 = std::chrono::steady_clock::now();
  for (uint32_t i = 0; i < nq; ++i) {
    cudaEventRecord(e0, st);
    ok(cagra_search_dev(ix, dq + (size_t)i * ld, 1, &p, &o, di, dd, nullptr, nullptr, st));
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    dev_ms += ms;
  }
  const double el2 = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  std::printf("{\"device_resident_call_us\": %.1f, \"device_time_us\": %.1f}\n", el2 / nq * 1e6,
              dev_ms / nq * 1e3);
  cagra_index_destroy(ix);
  return 0;
}
