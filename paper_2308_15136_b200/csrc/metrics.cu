// Graph quality metrics on the device (graph_metrics.hpp):
//
//  * avg_2hop_count (graph_metrics.cpp:78-120): per node v, the number of
//    distinct u != v reachable in <= 2 edges.  One CTA per node (grid-stride),
//    the node's d + d^2 candidates inserted into a CTA-private open-addressing
//    set (shared memory, or a global scratch slice for very large degrees);
//    successful inserts are counted.  The exact integer total is returned, so
//    total / n equals the reference's double bit for bit.
//
//  * strong_cc_count (graph_metrics.cpp:20-76, iterative Tarjan there): the
//    number of strongly connected components by trimming + forward colouring
//    on the device.  Each round: nodes left with no live in- or out-edge are
//    singleton components; every live node takes the largest id that reaches
//    it (max-label propagation to a fixpoint); a node whose colour is its own
//    id roots a component = the nodes of its colour that reach it (backward
//    closure inside the colour, again to a fixpoint).  Those components are
//    counted and removed.  The live node of largest id is always a root, so
//    every round removes at least one component.
#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int MT_NT = 256;

__global__ void __launch_bounds__(MT_NT)
two_hop_kernel(const uint32_t* __restrict__ g, uint32_t n, uint32_t d, uint32_t H,
               uint32_t* __restrict__ gscratch, unsigned long long* __restrict__ total) {
  extern __shared__ __align__(16) uint32_t set_smem[];
  uint32_t* set = gscratch ? gscratch + (size_t)blockIdx.x * H : set_smem;
  const uint32_t mask = H - 1, cand = d + d * d;
  unsigned long long mine = 0;
  for (uint32_t v = blockIdx.x; v < n; v += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < H; i += MT_NT) set[i] = kInvalidId;
    __syncthreads();
    const uint32_t* row = g + (size_t)v * d;
    for (uint32_t j = threadIdx.x; j < cand; j += MT_NT) {
      // j < d: the first hop row[j]; else the second hop row[a][b]
      uint32_t u;
      if (j < d) {
        u = __ldg(row + j);
      } else {
        const uint32_t a = (j - d) / d, b = (j - d) - a * d;
        u = __ldg(g + (size_t)__ldg(row + a) * d + b);
      }
      if (u == v) continue;
      uint32_t h = hash_id(u, mask);
      for (;;) {
        const uint32_t old = atomicCAS(&set[h], kInvalidId, u);
        if (old == kInvalidId) {
          ++mine;
          break;
        }
        if (old == u) break;
        h = (h + 1) & mask;
      }
    }
    __syncthreads();
  }
  // block reduction of the per-thread insert counts
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  __shared__ unsigned long long wsum[MT_NT / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < MT_NT / 32; ++w) s += wsum[w];
    atomicAdd(total, s);
  }
}

// ---- strongly connected components -----------------------------------------
// live[v]: 1 while v is not yet assigned to a component.

// in-degree over live edges (self-loops excluded)
__global__ void scc_indeg_kernel(const uint32_t* __restrict__ g, uint32_t n, uint32_t d,
                                 const uint8_t* __restrict__ live, uint32_t* __restrict__ indeg) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (uint64_t)n * d) return;
  const uint32_t v = (uint32_t)(e / d), w = g[e];
  if (live[v] && live[w] && w != v) atomicAdd(&indeg[w], 1u);
}

// nodes with no live in-edge or no live out-edge (other than to themselves)
// are singleton components
__global__ void scc_trim_kernel(const uint32_t* __restrict__ g, uint32_t n, uint32_t d,
                                uint8_t* __restrict__ live, const uint32_t* __restrict__ indeg,
                                unsigned long long* __restrict__ count, int* __restrict__ changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !live[v]) return;
  bool out = false;
  for (uint32_t j = 0; j < d && !out; ++j) {
    const uint32_t w = g[(size_t)v * d + j];
    out = w != v && live[w];
  }
  if (!out || indeg[v] == 0) {
    live[v] = 0;
    atomicAdd(count, 1ull);
    *changed = 1;
  }
}

__global__ void scc_color_init_kernel(uint32_t n, const uint8_t* __restrict__ live,
                                      uint32_t* __restrict__ color, uint8_t* __restrict__ mark) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  color[v] = live[v] ? v : kInvalidId;
  mark[v] = 0;
}

// colour[w] = max(colour[w], colour[v]) along live edges v -> w
__global__ void scc_propagate_kernel(const uint32_t* __restrict__ g, uint32_t n, uint32_t d,
                                     const uint8_t* __restrict__ live, uint32_t* __restrict__ color,
                                     int* __restrict__ changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !live[v]) return;
  const uint32_t c = color[v];
  bool ch = false;
  for (uint32_t j = 0; j < d; ++j) {
    const uint32_t w = g[(size_t)v * d + j];
    if (live[w] && color[w] < c) {  // volatile-free: a stale read only costs a sweep
      atomicMax(&color[w], c);
      ch = true;
    }
  }
  if (ch) *changed = 1;
}

// roots: colour == own id
__global__ void scc_roots_kernel(uint32_t n, const uint8_t* __restrict__ live,
                                 const uint32_t* __restrict__ color, uint8_t* __restrict__ mark,
                                 unsigned long long* __restrict__ count) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !live[v] || color[v] != v) return;
  mark[v] = 1;
  atomicAdd(count, 1ull);
}

// v joins its colour's component if it has an edge into a marked node of the
// same colour (backward closure from the root)
__global__ void scc_backward_kernel(const uint32_t* __restrict__ g, uint32_t n, uint32_t d,
                                    const uint8_t* __restrict__ live,
                                    const uint32_t* __restrict__ color, uint8_t* __restrict__ mark,
                                    int* __restrict__ changed) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !live[v] || mark[v]) return;
  const uint32_t c = color[v];
  for (uint32_t j = 0; j < d; ++j) {
    const uint32_t w = g[(size_t)v * d + j];
    if (live[w] && color[w] == c && *(volatile uint8_t*)&mark[w]) {
      mark[v] = 1;
      *changed = 1;
      return;
    }
  }
}

__global__ void scc_remove_kernel(uint32_t n, uint8_t* __restrict__ live,
                                  const uint8_t* __restrict__ mark, int* __restrict__ any_live) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || !live[v]) return;
  if (mark[v]) live[v] = 0;
  else *any_live = 1;
}

int blocks_for(uint64_t work) { return (int)std::max<uint64_t>(1, (work + MT_NT - 1) / MT_NT); }

struct Scratch {
  void* p = nullptr;
  explicit Scratch(size_t b) { CAGRA_CUDA_TRY(cudaMalloc(&p, b ? b : 16)); }
  ~Scratch() { cudaFree(p); }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

int read_int(const int* d_v, cudaStream_t s) {
  int h = 0;
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&h, d_v, sizeof(int), cudaMemcpyDeviceToHost, s));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

uint64_t two_hop_total(const uint32_t* d_graph, uint32_t n, uint32_t d, int sm_count,
                       cudaStream_t s) {
  if (n == 0 || d == 0) return 0;
  uint64_t want = 1;
  while (want < 2ull * ((uint64_t)d + (uint64_t)d * d)) want <<= 1;  // load factor <= 1/2
  const uint32_t H = (uint32_t)want;
  const size_t smem = 4ull * H;
  const bool in_smem = smem <= 96 * 1024;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(n, (uint64_t)sm_count * (in_smem ? 4 : 2));
  Scratch tot(8), glob(in_smem ? 0 : smem * grid);
  CAGRA_CUDA_TRY(cudaMemsetAsync(tot.p, 0, 8, s));
  if (in_smem)
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(two_hop_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  two_hop_kernel<<<grid, MT_NT, in_smem ? smem : 0, s>>>(
      d_graph, n, d, H, in_smem ? nullptr : glob.as<uint32_t>(), tot.as<unsigned long long>());
  CAGRA_LAUNCH_CHECK();
  unsigned long long h = 0;
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&h, tot.p, 8, cudaMemcpyDeviceToHost, s));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  return h;
}

uint64_t scc_count(const uint32_t* d_graph, uint32_t n, uint32_t d, cudaStream_t s) {
  if (n == 0) return 0;
  Scratch live(n), mark(n), color(4ull * n), indeg(4ull * n), cnt(8), flag(sizeof(int));
  CAGRA_CUDA_TRY(cudaMemsetAsync(live.p, 1, n, s));
  CAGRA_CUDA_TRY(cudaMemsetAsync(cnt.p, 0, 8, s));
  const int nb = blocks_for(n), eb = blocks_for((uint64_t)n * d);
  auto* L = live.as<uint8_t>();
  auto* M = mark.as<uint8_t>();
  auto* C = color.as<uint32_t>();
  auto* F = flag.as<int>();
  auto* K = cnt.as<unsigned long long>();
  for (;;) {
    // trim to a fixpoint (cheap sweeps; removes the many singleton components)
    for (int t = 0; t < 64; ++t) {
      CAGRA_CUDA_TRY(cudaMemsetAsync(indeg.p, 0, 4ull * n, s));
      CAGRA_CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(int), s));
      if (d) scc_indeg_kernel<<<eb, MT_NT, 0, s>>>(d_graph, n, d, L, indeg.as<uint32_t>());
      scc_trim_kernel<<<nb, MT_NT, 0, s>>>(d_graph, n, d, L, indeg.as<uint32_t>(), K, F);
      CAGRA_LAUNCH_CHECK();
      if (!read_int(F, s)) break;
    }
    scc_color_init_kernel<<<nb, MT_NT, 0, s>>>(n, L, C, M);
    do {
      CAGRA_CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(int), s));
      scc_propagate_kernel<<<nb, MT_NT, 0, s>>>(d_graph, n, d, L, C, F);
      CAGRA_LAUNCH_CHECK();
    } while (read_int(F, s));
    scc_roots_kernel<<<nb, MT_NT, 0, s>>>(n, L, C, M, K);
    do {
      CAGRA_CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(int), s));
      scc_backward_kernel<<<nb, MT_NT, 0, s>>>(d_graph, n, d, L, C, M, F);
      CAGRA_LAUNCH_CHECK();
    } while (read_int(F, s));
    CAGRA_CUDA_TRY(cudaMemsetAsync(F, 0, sizeof(int), s));
    scc_remove_kernel<<<nb, MT_NT, 0, s>>>(n, L, M, F);
    CAGRA_LAUNCH_CHECK();
    if (!read_int(F, s)) break;
  }
  unsigned long long h = 0;
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&h, K, 8, cudaMemcpyDeviceToHost, s));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  return h;
}

}  // namespace cagra
