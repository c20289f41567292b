// Exact k-nearest-neighbour tiles: ground truth (exact_topk, topk.cpp:10-43)
// and the exact kNN graph (exact_knn_graph, knn_build.cpp:40-63).
//
// Every distance is the reference's sequential fp32 chain
//   acc = acc + (x_i - q_i)^2   for i = 0 .. dim-1, each op rounded
// (dataset.hpp:33-43).  A register-blocked tile keeps 32 independent chains
// per thread, all advancing in dimension order, so the blocking never
// reassociates a sum: results are bit-identical to the CPU reference and the
// (dist, id) tie order of exact_topk is reproduced exactly.
//
// Layout: a CTA owns BQ=64 query rows and streams the whole dataset in tiles
// of BN=128 points x BK=32 dims through shared memory.  Candidates beating a
// row's current k-th key are appended to a per-row shared buffer; a warp
// merges a row's buffer into its running top-k (kept in global memory) when
// the buffer passes half capacity.  Insertions decay like k*ln(N/k), so the
// merges cost little after the first tiles.
#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int BQ = 64;
constexpr int BN = 128;
constexpr int BK = 32;
constexpr int NT = 256;
constexpr int CAP = 192;                // per-row candidate buffer
constexpr int MERGE_AT = CAP - BN;      // merge when a row holds more than this
constexpr int QS = BQ + 1;              // padded strides (bank-conflict free)
constexpr int XS = BN + 1;
constexpr int MAX_K = 1024;

__device__ __forceinline__ uint32_t lower_bound_smem(const uint64_t* a, uint32_t len,
                                                     uint64_t key) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Warp-cooperative bitonic sort of a[0..P) (P power of two) in shared memory.
__device__ __forceinline__ void warp_bitonic_sort(uint64_t* a, uint32_t P, int lane) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = lane; i < P; i += 32) {
        uint32_t ixj = i ^ j;
        if (ixj > i) {
          uint64_t x = a[i], y = a[ixj];
          bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Merge row r's candidate buffer into its global top-K list (see file header).
__device__ void merge_row(int r, uint32_t K, uint64_t* __restrict__ row_topk, uint64_t* buf_r,
                          uint32_t* cnt, uint64_t* thr, uint64_t* scratchT, uint64_t* scratchB,
                          int lane) {
  uint32_t c = cnt[r];
  if (c == 0) return;
  uint32_t P = next_pow2_u32(c);
  for (uint32_t i = lane; i < P; i += 32) scratchB[i] = i < c ? buf_r[i] : kDummyKey;
  for (uint32_t i = lane; i < K; i += 32) scratchT[i] = row_topk[i];
  __syncwarp();
  warp_bitonic_sort(scratchB, P, lane);
  for (uint32_t j = lane; j < c; j += 32) {
    uint64_t v = scratchB[j];
    uint32_t pos = j + lower_bound_smem(scratchT, K, v);
    if (pos < K) row_topk[pos] = v;
  }
  for (uint32_t i = lane; i < K; i += 32) {
    uint64_t v = scratchT[i];
    uint32_t pos = i + lower_bound_smem(scratchB, c, v);
    if (pos < K) row_topk[pos] = v;
  }
  __syncwarp();
  __threadfence_block();
  if (lane == 0) {
    thr[r] = row_topk[K - 1];
    cnt[r] = 0;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(NT, 1)
exact_topk_kernel(const float* __restrict__ data, uint32_t n, uint32_t ld,
                  const float* __restrict__ queries, uint32_t nq, uint32_t qld, uint32_t dim,
                  uint32_t K, int exclude_self, const uint32_t* __restrict__ self_ids,
                  uint64_t* __restrict__ topk,
                  uint32_t* __restrict__ out_ids, float* __restrict__ out_dists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw);            // BQ*CAP
  uint64_t* thr = buf + BQ * CAP;                                    // BQ
  uint64_t* scratch = thr + BQ;                                      // 8 warps*(K+256)
  float* Qs = reinterpret_cast<float*>(scratch + (NT / 32) * (K + 256));  // BK*QS
  float* Xs = Qs + BK * QS;                                          // BK*XS
  uint32_t* cnt = reinterpret_cast<uint32_t*>(Xs + BK * XS);         // BQ
  __shared__ int need_merge;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ty = tid >> 4, tx = tid & 15;
  const uint32_t q0 = blockIdx.x * BQ;
  uint64_t* scratchT = scratch + warp * (K + 256);
  uint64_t* scratchB = scratchT + K;

  for (int r = tid; r < BQ; r += NT) {
    thr[r] = kDummyKey;
    cnt[r] = 0;
  }
  for (uint32_t i = tid; i < BQ * K; i += NT) {
    uint32_t r = i / K;
    if (q0 + r < nq) topk[(size_t)(q0 + r) * K + (i % K)] = kDummyKey;
  }
  if (tid == 0) need_merge = 0;
  __syncthreads();

  for (uint32_t t0 = 0; t0 < n; t0 += BN) {
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;

    for (uint32_t k0 = 0; k0 < dim; k0 += BK) {
      __syncthreads();
      // Q tile: BQ rows x BK dims, stored Qs[k][row]
      for (int i = tid; i < BQ * BK; i += NT) {
        int row = i / BK, kk = i % BK;
        uint32_t qi = q0 + row, d = k0 + kk;
        Qs[kk * QS + row] = (qi < nq && d < dim) ? queries[(size_t)qi * qld + d] : 0.0f;
      }
      // X tile: BN points x BK dims, stored Xs[k][point]
      for (int i = tid; i < BN * BK; i += NT) {
        int p = i / BK, kk = i % BK;
        uint32_t j = t0 + p, d = k0 + kk;
        Xs[kk * XS + p] = (j < n && d < dim) ? __ldg(&data[(size_t)j * ld + d]) : 0.0f;
      }
      __syncthreads();
      uint32_t kend = min((uint32_t)BK, dim - k0);
      for (uint32_t kk = 0; kk < kend; ++kk) {
        float qv[4], xv[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) qv[r] = Qs[kk * QS + ty + 16 * r];
#pragma unroll
        for (int c = 0; c < 8; ++c) xv[c] = Xs[kk * XS + tx + 16 * c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = seq_step(acc[r][c], xv[c], qv[r]);
      }
    }
    // append candidates that beat the row threshold
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int row = ty + 16 * r;
      uint32_t qi = q0 + row;
      if (qi >= nq) continue;
      uint64_t th = thr[row];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t j = t0 + tx + 16 * c;
        if (j >= n || (exclude_self && j == (self_ids ? self_ids[qi] : qi))) continue;
        uint64_t key = make_key(acc[r][c], j);
        if (key < th) {
          uint32_t slot = atomicAdd(&cnt[row], 1u);
          buf[row * CAP + slot] = key;
          if (slot + 1 > (uint32_t)MERGE_AT) need_merge = 1;
        }
      }
    }
    __syncthreads();
    if (need_merge) {
      for (int row = warp; row < BQ; row += NT / 32) {
        if (cnt[row] > (uint32_t)MERGE_AT && q0 + row < nq)
          merge_row(row, K, topk + (size_t)(q0 + row) * K, buf + row * CAP, cnt, thr, scratchT,
                    scratchB, lane);
      }
      __syncthreads();
      if (tid == 0) need_merge = 0;
      __syncthreads();
    }
  }
  // final flush
  for (int row = warp; row < BQ; row += NT / 32) {
    if (q0 + row < nq)
      merge_row(row, K, topk + (size_t)(q0 + row) * K, buf + row * CAP, cnt, thr, scratchT,
                scratchB, lane);
  }
  __syncthreads();
  __threadfence_block();
  for (uint32_t i = tid; i < BQ * K; i += NT) {
    uint32_t r = i / K, qi = q0 + r;
    if (qi >= nq) continue;
    uint64_t v = topk[(size_t)qi * K + (i % K)];
    out_ids[(size_t)qi * K + (i % K)] = key_id(v);
    out_dists[(size_t)qi * K + (i % K)] = key_dist(v);
  }
}

size_t exact_topk_smem(uint32_t K) {
  return sizeof(uint64_t) * (BQ * CAP + BQ + (NT / 32) * (K + 256)) +
         sizeof(float) * (BK * QS + BK * XS) + sizeof(uint32_t) * BQ;
}

}  // namespace

__global__ void iota_kernel(uint32_t* __restrict__ out, uint32_t cnt, uint32_t base) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) out[i] = base + i;
}

void launch_exact_topk_simt(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                            uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K,
                            bool exclude_self, const uint32_t* d_self_ids,
                            uint64_t* d_topk_scratch, uint32_t* d_ids, float* d_dists,
                            cudaStream_t stream) {
  if (K > MAX_K) throw UsageErr("device exact top-k supports k <= 1024");
  if (nq == 0) return;
  size_t smem = exact_topk_smem(K);
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(exact_topk_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((nq + BQ - 1) / BQ);
  exact_topk_kernel<<<grid, NT, smem, stream>>>(d_data, n, ld, d_queries, nq, qld, dim, K,
                                                exclude_self ? 1 : 0, d_self_ids, d_topk_scratch,
                                                d_ids, d_dists);
  CAGRA_LAUNCH_CHECK();
}

void launch_exact_topk(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                       uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K, bool exclude_self,
                       uint32_t* d_ids, float* d_dists, cudaStream_t stream, uint32_t self_base) {
  if (K > MAX_K) throw UsageErr("device exact top-k supports k <= 1024");
  if (nq == 0) return;
  if (knn_tc_eligible(dim, K)) {
    launch_knn_tc(d_data, n, ld, d_queries, nq, qld, dim, K, exclude_self, self_base, d_ids,
                  d_dists, stream);
    return;
  }
  g_knn_tc_stats = KnnTcStats{};
  uint64_t* sc = nullptr;
  uint32_t* self = nullptr;
  CAGRA_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&sc), sizeof(uint64_t) * nq * K,
                                 stream));
  if (exclude_self && self_base) {
    CAGRA_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&self), sizeof(uint32_t) * nq, stream));
    iota_kernel<<<(nq + 255) / 256, 256, 0, stream>>>(self, nq, self_base);
    CAGRA_LAUNCH_CHECK();
  }
  launch_exact_topk_simt(d_data, n, ld, d_queries, nq, qld, dim, K, exclude_self, self, sc,
                         d_ids, d_dists, stream);
  CAGRA_CUDA_TRY(cudaFreeAsync(sc, stream));
  if (self) CAGRA_CUDA_TRY(cudaFreeAsync(self, stream));
}

}  // namespace cagra
