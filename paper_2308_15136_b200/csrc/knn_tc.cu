// K1 on the 5th-gen tensor cores: exact k-nearest-neighbour selection for the
// kNN graph (exact_knn_graph, knn_build.cpp:40-63) and ground truth
// (exact_topk, topk.cpp:10-43), bit-identical to the reference.
//
// 1. prep      : every fp32 row x is split into bf16 parts x = b0 + b1 + r
//                (|r| <= 2^-16 |x|) and laid out as P = [b0 | b0 | b1] (query
//                side) and R = [b0 | b1 | b0] (data side), K = 3*dim padded to
//                64, so  P_q . R_x = b0.c0 + b0.c1 + b1.c0 ~= q . x  with
//                relative error ~2^-16.  Squared norms and max |x| on the side.
// 2. knn_tc    : one CTA per 128 query rows.  The query tile (A) stays in smem
//                for the whole sweep; 128-point data tiles (B) stream through
//                a TMA ring (SWIZZLE_128B, K-major); one elected thread issues
//                tcgen05.mma kind::f16 (bf16 x bf16 -> fp32) into a
//                double-buffered TMEM accumulator (2 x 128 columns).  Four
//                epilogue warps read the accumulator with tcgen05.ld (thread =
//                query row = TMEM lane), form d~ = |q|^2 + |x|^2 - 2 q.x and
//                keep each row's KC = k + 32 smallest (d~, id) keys in a
//                per-row max-heap (L2-resident), fed through a shared-memory
//                pending buffer so a warp drains its rows together.
// 3. rerank    : per row (one warp), with delta = a rigorous bound on
//                |d~ - d| for this row, every true top-k member has
//                d~ <= d~_(k) + 2*delta; those candidates get the reference's
//                sequential fp32 distance (dataset.hpp:33-43) and the k
//                smallest by (dist, id) are written — ids and dists
//                bit-identical to the CPU.  A row whose band does not fit in
//                the KC keys is re-done by the exact SIMT kernel (counted).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int TC_BM = 128;    // query rows per CTA (= TMEM lanes)
constexpr int TC_BN = 128;    // data points per tile (= accumulator columns)
constexpr int TC_BK = 64;     // bf16 per K-block (128 B rows, SWIZZLE_128B)
constexpr int TC_STAGES = 4;  // B ring depth
constexpr int TC_PEND = 64;   // pending keys per row in smem
constexpr int TC_THREADS = 192;  // w0 TMA, w1 MMA, w2..w5 epilogue
constexpr int TC_MAX_KB = 8;  // K <= 512 keeps the query tile resident
constexpr uint32_t TILE_BYTES = TC_BN * TC_BK * 2;  // 16 KB

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, bf16 inputs, fp32 accumulate.
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
// 32 lanes x 32 consecutive columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of
// 1024 B (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (uint64_t)(1024u >> 4) << 32 | 1ull << 46 |
         2ull << 61;
}
// Instruction descriptor: fp32 accumulate, bf16 A/B, both K-major, M=128, N=128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                            ((uint32_t)(TC_BM >> 4) << 24);

struct TcArgs {
  uint32_t nq, n, kblocks, KC, exclude_self;
  const float* qnorm;  // nq
  const float* xnorm;  // n
  uint64_t* heaps;     // nq * KC
};

__device__ __forceinline__ void heap_replace_top(uint64_t* h, uint32_t KC, uint64_t e) {
  uint32_t i = 0;
  for (;;) {
    uint32_t l = 2 * i + 1;
    if (l >= KC) break;
    uint64_t big = h[l];
    uint32_t bi = l;
    if (l + 1 < KC) {
      uint64_t r = h[l + 1];
      if (r > big) {
        big = r;
        bi = l + 1;
      }
    }
    if (big <= e) break;
    h[i] = big;
    i = bi;
  }
  h[i] = e;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcArgs P) {
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B tiles
  unsigned char* base = tc_smem_raw + ((1024 - (smem_u32(tc_smem_raw) & 1023)) & 1023);
  unsigned char* sA = base;                                   // kblocks x 16 KB
  unsigned char* sB = sA + (size_t)P.kblocks * TILE_BYTES;    // STAGES x 16 KB
  uint64_t* pend = reinterpret_cast<uint64_t*>(sB + TC_STAGES * TILE_BYTES);  // PEND x 128
  uint64_t* bars = pend + TC_PEND * TC_BM;
  // bars: full[S] empty[S] afull tfull[2] tempty[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TC_STAGES + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row0 = blockIdx.x * TC_BM;
  const uint32_t ntiles = (P.n + TC_BN - 1) / TC_BN;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + TC_STAGES);
  const uint32_t afull = smem_u32(bars + 2 * TC_STAGES);
  const uint32_t tfull0 = afull + 8, tempty0 = afull + 24;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(afull, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      mbar_expect_tx(afull, P.kblocks * TILE_BYTES);
      for (uint32_t kb = 0; kb < P.kblocks; ++kb)
        tma_load_2d(smem_u32(sA + kb * TILE_BYTES), &tmA, afull, kb * TC_BK, row0);
      uint32_t it = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        for (uint32_t kb = 0; kb < P.kblocks; ++kb, ++it) {
          const uint32_t s = it % TC_STAGES, ph = (it / TC_STAGES) & 1;
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          mbar_expect_tx(full0 + 8 * s, TILE_BYTES);
          tma_load_2d(smem_u32(sB + s * TILE_BYTES), &tmB, full0 + 8 * s, kb * TC_BK,
                      t * TC_BN);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      mbar_wait(afull, 0);
      tc_fence_after();
      uint32_t it = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t acc = t & 1, aph = (t >> 1) & 1;
        mbar_wait(tempty0 + 8 * acc, aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc * TC_BN;
        for (uint32_t kb = 0; kb < P.kblocks; ++kb, ++it) {
          const uint32_t s = it % TC_STAGES, ph = (it / TC_STAGES) & 1;
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint64_t ad = sw128_desc(smem_u32(sA + kb * TILE_BYTES));
          const uint64_t bd = sw128_desc(smem_u32(sB + s * TILE_BYTES));
#pragma unroll
          for (uint32_t k = 0; k < TC_BK / 16; ++k)  // 16 bf16 = 32 B = +2 in the address field
            tc_mma(dcol, ad + 2 * k, bd + 2 * k, kIdesc, (kb | k) != 0);
          tc_commit(empty0 + 8 * s);
        }
        tc_commit(tfull0 + 8 * acc);
      }
    }
  } else {
    // ---------------- epilogue: thread = query row = TMEM lane
    const uint32_t q4 = warp & 3;               // TMEM lane quarter this warp may access
    const uint32_t rl = q4 * 32 + lane;         // row within the tile
    const uint32_t row = row0 + rl;
    const bool live = row < P.nq;
    uint64_t* heap = P.heaps + (size_t)(live ? row : 0) * P.KC;
    if (live)
      for (uint32_t i = 0; i < P.KC; ++i) heap[i] = kDummyKey;
    const float qn = live ? P.qnorm[row] : 0.0f;
    uint64_t tau = kDummyKey;
    float tau_f = __int_as_float(0x7f800000);
    uint32_t cnt = 0;
    auto flush = [&]() {
      for (uint32_t i = 0; i < cnt; ++i) {
        uint64_t e = pend[i * TC_BM + rl];
        if (e < tau) {
          heap_replace_top(heap, P.KC, e);
          tau = heap[0];
        }
      }
      cnt = 0;
      tau_f = key_dist(tau);
    };
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t acc = t & 1, aph = (t >> 1) & 1;
      mbar_wait(tfull0 + 8 * acc, aph);
      tc_fence_after();
      for (uint32_t c = 0; c < TC_BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + ((q4 * 32) << 16) + acc * TC_BN + c * 32, v);
        if (c == TC_BN / 32 - 1) {
          tc_fence_before();
          mbar_arrive(tempty0 + 8 * acc);
        }
        const uint32_t cbase = t * TC_BN + c * 32;
        const float xn_l = cbase + lane < P.n ? __ldg(P.xnorm + cbase + lane) : 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float xn = __shfl_sync(0xffffffffu, xn_l, i);
          float d = fmaf(-2.0f, __uint_as_float(v[i]), qn + xn);
          d = fmaxf(d, 0.0f);
          const uint32_t col = cbase + i;
          if (d <= tau_f && live && col < P.n && !(P.exclude_self && col == row)) {
            pend[cnt * TC_BM + rl] = make_key(d, col);
            ++cnt;
          }
        }
        if (__any_sync(0xffffffffu, cnt > TC_PEND - 32)) flush();
      }
    }
    flush();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// ----------------------------------------------------------------- prep ----
// x = b0 + b1 + r;  P = [b0 | b0 | b1 | 0],  R = [b0 | b1 | b0 | 0]
__global__ void tc_split_kernel(const float* __restrict__ src, uint32_t rows, uint32_t ld,
                                uint32_t dim, uint32_t Kp, __nv_bfloat16* __restrict__ P,
                                __nv_bfloat16* __restrict__ R, float* __restrict__ norms,
                                uint32_t* __restrict__ maxnorm_bits) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = src + (size_t)row * ld;
  __nv_bfloat16* p = P ? P + (size_t)row * Kp : nullptr;
  __nv_bfloat16* r = R ? R + (size_t)row * Kp : nullptr;
  float ss = 0.0f;
  for (uint32_t i = lane; i < Kp; i += 32) {
    if (i < dim) {
      float v = x[i];
      ss = fmaf(v, v, ss);
      __nv_bfloat16 b0 = __float2bfloat16_rn(v);
      __nv_bfloat16 b1 = __float2bfloat16_rn(v - __bfloat162float(b0));
      if (p) {
        p[i] = b0;
        p[dim + i] = b0;
        p[2 * dim + i] = b1;
      }
      if (r) {
        r[i] = b0;
        r[dim + i] = b1;
        r[2 * dim + i] = b0;
      }
    } else if (i >= 3 * dim) {
      if (p) p[i] = __float2bfloat16_rn(0.0f);
      if (r) r[i] = __float2bfloat16_rn(0.0f);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    norms[row] = ss;
    if (maxnorm_bits) atomicMax(maxnorm_bits, __float_as_uint(ss));
  }
}

// --------------------------------------------------------------- rerank ----
// One warp per query row: band selection on d~, exact sequential-chain
// distances, (dist, id) sort, first k.  Rows whose band overflows the KC keys
// are queued for the exact SIMT kernel.
__global__ void tc_rerank_kernel(const uint64_t* __restrict__ heaps, uint32_t nq, uint32_t KC,
                                 uint32_t K, const float* __restrict__ qnorm,
                                 const uint32_t* __restrict__ maxnorm_bits, float eps_rel,
                                 float eps_norm, const float* __restrict__ data, uint32_t ld,
                                 const float* __restrict__ queries, uint32_t qld, uint32_t dim,
                                 uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                                 uint32_t* __restrict__ fail_rows, uint32_t* __restrict__ fail_cnt,
                                 unsigned long long* __restrict__ reranked) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= nq) return;
  constexpr int E = 8;  // 256 keys per warp
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t i = lane * E + e;
    v[e] = i < KC ? heaps[(size_t)row * KC + i] : kDummyKey;
  }
  warp_sort_regs<E>(v, lane);
  // number of real keys (dummies sort last)
  uint32_t live = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) live += key_is_dummy(v[e]) ? 0u : 1u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
  const uint32_t src_k = (K - 1) / E, src_last = (KC - 1) / E;
  uint64_t kth = __shfl_sync(0xffffffffu, v[(K - 1) % E], src_k);
  uint64_t last = __shfl_sync(0xffffffffu, v[(KC - 1) % E], src_last);
  const float qn = qnorm[row];
  const float xm = __uint_as_float(*maxnorm_bits);
  const float delta = eps_rel * sqrtf(qn) * sqrtf(xm) + eps_norm * (qn + xm);
  const float bound = key_dist(kth) + 2.0f * delta;
  if (live == KC && key_dist(last) <= bound) {
    if (lane == 0) fail_rows[atomicAdd(fail_cnt, 1u)] = row;
    return;
  }
  const float* q = queries + (size_t)row * qld;
  uint32_t nre = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (!key_is_dummy(v[e]) && key_dist(v[e]) <= bound) {
      uint32_t id = key_id(v[e]);
      const float* x = data + (size_t)id * ld;
      float acc = 0.0f;
      for (uint32_t i = 0; i < dim; ++i) acc = seq_step(acc, __ldg(x + i), __ldg(q + i));
      v[e] = make_key(acc, id);
      ++nre;
    } else {
      v[e] = kDummyKey;
    }
  }
  warp_sort_regs<E>(v, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t i = lane * E + e;
    if (i < K) {
      out_ids[(size_t)row * K + i] = key_id(v[e]);
      out_dists[(size_t)row * K + i] = key_dist(v[e]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nre += __shfl_xor_sync(0xffffffffu, nre, o);
  if (lane == 0 && reranked) atomicAdd(reranked, (unsigned long long)nre);
}

__global__ void gather_rows_kernel(const float* __restrict__ src, uint32_t ld,
                                   const uint32_t* __restrict__ rows, uint32_t cnt,
                                   float* __restrict__ dst) {
  uint32_t r = blockIdx.x;
  if (r >= cnt) return;
  const float* s = src + (size_t)rows[r] * ld;
  for (uint32_t i = threadIdx.x; i < ld; i += blockDim.x) dst[(size_t)r * ld + i] = s[i];
}

__global__ void scatter_rows_kernel(const uint32_t* __restrict__ rows, uint32_t cnt, uint32_t K,
                                    const uint32_t* __restrict__ ids_in,
                                    const float* __restrict__ d_in, uint32_t* __restrict__ ids,
                                    float* __restrict__ dists) {
  uint32_t r = blockIdx.x;
  if (r >= cnt) return;
  for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) {
    ids[(size_t)rows[r] * K + i] = ids_in[(size_t)r * K + i];
    dists[(size_t)rows[r] * K + i] = d_in[(size_t)r * K + i];
  }
}

// ------------------------------------------------------------ host side ----
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t b) { CAGRA_CUDA_TRY(cudaMalloc(&p, b ? b : 16)); }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CAGRA_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaErr("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

CUtensorMap make_map(const void* base, uint32_t rows, uint32_t Kp) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {Kp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2};
  cuuint32_t box[2] = {TC_BK, TC_BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed");
  return tm;
}

size_t tc_smem_bytes(uint32_t kblocks) {
  return 1024 + (size_t)kblocks * TILE_BYTES + TC_STAGES * TILE_BYTES +
         sizeof(uint64_t) * (TC_PEND * TC_BM + 2 * TC_STAGES + 5) + 16;
}

}  // namespace

KnnTcStats g_knn_tc_stats;

bool knn_tc_eligible(uint32_t dim, uint32_t K) {
  const char* env = std::getenv("CAGRA_KNN_PATH");
  if (env && std::strcmp(env, "simt") == 0) return false;
  uint32_t Kp = round_up_u32(3 * dim, TC_BK);
  return Kp / TC_BK <= TC_MAX_KB && K + 32 <= 256;
}

void launch_knn_tc(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                   uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K, bool exclude_self,
                   uint32_t* d_ids, float* d_dists, cudaStream_t stream) {
  if (nq == 0) return;
  const uint32_t Kp = round_up_u32(3 * dim, TC_BK), kblocks = Kp / TC_BK;
  const uint32_t KC = K + 32;  // heap size (dummy keys pad inputs with fewer points)
  const bool same = exclude_self;  // kNN graph: queries are the data rows
  Dev dP((size_t)nq * Kp * 2), dR((size_t)n * Kp * 2), dqn(4ull * nq),
      dxn(4ull * n), dmax(4), heaps(8ull * nq * KC), fails(4ull * nq + 4), rer(8);
  CAGRA_CUDA_TRY(cudaMemsetAsync(dmax.p, 0, 4, stream));
  CAGRA_CUDA_TRY(cudaMemsetAsync(fails.p, 0, 4ull * nq + 4, stream));
  CAGRA_CUDA_TRY(cudaMemsetAsync(rer.p, 0, 8, stream));
  // data side: R (and P when the queries are the data), norms, max norm
  tc_split_kernel<<<(n + 7) / 8, 256, 0, stream>>>(d_data, n, ld, dim, Kp,
                                                   same ? dP.as<__nv_bfloat16>() : nullptr,
                                                   dR.as<__nv_bfloat16>(), dxn.as<float>(),
                                                   dmax.as<uint32_t>());
  CAGRA_LAUNCH_CHECK();
  const float* qnorm = dxn.as<float>();
  if (!same) {
    tc_split_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(d_queries, nq, qld, dim, Kp,
                                                      dP.as<__nv_bfloat16>(), nullptr,
                                                      dqn.as<float>(), nullptr);
    CAGRA_LAUNCH_CHECK();
    qnorm = dqn.as<float>();
  }
  CUtensorMap tmA = make_map(dP.p, nq, Kp), tmB = make_map(dR.p, n, Kp);
  TcArgs a;
  a.nq = nq;
  a.n = n;
  a.kblocks = kblocks;
  a.KC = KC;
  a.exclude_self = exclude_self ? 1 : 0;
  a.qnorm = qnorm;
  a.xnorm = dxn.as<float>();
  a.heaps = heaps.as<uint64_t>();
  size_t smem = tc_smem_bytes(kblocks);
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  knn_tc_kernel<<<(nq + TC_BM - 1) / TC_BM, TC_THREADS, smem, stream>>>(tmA, tmB, a);
  CAGRA_LAUNCH_CHECK();
  // error bound of d~ (see file header): split ~3.1*2^-16, fp32 accumulation
  // over Kp terms, norms over dim terms; x2 for the -2 q.x term.
  const float eps_rel = 2.0f * (3.1f * 1.52587890625e-05f + (float)Kp * 1.1920929e-07f);
  const float eps_norm = (float)(dim + 8) * 2.384185791e-07f;
  uint32_t* fail_rows = fails.as<uint32_t>() + 1;
  uint32_t* fail_cnt = fails.as<uint32_t>();
  tc_rerank_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(
      heaps.as<uint64_t>(), nq, KC, K, qnorm, dmax.as<uint32_t>(), eps_rel, eps_norm, d_data, ld,
      d_queries, qld, dim, d_ids, d_dists, fail_rows, fail_cnt,
      rer.as<unsigned long long>());
  CAGRA_LAUNCH_CHECK();
  uint32_t nf = 0;
  unsigned long long nre = 0;
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&nf, fail_cnt, 4, cudaMemcpyDeviceToHost, stream));
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&nre, rer.p, 8, cudaMemcpyDeviceToHost, stream));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
  g_knn_tc_stats.rows = nq;
  g_knn_tc_stats.fallback_rows = nf;
  g_knn_tc_stats.reranked = nre;
  if (nf) {
    // exact SIMT kernel for the rows whose candidate band overflowed
    Dev q((size_t)nf * qld * 4), sc(8ull * nf * K), fi(4ull * nf * K), fd(4ull * nf * K);
    gather_rows_kernel<<<nf, 128, 0, stream>>>(d_queries, qld, fail_rows, nf, q.as<float>());
    CAGRA_LAUNCH_CHECK();
    launch_exact_topk_simt(d_data, n, ld, q.as<float>(), nf, qld, dim, K, exclude_self,
                           exclude_self ? fail_rows : nullptr, sc.as<uint64_t>(),
                           fi.as<uint32_t>(), fd.as<float>(), stream);
    scatter_rows_kernel<<<nf, 128, 0, stream>>>(fail_rows, nf, K, fi.as<uint32_t>(),
                                                fd.as<float>(), d_ids, d_dists);
    CAGRA_LAUNCH_CHECK();
    CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
  }
}

}  // namespace cagra
