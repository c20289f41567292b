// K1 on the 5th-gen tensor cores: exact k-nearest-neighbour selection for the
// kNN graph (exact_knn_graph, knn_build.cpp:40-63) and ground truth
// (exact_topk, topk.cpp:10-43), bit-identical to the reference.
//
// 1. prep      : every fp32 row x is split into bf16 parts x = b0 + b1 + r
//                (|r| <= 2^-16 |x|), its squared norm n = n0 + n1 + n2 likewise,
//                and laid out as
//                  P_q = [-2b0 | -2b0 | -2b1 | 1 1 1 | n0 n1 n2 | 0..]  (query)
//                  R_x = [  c0 |   c1 |   c0 | m0 m1 m2 | 1 1 1 | 0..]  (data)
//                (K = 3*dim + 6 padded to 64), so the GEMM itself yields
//                  P_q . R_x = |q|^2 + |x|^2 - 2 (b0.c0 + b0.c1 + b1.c0) = d~
//                with relative error ~2^-16 on the cross term.
// 2. knn_tc    : one CTA per 128 query rows.  The query tile (A) stays in smem
//                for the whole sweep; 128-point data tiles (B) stream through
//                a TMA ring (SWIZZLE_128B, K-major); one elected thread issues
//                tcgen05.mma kind::f16 (bf16 x bf16 -> fp32) into a
//                double-buffered TMEM accumulator (2 x 128 columns).  Four
//                epilogue warps read d~ from the accumulator with tcgen05.ld
//                (thread = query row = TMEM lane), build a 32-bit pass mask
//                per 32 columns against the row's threshold (branch-free),
//                append passing (d~, id) keys to a shared-memory pending
//                buffer, and a warp merges full buffers into each row's sorted
//                list of the KC = k + 32 smallest keys (L2-resident) with a
//                warp-wide bitonic sort; the threshold is the list's last key.
//                Two passes when N >= 64k: pass 1 runs this over every 16th
//                point keeping the r smallest (r ~ 3(k+16)/16); the r-th
//                smallest d~ of any subset is an upper bound tau* of the r-th
//                smallest overall, so pass 2 over all points just appends
//                every d~ <= tau* (~3(k+16) per row) — no merging.  Rows
//                whose tau* does not bracket their band re-run single-pass.
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
#include <cstdio>
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
constexpr int TC_STAGES = 8;  // max B ring depth (as smem allows)
constexpr int TC_PEND = 48;   // pending keys per row in smem (list mode)
constexpr int TC_PEND_APPEND = 32;  // append mode: spills are cheap, smem goes to the TMA ring
constexpr int TC_THREADS = 192;  // w0 TMA, w1 MMA, w2..w5 epilogue
constexpr int TC_EPI_WARPS = 4;
// A (the CTA's query tile, constant for the whole sweep) lives in TMEM and the
// MMA reads it from there (tcgen05.mma ... [a_tmem]): shared memory only
// feeds B, halving the operand traffic that bounds the SS form.
#ifndef CAGRA_KNN_TS
#define CAGRA_KNN_TS 1
#endif
constexpr uint32_t TC_A_COL = 2 * 128;         // TS: A at TMEM columns [256, 256 + Kp/2)
constexpr int TC_MAX_KB = 8;  // K <= 512 keeps the query tile resident
constexpr int TC_MAX_KB_STREAM = 64;  // beyond: query tile streamed with each data tile (SA)
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
#ifndef CAGRA_TC_WATCHDOG
#define CAGRA_TC_WATCHDOG 0  // 1: trap a barrier wait that exceeds ~10 s (pipeline debugging)
#endif

// ---- CTA-pair (cluster of 2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// arrive on the barrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar),
      "r"(cta)
      : "memory");
}
// 2-SM TMA: each CTA loads its share, completion counted on the LEADER's
// barrier (peer bit cleared in the barrier address).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* tm, uint32_t bar,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, M split over the pair] . B[smem, N split]^T
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit: arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"((unsigned short)3)
      : "memory");
}

// Waits for the barrier phase; a wait that never completes (a pipeline bug)
// traps after ~10 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
#if CAGRA_TC_WATCHDOG
  const long long t0 = clock64();
#endif
  do {
#if CAGRA_TC_WATCHDOG
    if (clock64() - t0 > 20000000000ll) __trap();
#endif
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
// D[tmem] (+)= A[tmem] . B[smem]^T (A: lane = row, 2 bf16 per 32-bit column).
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 32 consecutive columns <- 32 registers per thread.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
// 32 lanes x 32 consecutive columns -> 32 registers per thread (no wait).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
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
  uint32_t nq, n, kblocks, KC, exclude_self, stages, pend_cap;
  uint32_t mode;        // 0: running sorted list of KC keys; 1: append d~ <= fixed tau
  uint32_t col_stride;  // B row c is data point c * col_stride (sample pass)
  uint64_t* lists;      // mode 0: nq * KC sorted keys (dist bits << 32 | id)
  const uint64_t* tau_keys;  // mode 1: row's threshold = key_dist(tau_keys[row * tau_ld + tau_ld - 1])
  uint32_t tau_ld;
  uint64_t* bufs;       // mode 1: nq * capg appended keys
  uint32_t* bcount;     // mode 1: keys appended per row (> capg: overflow), zeroed by the host
  uint32_t capg;
  const uint32_t* self_ids;  // optional: data id of each query row (self exclusion)
  uint32_t self_base;        // else: query row r is data point self_base + r
  const uint32_t* prow;      // TS: query-side rows (nq x Kp bf16, as Kp/2 u32) for TMEM
  uint32_t groups;           // CTAs start their sweep at one of `groups` evenly spaced tiles
};

// PAIR: a cluster of 2 CTAs shares each data tile: every CTA keeps its own
// 128 query rows (A, smem) and loads HALF of the 128-point B tile; the leader
// issues tcgen05.mma.cta_group::2 (M = 256) and each CTA's TMEM receives its
// rows x all 128 points.  Per-SM B traffic from L2 halves.
// SA (K > 512, e.g. 960-d): the query tile does not fit next to the ring, so
// every stage carries the A k-block together with the B k-block (a plain
// streamed GEMM main loop; A is re-read from L2 once per data tile).
template <bool PAIR, bool SA = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcArgs P) {
  static_assert(!(PAIR && SA), "streamed A is single-CTA");
  constexpr bool TS = CAGRA_KNN_TS && !PAIR && !SA;
  // SA data tiles are 256 points wide (one N=256 MMA per k-block), so every
  // streamed A k-block is used against two 128-point B tiles
  constexpr uint32_t W = SA ? 2 * TC_BN : TC_BN;  // data points per tile
  constexpr int ACC = TS || SA ? 2 : 4;           // W-column accumulators in 512 TMEM columns
  constexpr uint32_t BTILE = PAIR ? TILE_BYTES / 2 : TILE_BYTES;  // B bytes per stage per CTA
  constexpr uint32_t STAGE = SA ? 3 * TILE_BYTES : BTILE;         // [A k-block |] B k-block(s)
  constexpr uint32_t idesc = PAIR ? ((1u << 4) | (1u << 7) | (1u << 10) |
                                     ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24))
                           : SA ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(W >> 3) << 17) |
                                   ((uint32_t)(TC_BM >> 4) << 24))
                                : kIdesc;
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B tiles
  unsigned char* base = tc_smem_raw + ((1024 - (smem_u32(tc_smem_raw) & 1023)) & 1023);
  unsigned char* sA = base;                                   // SS: kblocks x 16 KB
  unsigned char* sB = sA + (TS || SA ? 0 : (size_t)P.kblocks * TILE_BYTES);  // stages x STAGE
  uint64_t* pend = reinterpret_cast<uint64_t*>(sB + P.stages * STAGE);  // PEND x 128
  uint64_t* bars = pend + P.pend_cap * TC_BM;
  // bars: full[S] empty[S] afull tfull[ACC] tempty[ACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P.stages + 1 + 2 * ACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const uint32_t row0 = PAIR ? (blockIdx.x >> 1) * 2 * TC_BM + rank * TC_BM : blockIdx.x * TC_BM;
  const uint32_t ntiles = (P.n + W - 1) / W;
  const uint32_t S = P.stages;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
  const uint32_t afull = smem_u32(bars + 2 * S);
  const uint32_t tfull0 = afull + 8, tempty0 = afull + 8 + 8 * ACC;
  // Staggered sweep: CTAs of group g start at tile g*ntiles/groups, so the
  // resident CTAs spread their B-tile reads over `groups` regions of L2
  // instead of all hitting the same lines (results do not depend on order).
  const uint32_t start_tile =
      !PAIR && P.groups > 1 ? (uint32_t)(((uint64_t)(blockIdx.x % P.groups) * ntiles) / P.groups)
                            : 0u;
  auto tile_of = [&](uint32_t t) {
    const uint32_t x = t + start_tile;
    return x >= ntiles ? x - ntiles : x;
  };

  if (threadIdx.x == 0) {
    // PAIR: full/afull/tempty are counted on the leader (both CTAs arrive);
    // empty/tfull get the leader's multicast commit in each CTA
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, PAIR ? 2 : 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(afull, TS ? 4 : (PAIR ? 2 : 1));  // TS: the 4 epilogue warps write A
    for (int a = 0; a < ACC; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, (PAIR ? 2 : 1) * TC_EPI_WARPS);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      if (PAIR) {
        // own 128 rows of A; the leader's barrier counts both CTAs' bytes
        for (uint32_t kb = 0; kb < P.kblocks; ++kb)
          tma_load_2d_pair(smem_u32(sA + kb * TILE_BYTES), &tmA, afull, kb * TC_BK, row0);
        if (leader) mbar_expect_tx(afull, 2 * P.kblocks * TILE_BYTES);
        else mbar_arrive_remote(afull, 0);
      } else if (SA) {
        mbar_arrive(afull);  // nothing resident: A arrives with every stage
      } else if (!TS) {
        mbar_expect_tx(afull, P.kblocks * TILE_BYTES);
        for (uint32_t kb = 0; kb < P.kblocks; ++kb)
          tma_load_2d(smem_u32(sA + kb * TILE_BYTES), &tmA, afull, kb * TC_BK, row0);
      }
      uint32_t it = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        for (uint32_t kb = 0; kb < P.kblocks; ++kb, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1;
          mbar_wait(empty0 + 8 * s, ph ^ 1);
          if (PAIR) {
            // this CTA's half of the tile: points [tile*128 + rank*64, +64)
            tma_load_2d_pair(smem_u32(sB + s * BTILE), &tmB, full0 + 8 * s, kb * TC_BK,
                             tile_of(t) * TC_BN + rank * (TC_BN / 2));
            if (leader) mbar_expect_tx(full0 + 8 * s, 2 * BTILE);
            else mbar_arrive_remote(full0 + 8 * s, 0);
          } else if (SA) {
            // A k-block, then the two 128-row halves of the 256-point B k-block
            // back to back (one K-major SWIZZLE_128B operand of 256 rows)
            mbar_expect_tx(full0 + 8 * s, 3 * TILE_BYTES);
            tma_load_2d(smem_u32(sB + s * STAGE), &tmA, full0 + 8 * s, kb * TC_BK, row0);
            tma_load_2d(smem_u32(sB + s * STAGE + TILE_BYTES), &tmB, full0 + 8 * s, kb * TC_BK,
                        tile_of(t) * W);
            tma_load_2d(smem_u32(sB + s * STAGE + 2 * TILE_BYTES), &tmB, full0 + 8 * s,
                        kb * TC_BK, tile_of(t) * W + TC_BN);
          } else {
            mbar_expect_tx(full0 + 8 * s, TILE_BYTES);
            tma_load_2d(smem_u32(sB + s * TILE_BYTES), &tmB, full0 + 8 * s, kb * TC_BK,
                        tile_of(t) * TC_BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread; the leader's, for a pair)
    if (lane == 0 && leader) {
      mbar_wait(afull, 0);
      tc_fence_after();
      uint32_t it = 0;
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t acc = t % ACC, aph = (t / ACC) & 1;
        mbar_wait(tempty0 + 8 * acc, aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc * W;
        for (uint32_t kb = 0; kb < P.kblocks; ++kb, ++it) {
          const uint32_t s = it % S, ph = (it / S) & 1;
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint64_t bd = sw128_desc(smem_u32(sB + s * STAGE + (SA ? TILE_BYTES : 0)));
          if (TS) {
#pragma unroll
            for (uint32_t k = 0; k < TC_BK / 16; ++k)  // A: 16 bf16 = 8 TMEM columns per step
              tc_mma_ts(dcol, tmem + TC_A_COL + kb * (TC_BK / 2) + k * 8, bd + 2 * k, idesc,
                        (kb | k) != 0);
          } else {
            const uint64_t ad = sw128_desc(smem_u32(SA ? sB + s * STAGE : sA + kb * TILE_BYTES));
#pragma unroll
            for (uint32_t k = 0; k < TC_BK / 16; ++k) {  // 16 bf16 = 32 B = +2 in the address
              if (PAIR) tc_mma_pair(dcol, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
              else tc_mma(dcol, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            }
          }
          if (PAIR) tc_commit_pair(empty0 + 8 * s);
          else tc_commit(empty0 + 8 * s);
        }
        if (PAIR) tc_commit_pair(tfull0 + 8 * acc);
        else tc_commit(tfull0 + 8 * acc);
      }
    }
  } else {
    // ---------------- epilogue: thread = query row = TMEM lane
    const uint32_t q4 = warp & 3;               // TMEM lane quarter this warp may access
    const uint32_t rl = q4 * 32 + lane;         // row within the tile
    const uint32_t row = row0 + rl;
    const bool live = row < P.nq;
    uint64_t* mypend = pend;
    const uint32_t c_lo = 0, c_hi = W / 32;
    if (TS) {
      // this row of A -> TMEM lane rl, columns [TC_A_COL, TC_A_COL + Kp/2)
      const uint32_t half = P.kblocks * (TC_BK / 2);
      const uint32_t* src = P.prow + (size_t)(live ? row : 0) * half;
      for (uint32_t c0 = 0; c0 < half; c0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = live ? __ldg(src + c0 + i) : 0u;
        tmem_st32(tmem + ((q4 * 32) << 16) + TC_A_COL + c0, v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(afull);
    }
    if (P.mode == 0) {
      for (uint32_t r = 0; r < 32; ++r) {          // lists start as dummies (coalesced)
        const uint32_t rr = row0 + q4 * 32 + r;
        if (rr < P.nq)
          for (uint32_t i = lane; i < P.KC; i += 32) P.lists[(size_t)rr * P.KC + i] = kDummyKey;
      }
    }
    __syncwarp();
    uint64_t tau = kDummyKey;
    float tau_f = __int_as_float(0x7f800000);
    if (P.mode == 1 && live)
      tau_f = key_dist(P.tau_keys[(size_t)row * P.tau_ld + P.tau_ld - 1]);
    uint32_t cnt = 0, gcnt = 0;
    // this row's own column in B coordinates (self exclusion), or none
    const uint32_t self_id = live && P.self_ids ? P.self_ids[row] : row + P.self_base;
    const uint32_t self_c = (P.exclude_self && self_id % P.col_stride == 0)
                                ? self_id / P.col_stride
                                : 0xffffffffu;
    // append mode: copy every lane's pending keys to its row's global buffer
    // (this lane owns the row: a register count, no atomics; a final count
    // above capg marks an overflowed row for the fallback)
    auto spill = [&]() {
      if (live && cnt) {
        uint64_t* b = P.bufs + (size_t)row * P.capg;
        for (uint32_t i = 0; i < cnt && gcnt + i < P.capg; ++i)
          b[gcnt + i] = mypend[i * TC_BM + rl];
        gcnt += cnt;
      }
      cnt = 0;
      __syncwarp();
    };
    // Merge the pending keys of every lane with cnt > min_cnt into its row's
    // sorted list, one row at a time, warp-wide: the pending keys are sorted
    // (64 keys, 2 per lane) and appended in descending order behind the list
    // (ascending, dummy padded to 192), and one bitonic merge of the 256 keys
    // leaves the KC smallest in front.
    auto flush = [&](uint32_t min_cnt) {
      __syncwarp();
      unsigned todo = __ballot_sync(0xffffffffu, cnt > min_cnt);
      while (todo) {
        const int r = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t rr = q4 * 32 + r;
        const uint32_t rcnt = __shfl_sync(0xffffffffu, cnt, r);
        uint64_t p[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t i = lane * 2 + e;
          p[e] = i < rcnt ? pend[i * TC_BM + rr] : kDummyKey;
        }
        warp_sort_regs<2>(p, lane);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (lane * 2 + e < TC_PEND) pend[(lane * 2 + e) * TC_BM + rr] = p[e];
        __syncwarp();
        uint64_t* lst = P.lists + (size_t)(row0 + rr) * P.KC;
        uint64_t v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t i = lane * 8 + e;
          v[e] = i < P.KC ? lst[i]
                          : (i < 256 - TC_PEND ? kDummyKey : pend[(255 - i) * TC_BM + rr]);
        }
        warp_merge_regs<8>(v, lane);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t i = lane * 8 + e;
          if (i < P.KC) lst[i] = v[e];
        }
        // new threshold: key KC-1 (lane (KC-1)/8, slot (KC-1)%8)
        const uint32_t last = P.KC - 1;
        uint64_t lastv = v[0];
#pragma unroll
        for (int e = 1; e < 8; ++e)
          if ((uint32_t)e == last % 8) lastv = v[e];
        lastv = __shfl_sync(0xffffffffu, lastv, last / 8);
        if (lane == r) {
          tau = lastv;
          tau_f = key_dist(tau);
          cnt = 0;
        }
      }
      __syncwarp();
    };
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t acc = t % ACC, aph = (t / ACC) & 1;
      mbar_wait(tfull0 + 8 * acc, aph);
      tc_fence_after();
#pragma unroll 1
      for (uint32_t c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32_nowait(tmem + ((q4 * 32) << 16) + acc * W + c * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == c_hi - 1) {
          // release the accumulator: one arrival per warp, at the leader for a pair
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR) mbar_arrive_remote(tempty0 + 8 * acc, 0);
            else mbar_arrive(tempty0 + 8 * acc);
          }
        }
        // fast path: the chunk's minimum against the threshold (FMNMX3 tree)
        float m3[11];
#pragma unroll
        for (int i = 0; i < 10; ++i) {
          float r3;
          asm("min.f32 %0, %1, %2, %3;"
              : "=f"(r3)
              : "f"(__uint_as_float(v[3 * i])), "f"(__uint_as_float(v[3 * i + 1])),
                "f"(__uint_as_float(v[3 * i + 2])));
          m3[i] = r3;
        }
        m3[10] = fminf(__uint_as_float(v[30]), __uint_as_float(v[31]));
        float mn;
        {
          float a0, a1, a2, a3;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(a0) : "f"(m3[0]), "f"(m3[1]), "f"(m3[2]));
          asm("min.f32 %0, %1, %2, %3;" : "=f"(a1) : "f"(m3[3]), "f"(m3[4]), "f"(m3[5]));
          asm("min.f32 %0, %1, %2, %3;" : "=f"(a2) : "f"(m3[6]), "f"(m3[7]), "f"(m3[8]));
          a3 = fminf(m3[9], m3[10]);
          float b0;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(b0) : "f"(a0), "f"(a1), "f"(a2));
          mn = fminf(b0, a3);
        }
        const bool hit = live && mn <= tau_f && gcnt <= P.capg;
        if (!__any_sync(0xffffffffu, hit)) continue;
        // slow path: only the FMNMX3 groups whose minimum passes are
        // examined element by element (appends are rare after the first tiles)
        const uint32_t cbase = tile_of(t) * W + c * 32;
        if (hit) {
          auto take = [&](int i) {
            const float d = __uint_as_float(v[i]);
            const uint32_t col = cbase + i;
            if (d <= tau_f && col < P.n && col != self_c) {
              mypend[cnt * TC_BM + rl] = make_key(fmaxf(d, 0.0f), col * P.col_stride);
              ++cnt;
            }
          };
#pragma unroll
          for (int g = 0; g < 10; ++g) {
            if (m3[g] <= tau_f) {
              take(3 * g);
              take(3 * g + 1);
              take(3 * g + 2);
            }
          }
          if (m3[10] <= tau_f) {
            take(30);
            take(31);
          }
        }
        if (__any_sync(0xffffffffu, cnt > P.pend_cap - 32)) {
          if (P.mode == 0) flush(TC_PEND / 4);
          else spill();
        }
      }
    }
    if (P.mode == 0) {
      flush(0);
    } else {
      spill();
      if (live) P.bcount[row] = gcnt;
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();  // the peer's TMEM is written by the leader's MMAs
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ----------------------------------------------------------------- prep ----
// x = b0 + b1 + r,  |x|^2 = n0 + n1 + n2 (bf16 parts)
//   query side P = [-2b0 | -2b0 | -2b1 | 1 1 1 | n0 n1 n2 | 0]
//   data side  R = [  b0 |   b1 |   b0 | n0 n1 n2 | 1 1 1 | 0]
// Column means of the dataset (the centring offset mu of the split), in two
// fixed-order stages so mu is deterministic: per (32-column group, row chunk)
// double partial sums, then a sequential sum over the chunks.
constexpr uint32_t kMeanChunks = 256;
__global__ void col_mean_partial_kernel(const float* __restrict__ data, uint32_t n, uint32_t ld,
                                        uint32_t dim, double* __restrict__ part) {
  const uint32_t col = blockIdx.x * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
  const uint32_t r0 = (uint32_t)((uint64_t)n * blockIdx.y / kMeanChunks);
  const uint32_t r1 = (uint32_t)((uint64_t)n * (blockIdx.y + 1) / kMeanChunks);
  double acc = 0.0;
  if (col < dim)
    for (uint32_t r = r0 + w; r < r1; r += blockDim.x / 32) acc += data[(size_t)r * ld + col];
  __shared__ double red[8][32];
  red[w][threadIdx.x & 31] = acc;
  __syncthreads();
  if (w == 0 && col < dim) {
    double t = 0.0;
    for (uint32_t k = 0; k < blockDim.x / 32; ++k) t += red[k][threadIdx.x];
    part[(size_t)blockIdx.y * dim + col] = t;
  }
}
__global__ void col_mean_final_kernel(const double* __restrict__ part, uint32_t n, uint32_t dim,
                                      float* __restrict__ mu) {
  const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= dim) return;
  double t = 0.0;
  for (uint32_t k = 0; k < kMeanChunks; ++k) t += part[(size_t)k * dim + col];
  mu[col] = (float)(t / n);
}

// mu: the dataset mean, subtracted from every row (data and queries) before
// the split.  Distances are translation-invariant; centring shrinks |x|, |q|
// and with them the error bound delta, which matters at high dimension.
__global__ void tc_split_kernel(const float* __restrict__ src, uint32_t rows, uint32_t ld,
                                uint32_t dim, uint32_t Kp, const float* __restrict__ mu,
                                __nv_bfloat16* __restrict__ P, __nv_bfloat16* __restrict__ R,
                                float* __restrict__ norms, uint32_t* __restrict__ maxnorm_bits) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = src + (size_t)row * ld;
  __nv_bfloat16* p = P ? P + (size_t)row * Kp : nullptr;
  __nv_bfloat16* r = R ? R + (size_t)row * Kp : nullptr;
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.0f), one = __float2bfloat16_rn(1.0f);
  float ss = 0.0f;
  for (uint32_t i = lane; i < dim; i += 32) {
    float v = x[i] - mu[i];
    ss = fmaf(v, v, ss);
    __nv_bfloat16 b0 = __float2bfloat16_rn(v);
    __nv_bfloat16 b1 = __float2bfloat16_rn(v - __bfloat162float(b0));
    if (p) {
      __nv_bfloat16 m0 = __float2bfloat16_rn(-2.0f * __bfloat162float(b0));  // exact
      __nv_bfloat16 m1 = __float2bfloat16_rn(-2.0f * __bfloat162float(b1));
      p[i] = m0;
      p[dim + i] = m0;
      p[2 * dim + i] = m1;
    }
    if (r) {
      r[i] = b0;
      r[dim + i] = b1;
      r[2 * dim + i] = b0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const __nv_bfloat16 n0 = __float2bfloat16_rn(ss);
  const float rem = ss - __bfloat162float(n0);
  const __nv_bfloat16 n1 = __float2bfloat16_rn(rem);
  const __nv_bfloat16 n2 = __float2bfloat16_rn(rem - __bfloat162float(n1));
  for (uint32_t i = 3 * dim + lane; i < Kp; i += 32) {
    const uint32_t j = i - 3 * dim;
    if (p) p[i] = j < 3 ? one : (j == 3 ? n0 : (j == 4 ? n1 : (j == 5 ? n2 : zero)));
    if (r) r[i] = j == 0 ? n0 : (j == 1 ? n1 : (j == 2 ? n2 : (j < 6 ? one : zero)));
  }
  if (lane == 0) {
    norms[row] = ss;
    if (maxnorm_bits) atomicMax(maxnorm_bits, __float_as_uint(ss));
  }
}

// --------------------------------------------------------------- rerank ----
// One warp per query row: band selection on d~, exact sequential-chain
// distances, (dist, id) sort, first k.  Rows whose band overflows the KC keys
// are queued for the exact SIMT kernel.
__global__ void tc_rerank_kernel(const uint64_t* __restrict__ lists, uint32_t nq, uint32_t KC,
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
    v[e] = i < KC ? lists[(size_t)row * KC + i] : kDummyKey;
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

// Append-mode rerank: one warp per row.  The buffer holds EVERY point with
// d~ <= tau* (tau* from the sample pass).  Valid iff K <= count <= capg and
// d~_(K) + 2 delta <= tau* (then every point that can be a true top-K member
// is in the buffer); otherwise the row is queued for the list-mode pass.
__global__ void tc_rerank_append_kernel(uint64_t* __restrict__ bufs,
                                        const uint32_t* __restrict__ bcount, uint32_t capg,
                                        const uint64_t* __restrict__ tau_keys, uint32_t tau_ld,
                                        uint32_t nq, uint32_t K, const float* __restrict__ qnorm,
                                        const uint32_t* __restrict__ maxnorm_bits, float eps_rel,
                                        float eps_norm, const float* __restrict__ data, uint32_t ld,
                                        const float* __restrict__ queries, uint32_t qld,
                                        uint32_t dim, uint32_t* __restrict__ out_ids,
                                        float* __restrict__ out_dists,
                                        uint32_t* __restrict__ fail_rows,
                                        uint32_t* __restrict__ fail_cnt,
                                        unsigned long long* __restrict__ reranked) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= nq) return;
  const uint32_t c = bcount[row];
  const float tau_star = key_dist(tau_keys[(size_t)row * tau_ld + tau_ld - 1]);
  uint64_t* b = bufs + (size_t)row * capg;
  bool ok = c >= K && c <= capg;
  float bound = 0.0f;
  if (ok) {
    constexpr int E = 32;  // up to 1024 keys
    uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = lane * E + e;
      v[e] = i < c ? b[i] : kDummyKey;
    }
    warp_sort_regs<E>(v, lane);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t i = lane * E + e;
      if (i < c) b[i] = v[e];
    }
    __syncwarp();
    const float qn = qnorm[row];
    const float xm = __uint_as_float(*maxnorm_bits);
    const float delta = eps_rel * sqrtf(qn) * sqrtf(xm) + eps_norm * (qn + xm);
    bound = key_dist(b[K - 1]) + 2.0f * delta;
    ok = bound <= tau_star;
  }
  if (!ok) {
    if (lane == 0) fail_rows[atomicAdd(fail_cnt, 1u)] = row;
    return;
  }
  // exact sequential-chain distances for the band, cyclic over lanes
  constexpr int E2 = 8;
  uint64_t w[E2];
  const float* q = queries + (size_t)row * qld;
  uint32_t nre = 0;
  bool over = false;
#pragma unroll
  for (int e = 0; e < E2; ++e) {
    const uint32_t i = e * 32 + lane;
    uint64_t key = i < c ? b[i] : kDummyKey;
    if (!key_is_dummy(key) && key_dist(key) <= bound) {
      const uint32_t id = key_id(key);
      const float* x = data + (size_t)id * ld;
      float acc = 0.0f;
      for (uint32_t d = 0; d < dim; ++d) acc = seq_step(acc, __ldg(x + d), __ldg(q + d));
      w[e] = make_key(acc, id);
      ++nre;
    } else {
      w[e] = kDummyKey;
    }
  }
  // the band must fit the 256 re-rank slots
  if (c > 32 * E2 && key_dist(b[32 * E2]) <= bound) over = true;
  if (__any_sync(0xffffffffu, over)) {
    if (lane == 0) fail_rows[atomicAdd(fail_cnt, 1u)] = row;
    return;
  }
  warp_sort_regs<E2>(w, lane);
#pragma unroll
  for (int e = 0; e < E2; ++e) {
    const uint32_t i = lane * E2 + e;
    if (i < K) {
      out_ids[(size_t)row * K + i] = key_id(w[e]);
      out_dists[(size_t)row * K + i] = key_dist(w[e]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nre += __shfl_xor_sync(0xffffffffu, nre, o);
  if (lane == 0 && reranked) atomicAdd(reranked, (unsigned long long)nre);
}

__global__ void gather_u16_rows_kernel(const uint16_t* __restrict__ src, uint32_t ld,
                                       const uint32_t* __restrict__ rows, uint32_t cnt,
                                       uint16_t* __restrict__ dst) {
  uint32_t r = blockIdx.x;
  if (r >= cnt) return;
  const uint16_t* s = src + (size_t)rows[r] * ld;
  for (uint32_t i = threadIdx.x; i < ld; i += blockDim.x) dst[(size_t)r * ld + i] = s[i];
}

__global__ void gather_f32_kernel(const float* __restrict__ src, const uint32_t* __restrict__ rows,
                                  uint32_t cnt, float* __restrict__ dst) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = src[rows[i]];
}

__global__ void offset_ids_kernel(const uint32_t* __restrict__ rows, uint32_t cnt, uint32_t base,
                                  uint32_t* __restrict__ dst) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = rows[i] + base;
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
// Scratch of one kNN call.  (A stream-ordered pool was measured slower for
// the first, cold build — the one a graph build pays — so plain cudaMalloc.)
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

// rows x Kp bf16, consecutive rows `row_step` rows apart in memory; boxes of
// 64 bf16 x box_rows rows
CUtensorMap make_map(const void* base, uint32_t rows, uint32_t Kp, uint32_t row_step,
                     uint32_t box_rows = TC_BN) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {Kp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2 * row_step};
  cuuint32_t box[2] = {TC_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed");
  return tm;
}

// the query tile is streamed (SA) when it cannot stay resident
bool tc_streamed(uint32_t kblocks) { return kblocks > TC_MAX_KB; }

size_t tc_smem_bytes(uint32_t kblocks, uint32_t stages, uint32_t pend_cap = TC_PEND,
                     bool pair = false) {
  const bool sa = tc_streamed(kblocks);
  const bool ts = CAGRA_KNN_TS && !pair && !sa;
  const size_t stage = sa ? 3 * TILE_BYTES : (pair ? TILE_BYTES / 2 : TILE_BYTES);
  return 1024 + (ts || sa ? 0 : (size_t)kblocks * TILE_BYTES) + stages * stage +
         sizeof(uint64_t) * (pend_cap * TC_BM + 2 * stages + 1 + 2 * (ts || sa ? 2 : 4)) + 16;
}

constexpr size_t kSmemLimit = 227 * 1024;

// deepest B ring that fits next to the resident query tile
uint32_t tc_stages(uint32_t kblocks, uint32_t pend_cap = TC_PEND, bool pair = false) {
  uint32_t s = pair ? 2 * TC_STAGES : TC_STAGES;  // pair stages hold half tiles
  while (s > 2 && tc_smem_bytes(kblocks, s, pend_cap, pair) > kSmemLimit) --s;
  return s;
}

}  // namespace

KnnTcStats g_knn_tc_stats;

bool knn_tc_eligible(uint32_t dim, uint32_t K) {
  const char* env = std::getenv("CAGRA_KNN_PATH");
  if (env && std::strcmp(env, "simt") == 0) return false;
  uint32_t Kp = round_up_u32(3 * dim + 6, TC_BK);
  const uint32_t kb = Kp / TC_BK;
  if (kb > TC_MAX_KB_STREAM || K + 32 + TC_PEND > 256) return false;
  if (tc_streamed(kb)) return tc_smem_bytes(kb, 3) <= kSmemLimit;  // >= 3-deep A+B+B ring
  return tc_smem_bytes(kb, tc_stages(kb, TC_PEND, true), TC_PEND, true) <= kSmemLimit;
}

namespace {

// Everything one kNN / top-k call shares between its passes.
struct TcCall {
  const float* data;
  uint32_t n, ld, dim, K, Kp, kblocks, stages;
  bool exclude_self;
  uint32_t self_base;  // kNN rows [self_base, self_base + nq) of the graph (row-sharded builds)
  float eps_rel, eps_norm;
  const uint32_t* maxnorm;
  const void* R;  // n x Kp bf16
  cudaStream_t stream;
};

// CTA pairs (cluster of 2, cta_group::2 MMA) with CAGRA_TC_PAIR=1.
bool tc_pair_enabled() {
  const char* e = std::getenv("CAGRA_TC_PAIR");  // measured slower than single CTAs: opt-in
  return e && e[0] == '1';
}

void run_tc_kernel(const TcCall& c, const void* Pq, const CUtensorMap& tmA,
                   const CUtensorMap& tmB, TcArgs a, uint32_t nq) {
  const bool sa = tc_streamed(c.kblocks);
  const bool pair = tc_pair_enabled() && !sa;
  a.kblocks = c.kblocks;
  a.prow = reinterpret_cast<const uint32_t*>(Pq);
  const char* ge = std::getenv("CAGRA_TC_GROUPS");
  a.groups = ge ? (uint32_t)std::atoi(ge) : 1u;  // measured: the lockstep sweep wins (L2 reuse)
  a.pend_cap = a.mode == 1 ? TC_PEND_APPEND : TC_PEND;
  a.stages = tc_stages(c.kblocks, a.pend_cap, pair);
  a.exclude_self = c.exclude_self ? 1 : 0;
  a.nq = nq;
  const size_t smem = tc_smem_bytes(c.kblocks, a.stages, a.pend_cap, pair);
  if (sa) {
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    knn_tc_kernel<false, true>
        <<<(nq + TC_BM - 1) / TC_BM, TC_THREADS, smem, c.stream>>>(tmA, tmB, a);
    CAGRA_LAUNCH_CHECK();
    return;
  }
  if (!pair) {
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    knn_tc_kernel<false><<<(nq + TC_BM - 1) / TC_BM, TC_THREADS, smem, c.stream>>>(tmA, tmB, a);
    CAGRA_LAUNCH_CHECK();
    return;
  }
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * ((nq + 2 * TC_BM - 1) / (2 * TC_BM)));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CAGRA_CUDA_TRY(cudaLaunchKernelEx(&cfg, knn_tc_kernel<true>, tmA, tmB, a));
}

// Rows [0, nq) of the query side P (bf16, Kp wide; norms qnorm; fp32 rows
// queries for the exact re-rank; self_ids for kNN rows) -> ids/dists [nq][K].
// Single pass: running list of the K+32 smallest d~ per row.  Rows whose band
// overflows go to the SIMT sequential-chain kernel.
void list_pass(const TcCall& c, const void* P, uint32_t nq, const float* qnorm,
               const float* queries, uint32_t qld, const uint32_t* self_ids, uint32_t* ids,
               float* dists, uint64_t& reranked, uint64_t& fallback) {
  const uint32_t KC = c.K + 32;
  Dev lists(8ull * nq * KC), fails(4ull * nq + 4), rer(8);
  CAGRA_CUDA_TRY(cudaMemsetAsync(fails.p, 0, 4ull * nq + 4, c.stream));
  CAGRA_CUDA_TRY(cudaMemsetAsync(rer.p, 0, 8, c.stream));
  const uint32_t brows = tc_pair_enabled() && !tc_streamed(c.kblocks) ? TC_BN / 2 : TC_BN;
  CUtensorMap tmA = make_map(P, nq, c.Kp, 1), tmB = make_map(c.R, c.n, c.Kp, 1, brows);
  TcArgs a{};
  a.n = c.n;
  a.KC = KC;
  a.mode = 0;
  a.col_stride = 1;
  a.lists = lists.as<uint64_t>();
  a.self_ids = self_ids;
  a.self_base = self_ids ? 0 : c.self_base;
  run_tc_kernel(c, P, tmA, tmB, a, nq);
  uint32_t* fail_cnt = fails.as<uint32_t>();
  uint32_t* fail_rows = fail_cnt + 1;
  tc_rerank_kernel<<<(nq + 7) / 8, 256, 0, c.stream>>>(
      lists.as<uint64_t>(), nq, KC, c.K, qnorm, c.maxnorm, c.eps_rel, c.eps_norm, c.data, c.ld,
      queries, qld, c.dim, ids, dists, fail_rows, fail_cnt, rer.as<unsigned long long>());
  CAGRA_LAUNCH_CHECK();
  uint32_t nf = 0;
  unsigned long long nre = 0;
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&nf, fail_cnt, 4, cudaMemcpyDeviceToHost, c.stream));
  CAGRA_CUDA_TRY(cudaMemcpyAsync(&nre, rer.p, 8, cudaMemcpyDeviceToHost, c.stream));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(c.stream));
  reranked += nre;
  fallback += nf;
  if (!nf) return;
  // exact SIMT kernel for the rows whose candidate band overflowed
  Dev q((size_t)nf * qld * 4), sid(4ull * nf), sc(8ull * nf * c.K), fi(4ull * nf * c.K),
      fd(4ull * nf * c.K);
  gather_rows_kernel<<<nf, 128, 0, c.stream>>>(queries, qld, fail_rows, nf, q.as<float>());
  CAGRA_LAUNCH_CHECK();
  const uint32_t* simt_self = nullptr;
  if (c.exclude_self) {
    if (self_ids) {
      gather_f32_kernel<<<(nf + 255) / 256, 256, 0, c.stream>>>(
          reinterpret_cast<const float*>(self_ids), fail_rows, nf, sid.as<float>());
      CAGRA_LAUNCH_CHECK();
      simt_self = sid.as<uint32_t>();
    } else if (c.self_base) {
      offset_ids_kernel<<<(nf + 255) / 256, 256, 0, c.stream>>>(fail_rows, nf, c.self_base,
                                                                 sid.as<uint32_t>());
      CAGRA_LAUNCH_CHECK();
      simt_self = sid.as<uint32_t>();
    } else {
      simt_self = fail_rows;
    }
  }
  launch_exact_topk_simt(c.data, c.n, c.ld, q.as<float>(), nf, qld, c.dim, c.K, c.exclude_self,
                         simt_self, sc.as<uint64_t>(), fi.as<uint32_t>(), fd.as<float>(),
                         c.stream);
  scatter_rows_kernel<<<nf, 128, 0, c.stream>>>(fail_rows, nf, c.K, fi.as<uint32_t>(),
                                                fd.as<float>(), ids, dists);
  CAGRA_LAUNCH_CHECK();
  CAGRA_CUDA_TRY(cudaStreamSynchronize(c.stream));
}

constexpr uint32_t kSampleStride = 16;

}  // namespace

void launch_knn_tc(const float* d_data, uint32_t n, uint32_t ld, const float* d_queries,
                   uint32_t nq, uint32_t qld, uint32_t dim, uint32_t K, bool exclude_self,
                   uint32_t self_base, uint32_t* d_ids, float* d_dists, cudaStream_t stream) {
  if (nq == 0) return;
  TcCall c;
  c.self_base = exclude_self ? self_base : 0;
  c.data = d_data;
  c.n = n;
  c.ld = ld;
  c.dim = dim;
  c.K = K;
  c.Kp = round_up_u32(3 * dim + 6, TC_BK);
  c.kblocks = c.Kp / TC_BK;
  c.stages = tc_stages(c.kblocks);
  c.exclude_self = exclude_self;
  c.stream = stream;
  // error bound of d~ (file header): |d~ - d| <= eps_rel |q| max|x| +
  // eps_norm (|q|^2 + max|x|^2), norms of the centred rows x' = fl(x - mu):
  // the split's omitted terms (3.1*2^-16 of sum|q_i||x_i| <= |q||x|, doubled
  // by the -2), fp32 accumulation over Kp terms of total magnitude
  // 2|q||x| + |q|^2 + |x|^2, the fp32 norms, and the centring rounding
  // (|d - |x'-q'|^2| <= 2u (|x'| + |q'|)^2, u = 2^-24; counted with 2^-23).
  const float u23 = 1.1920929e-07f;
  c.eps_rel = 2.0f * 3.1f * 1.52587890625e-05f + 2.0f * (float)c.Kp * u23 + 4.0f * u23;
  c.eps_norm = (float)c.Kp * u23 + (float)(dim + 8) * u23 + 2.0f * u23;

  // kNN graph: the queries are data rows [self_base, self_base + nq), so the
  // data split also yields their query-side rows
  const bool same = exclude_self;
  Dev dP((size_t)(same ? n : nq) * c.Kp * 2), dR((size_t)n * c.Kp * 2), dqn(4ull * nq), dxn(4ull * n), dmax(4);
  CAGRA_CUDA_TRY(cudaMemsetAsync(dmax.p, 0, 4, stream));
  Dev dmu(4ull * dim), dpart(8ull * kMeanChunks * dim);
  col_mean_partial_kernel<<<dim3((dim + 31) / 32, kMeanChunks), 256, 0, stream>>>(
      d_data, n, ld, dim, dpart.as<double>());
  col_mean_final_kernel<<<(dim + 127) / 128, 128, 0, stream>>>(dpart.as<double>(), n, dim,
                                                               dmu.as<float>());
  CAGRA_LAUNCH_CHECK();
  // data side: R (and P when the queries are the data), norms, max norm
  tc_split_kernel<<<(n + 7) / 8, 256, 0, stream>>>(d_data, n, ld, dim, c.Kp, dmu.as<float>(),
                                                   same ? dP.as<__nv_bfloat16>() : nullptr,
                                                   dR.as<__nv_bfloat16>(), dxn.as<float>(),
                                                   dmax.as<uint32_t>());
  CAGRA_LAUNCH_CHECK();
  const float* qnorm = dxn.as<float>() + c.self_base;
  const void* Pq = dP.as<uint16_t>() + (size_t)c.self_base * c.Kp;
  if (!same) {
    tc_split_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(d_queries, nq, qld, dim, c.Kp,
                                                      dmu.as<float>(), dP.as<__nv_bfloat16>(),
                                                      nullptr,
                                                      dqn.as<float>(), nullptr);
    CAGRA_LAUNCH_CHECK();
    qnorm = dqn.as<float>();
  }
  c.maxnorm = dmax.as<uint32_t>();
  c.R = dR.p;
  uint64_t reranked = 0, fallback = 0, retried = 0;

  const char* onepass = std::getenv("CAGRA_TC_ONEPASS");
  const bool two_pass = n / kSampleStride >= 4096 && !(onepass && onepass[0] == '1');
  if (!two_pass) {
    list_pass(c, Pq, nq, qnorm, d_queries, qld, nullptr, d_ids, d_dists, reranked, fallback);
  } else {
    // pass 1: every 16th point; the r-th smallest d~ over the sample is an
    // upper bound of the r-th smallest over all points (valid for ANY r).
    const uint32_t ns = n / kSampleStride;
    const uint32_t r = std::max<uint32_t>(8, (3 * (K + 16) + kSampleStride - 1) / kSampleStride);
    const uint32_t capg = (uint64_t)nq * 1024 * 8 <= (8ull << 30) ? 1024 : 512;
    Dev lists1(8ull * r * nq), bufs(8ull * nq * capg), bcount(4ull * nq), fails(4ull * nq + 4),
        rer(8);
    CAGRA_CUDA_TRY(cudaMemsetAsync(fails.p, 0, 4ull * nq + 4, stream));
    CAGRA_CUDA_TRY(cudaMemsetAsync(rer.p, 0, 8, stream));
    CAGRA_CUDA_TRY(cudaMemsetAsync(bcount.p, 0, 4ull * nq, stream));  // append counters
    const uint32_t brows = tc_pair_enabled() && !tc_streamed(c.kblocks) ? TC_BN / 2 : TC_BN;
    CUtensorMap tmA = make_map(Pq, nq, c.Kp, 1);
    CUtensorMap tmS = make_map(dR.p, ns, c.Kp, kSampleStride, brows);
    CUtensorMap tmB = make_map(dR.p, n, c.Kp, 1, brows);
    TcArgs a{};
    a.n = ns;
    a.KC = r;
    a.mode = 0;
    a.col_stride = kSampleStride;
    a.lists = lists1.as<uint64_t>();
    run_tc_kernel(c, Pq, tmA, tmS, a, nq);
    // pass 2: every point with d~ <= tau* appended (no merging)
    TcArgs b{};
    b.n = n;
    b.KC = r;
    b.mode = 1;
    b.col_stride = 1;
    b.tau_keys = lists1.as<uint64_t>();
    b.tau_ld = r;
    b.bufs = bufs.as<uint64_t>();
    b.bcount = bcount.as<uint32_t>();
    b.capg = capg;
    run_tc_kernel(c, Pq, tmA, tmB, b, nq);
    uint32_t* fail_cnt = fails.as<uint32_t>();
    uint32_t* fail_rows = fail_cnt + 1;
    tc_rerank_append_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(
        bufs.as<uint64_t>(), bcount.as<uint32_t>(), capg, lists1.as<uint64_t>(), r, nq, K, qnorm,
        c.maxnorm, c.eps_rel, c.eps_norm, d_data, ld, d_queries, qld, dim, d_ids, d_dists,
        fail_rows, fail_cnt, rer.as<unsigned long long>());
    CAGRA_LAUNCH_CHECK();
    uint32_t nf = 0;
    unsigned long long nre = 0;
    CAGRA_CUDA_TRY(cudaMemcpyAsync(&nf, fail_cnt, 4, cudaMemcpyDeviceToHost, stream));
    CAGRA_CUDA_TRY(cudaMemcpyAsync(&nre, rer.p, 8, cudaMemcpyDeviceToHost, stream));
    CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    reranked += nre;
    retried = nf;
    if (nf) {
      // the rows whose threshold did not bracket their band: single-pass list
      // mode on just those rows
      Dev P2((size_t)nf * c.Kp * 2), qn2(4ull * nf), q2((size_t)nf * qld * 4), ids2(4ull * nf * K),
          d2(4ull * nf * K);
      gather_u16_rows_kernel<<<nf, 128, 0, stream>>>(static_cast<const uint16_t*>(Pq), c.Kp,
                                                     fail_rows, nf,
                                                     P2.as<uint16_t>());
      gather_f32_kernel<<<(nf + 255) / 256, 256, 0, stream>>>(qnorm, fail_rows, nf,
                                                              qn2.as<float>());
      gather_rows_kernel<<<nf, 128, 0, stream>>>(d_queries, qld, fail_rows, nf, q2.as<float>());
      CAGRA_LAUNCH_CHECK();
      // the retried rows' data ids (their self columns)
      Dev sid2(4ull * nf);
      const uint32_t* self2 = nullptr;
      if (exclude_self) {
        offset_ids_kernel<<<(nf + 255) / 256, 256, 0, stream>>>(fail_rows, nf, c.self_base,
                                                                sid2.as<uint32_t>());
        CAGRA_LAUNCH_CHECK();
        self2 = sid2.as<uint32_t>();
      }
      list_pass(c, P2.p, nf, qn2.as<float>(), q2.as<float>(), qld, self2, ids2.as<uint32_t>(),
                d2.as<float>(), reranked, fallback);
      scatter_rows_kernel<<<nf, 128, 0, stream>>>(fail_rows, nf, K, ids2.as<uint32_t>(),
                                                  d2.as<float>(), d_ids, d_dists);
      CAGRA_LAUNCH_CHECK();
      CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    }
  }
  g_knn_tc_stats.rows = nq;
  g_knn_tc_stats.fallback_rows = fallback;
  g_knn_tc_stats.reranked = reranked;
  g_knn_tc_stats.retried_rows = retried;
}

}  // namespace cagra
