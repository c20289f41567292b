// K1 on the 5th-gen tensor cores: exact k-nearest-neighbour selection for the
// kNN graph (exact_knn_graph, knn_build.cpp:40-63) and ground truth
// (exact_topk, topk.cpp:10-43), bit-identical to the reference.
//
// 1. prep      : rows are centred on the dataset mean (x' = fl(x - mu)) and
//                turned into 16-bit GEMM operands whose product is a filter
//                distance d~ with a rigorous error bound:
//                * fp16 single term (default): s = 2^e with s|x'| < 2^13,
//                    P_q = [-2 h(s q') | sig sig | 0..]   (query)
//                    R_x = [ h(s x')   | n0  n1  | 0..]   (data, n0+n1 =
//                                                 s^2|x'|^2/sig, sig = 2^14)
//                  (K = dim + 2), the epilogue adds the row constant
//                  s^2 |q'|^2: d~ = s^2 d (1 +- ~2^-10 on the cross term);
//                * bf16x3 (CAGRA_KNN_SPLIT=3): x = b0 + b1 + r (|r| <=
//                  2^-16 |x|), norms folded in, K = 3 dim + 6:
//                    P_q = [-2b0 | -2b0 | -2b1 | 1 1 1 | n0 n1 n2 | 0..]
//                    R_x = [  c0 |   c1 |   c0 | m0 m1 m2 | 1 1 1 | 0..]
//                K is padded to 64 (one SWIZZLE_128B k-block) in memory; the
//                MMA skips the all-zero 16-wide steps of the last block.
// 2. knn_tc    : one CTA per 128 query rows.  The query tile (A) stays in smem
//                for the whole sweep; 128-point data tiles (B) stream through
//                a TMA ring (SWIZZLE_128B, K-major); one elected thread issues
//                tcgen05.mma kind::f16 (fp16/bf16 -> fp32) into a
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
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <mutex>
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
constexpr int TC_PEND_APPEND = 48;  // append mode: a spill is issued when any lane holds > 16 keys
constexpr int TC_THREADS = 192;  // w0 TMA, w1 MMA, w2..w5 epilogue (w2..w9 with two halves)
constexpr int TC_EPI_WARPS = 4;  // per 128-row half
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
constexpr uint32_t BOX_ROWS = 64;                   // B tensor-map box: 64 points x 64 K
constexpr uint32_t BOX_BYTES = BOX_ROWS * TC_BK * 2;  // 8 KB
// Option: two-half CTAs stream 64-point data tiles into 4 accumulators per half
// (TMEM 2 x 4 x 64 columns): the MMA can run up to 3 tiles ahead of the
// epilogue instead of 1 (the epilogue's per-tile latency varies with its
// appends). Measured slower on 1M x 96 k=128 (0.60 s vs 0.404 s: twice the
// per-tile barrier and release work), so 128-point tiles stay the default.
// 1: mode-2 lists kept unsorted with a tracked maximum (see drain)
#ifndef CAGRA_TC_MAXLIST
#define CAGRA_TC_MAXLIST 1
#endif
#ifndef CAGRA_TC_W64
#define CAGRA_TC_W64 0
#endif

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
// 1: append-mode keys are staged in shared memory and copied out in spills;
// 0: every lane stores its row's keys straight to the row's buffer (measured
// 20% slower on the whole build: scattered 8-byte stores from every append)
#ifndef CAGRA_TC_STAGED_APPEND
#define CAGRA_TC_STAGED_APPEND 1
#endif
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
// Instruction descriptor (built in the kernel): fp32 accumulate, both
// operands K-major, M=128 (256 for a pair), N = the tile width; the A/B format
// bits (7-9, 10-12: 0 = f16, 1 = bf16) are OR-ed in at run time.

struct TcArgs {
  uint32_t nq, n, kblocks, KC, exclude_self, stages, pend_cap;
  uint32_t mode;        // 0: running sorted list of KC keys (warp merges, lists in L2);
                        // 1: append d~ <= fixed tau;
                        // 2: running sorted list of KC <= pend_cap keys, per-lane
                        //    insertion into the row's list in shared memory
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
  uint32_t ab_fmt;           // operand format bits of the instruction descriptor (f16 0, bf16 1)
  uint32_t ksteps_last;      // 16-wide MMA steps in the last k-block (the rest is zero padding)
  const float* qnorm;        // FP16 split: per-row |q'|^2 (original units), added in the epilogue
  float dscale;              // FP16 split: s^2, d~ is kept in GEMM units (s^2 * distance)
};

// Minimum of 32 accumulator values (FMNMX3 tree); m3 keeps the 11 group minima.
__device__ __forceinline__ float chunk_min(const uint32_t (&v)[32], float (&m3)[11]) {
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
  float a0, a1, a2, b0;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(a0) : "f"(m3[0]), "f"(m3[1]), "f"(m3[2]));
  asm("min.f32 %0, %1, %2, %3;" : "=f"(a1) : "f"(m3[3]), "f"(m3[4]), "f"(m3[5]));
  asm("min.f32 %0, %1, %2, %3;" : "=f"(a2) : "f"(m3[6]), "f"(m3[7]), "f"(m3[8]));
  const float a3 = fminf(m3[9], m3[10]);
  asm("min.f32 %0, %1, %2, %3;" : "=f"(b0) : "f"(a0), "f"(a1), "f"(a2));
  return fminf(b0, a3);
}

// PAIR: a cluster of 2 CTAs shares each data tile: every CTA keeps its own
// 128 query rows (A, smem) and loads HALF of the 128-point B tile; the leader
// issues tcgen05.mma.cta_group::2 (M = 256) and each CTA's TMEM receives its
// rows x all 128 points.  Per-SM B traffic from L2 halves.
// SA (K > 512, e.g. 960-d): the query tile does not fit next to the ring, so
// every stage carries the A k-block together with the B k-block (a plain
// streamed GEMM main loop; A is re-read from L2 once per data tile).
// HV = 2 (small K): the CTA owns 256 query rows as two 128-row halves (A in
// smem); every B stage feeds two M=128 MMAs, one per half, into the half's
// own TMEM accumulators, and 8 epilogue warps (two per TMEM lane quarter)
// scan them — twice the epilogue issue slots per SM and half the L2->SM B
// traffic per query row of HV = 1.
template <bool PAIR, bool SA = false, int HV = 1, int MODE = -1>
__global__ void __launch_bounds__(64 + 128 * HV, 1)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcArgs P) {
  // MODE >= 0: the epilogue mode fixed at compile time (no dead mode code)
  const uint32_t kmode = MODE >= 0 ? (uint32_t)MODE : P.mode;
  static_assert(!(PAIR && SA), "streamed A is single-CTA");
  static_assert(HV == 1 || (!PAIR && !SA), "two halves: single CTA, resident A");
  constexpr bool TS = CAGRA_KNN_TS && !PAIR && !SA && HV == 1;
  constexpr uint32_t ROWS = TC_BM * HV;  // query rows per CTA
  // SA data tiles are 256 points wide (one N=256 MMA per k-block), so every
  // streamed A k-block is used against two 128-point B tiles
  constexpr uint32_t W = SA ? 2 * TC_BN : (HV == 2 && CAGRA_TC_W64 ? 64u : (uint32_t)TC_BN);
  constexpr int ACC = TS || SA ? 2 : (HV == 2 ? (W == 64 ? 4 : 2) : 4);  // per half (512 cols)
  constexpr uint32_t BTILE = PAIR ? TILE_BYTES / 2 : W * TC_BK * 2;  // B bytes per stage per CTA
  constexpr uint32_t STAGE = SA ? 3 * TILE_BYTES : BTILE;            // [A k-block |] B k-block(s)
  constexpr uint32_t idesc_shape =
      PAIR ? ((1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24))
           : ((1u << 4) | ((uint32_t)(W >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24));
  const uint32_t idesc = idesc_shape | (P.ab_fmt << 7) | (P.ab_fmt << 10);
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B tiles
  unsigned char* base = tc_smem_raw + ((1024 - (smem_u32(tc_smem_raw) & 1023)) & 1023);
  unsigned char* sA = base;                                   // SS: HV x kblocks x 16 KB
  unsigned char* sB = sA + (TS || SA ? 0 : (size_t)HV * P.kblocks * TILE_BYTES);  // stages x STAGE
  uint64_t* pend = reinterpret_cast<uint64_t*>(sB + P.stages * STAGE);  // PEND x ROWS
  uint64_t* bars = pend + P.pend_cap * ROWS;
  // bars: full[S] empty[S] afull tfull[ACC] tempty[ACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P.stages + 1 + 2 * ACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const uint32_t row0 = PAIR ? (blockIdx.x >> 1) * 2 * TC_BM + rank * TC_BM : blockIdx.x * ROWS;
  // column split (list modes): blockIdx.y sweeps its share of the data tiles
  // into its own list slab, merged per row afterwards (small query batches
  // spread over the SMs instead of one CTA sweeping everything)
  const uint32_t ntiles_all = (P.n + W - 1) / W;
  const uint32_t tile_b = (uint32_t)((uint64_t)ntiles_all * blockIdx.y / gridDim.y);
  const uint32_t ntiles = (uint32_t)((uint64_t)ntiles_all * (blockIdx.y + 1) / gridDim.y) - tile_b;
  uint64_t* const lists = P.lists ? P.lists + (size_t)blockIdx.y * P.nq * P.KC : nullptr;
  const uint32_t S = P.stages;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
  const uint32_t afull = smem_u32(bars + 2 * S);
  const uint32_t tfull0 = afull + 8, tempty0 = afull + 8 + 8 * ACC;
  auto tile_of = [&](uint32_t t) { return tile_b + t; };

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
      mbar_init(tempty0 + 8 * a, (PAIR ? 2 : 1) * TC_EPI_WARPS * HV);  // one arrival per epilogue warp
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
        mbar_expect_tx(afull, HV * P.kblocks * TILE_BYTES);
        for (uint32_t h = 0; h < (uint32_t)HV; ++h)
          for (uint32_t kb = 0; kb < P.kblocks; ++kb)
            tma_load_2d(smem_u32(sA + (h * P.kblocks + kb) * TILE_BYTES), &tmA, afull, kb * TC_BK,
                        row0 + h * TC_BM);
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
#pragma unroll
            for (uint32_t b = 0; b < W / BOX_ROWS; ++b)  // 64-point boxes back to back
              tma_load_2d(smem_u32(sB + s * STAGE + TILE_BYTES + b * BOX_BYTES), &tmB,
                          full0 + 8 * s, kb * TC_BK, tile_of(t) * W + b * BOX_ROWS);
          } else {
            mbar_expect_tx(full0 + 8 * s, BTILE);
#pragma unroll
            for (uint32_t b = 0; b < W / BOX_ROWS; ++b)  // 64-point boxes back to back
              tma_load_2d(smem_u32(sB + s * BTILE + b * BOX_BYTES), &tmB, full0 + 8 * s,
                          kb * TC_BK, tile_of(t) * W + b * BOX_ROWS);
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
          // the last k-block may be partly zero padding: its all-zero steps are skipped
          const uint32_t nk = kb + 1 == P.kblocks ? P.ksteps_last : TC_BK / 16;
          if (TS) {
#pragma unroll
            for (uint32_t k = 0; k < TC_BK / 16; ++k)  // A: 16 x 16-bit = 8 TMEM columns per step
              if (k < nk)
                tc_mma_ts(dcol, tmem + TC_A_COL + kb * (TC_BK / 2) + k * 8, bd + 2 * k, idesc,
                          (kb | k) != 0);
          } else {
#pragma unroll
            for (uint32_t h = 0; h < (uint32_t)HV; ++h) {
              const uint64_t ad = sw128_desc(
                  smem_u32(SA ? sB + s * STAGE : sA + (h * P.kblocks + kb) * TILE_BYTES));
              const uint32_t dh = dcol + h * ACC * W;  // this half's accumulator
#pragma unroll
              for (uint32_t k = 0; k < TC_BK / 16; ++k) {  // 16 x 16-bit = 32 B = +2 in the address
                if (k >= nk) break;
                if (PAIR) tc_mma_pair(dh, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                else tc_mma(dh, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
              }
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
    const uint32_t hv = HV == 2 ? (uint32_t)(warp - 2) / 4 : 0u;  // the warp's half
    const uint32_t rl = hv * TC_BM + q4 * 32 + lane;  // row within the CTA
    const uint32_t row = row0 + rl;
    const bool live = row < P.nq;
    uint64_t* mypend = pend;
    const uint32_t c_hi = W / 32;
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
    if (kmode == 0) {
      for (uint32_t r = 0; r < 32; ++r) {          // lists start as dummies (coalesced)
        const uint32_t rr = row0 + hv * TC_BM + q4 * 32 + r;
        if (rr < P.nq)
          for (uint32_t i = lane; i < P.KC; i += 32) lists[(size_t)rr * P.KC + i] = kDummyKey;
      }
    }
    if (kmode == 2)  // the row's list starts as dummies
      for (uint32_t i = 0; i < P.KC; ++i) mypend[i * ROWS + rl] = kDummyKey;
    __syncwarp();
    uint64_t tau = kDummyKey;
    float tau_f = __int_as_float(0x7f800000);
    if (kmode == 1 && live)
      tau_f = key_dist(P.tau_keys[(size_t)row * P.tau_ld + P.tau_ld - 1]);
    // FP16 split: the GEMM yields e = s^2 (|x'|^2 - 2 q'.x'); the row constant
    // qoff = s^2 |q'|^2 completes d~ = e + qoff.  The chunk test compares e
    // against tau_e = tau - qoff, widened by a few ulps so it stays a
    // superset of the exact per-key test d~ <= tau done on the slow path.
    const float qoff = P.qnorm && live ? P.qnorm[row] * P.dscale : 0.0f;
    auto tau_e_of = [&](float t) {
      return P.qnorm ? (t - qoff) + (fabsf(t) + qoff) * 4.76837158e-7f : t;
    };
    float tau_e = tau_e_of(tau_f);
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
          b[gcnt + i] = mypend[i * ROWS + rl];
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
        const uint32_t rr = hv * TC_BM + q4 * 32 + r;
        const uint32_t rcnt = __shfl_sync(0xffffffffu, cnt, r);
        uint64_t p[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const uint32_t i = lane * 2 + e;
          p[e] = i < rcnt ? pend[i * ROWS + rr] : kDummyKey;
        }
        warp_sort_regs<2>(p, lane);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (lane * 2 + e < TC_PEND) pend[(lane * 2 + e) * ROWS + rr] = p[e];
        __syncwarp();
        uint64_t* lst = lists + (size_t)(row0 + rr) * P.KC;
        uint64_t v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t i = lane * 8 + e;
          v[e] = i < P.KC ? lst[i]
                          : (i < 256 - TC_PEND ? kDummyKey : pend[(255 - i) * ROWS + rr]);
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
          tau_e = tau_e_of(tau_f);
          cnt = 0;
        }
      }
      __syncwarp();
    };
    // mode 2: the row's sorted list occupies pending slots [0, KC); new keys
    // are appended behind it and drained into it by per-lane insertion
    // (thread = row, no warp cooperation; the threshold is the list's last key)
    const uint32_t pbase = kmode == 2 ? P.KC : 0u;
#if CAGRA_TC_MAXLIST
    // mode 2 as an UNSORTED list of KC keys whose maximum (the threshold) sits
    // at slot tmax: a key below it replaces it, then the maximum is found
    // again with KC independent shared loads (no dependent shift chain).  The
    // consumers read only the maximum (at KC - 1, placed after the pass) or
    // sort the list themselves.
    uint32_t tmax = 0;
    auto drain = [&]() {
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint64_t key = mypend[(pbase + i) * ROWS + rl];
        if (key >= tau) continue;
        mypend[tmax * ROWS + rl] = key;
        uint64_t m = 0;
        uint32_t mi = 0;
#pragma unroll 8
        for (uint32_t j = 0; j < P.KC; ++j) {
          const uint64_t v = mypend[j * ROWS + rl];
          if (v > m) {
            m = v;
            mi = j;
          }
        }
        tau = m;
        tmax = mi;
      }
      cnt = 0;
      tau_f = key_dist(tau);
      tau_e = tau_e_of(tau_f);
    };
#else
    auto drain = [&]() {
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint64_t key = mypend[(pbase + i) * ROWS + rl];
        if (key >= tau) continue;
        uint32_t j = P.KC - 1;
        for (; j > 0; --j) {
          const uint64_t prev = mypend[(j - 1) * ROWS + rl];
          if (prev <= key) break;
          mypend[j * ROWS + rl] = prev;
        }
        mypend[j * ROWS + rl] = key;
        tau = mypend[(P.KC - 1) * ROWS + rl];
      }
      cnt = 0;
      tau_f = key_dist(tau);
      tau_e = tau_e_of(tau_f);
    };
#endif
#if !CAGRA_TC_STAGED_APPEND
    // append mode: each lane owns its row's global buffer (no staging)
    uint64_t* const row_buf = kmode == 1 && live ? P.bufs + (size_t)row * P.capg : nullptr;
#endif
    // slow path of one 32-column chunk: only the FMNMX3 groups whose minimum
    // passes are examined element by element (appends are rare after the
    // first tiles); warp-uniform entry (the pending-buffer check is a vote)
    auto scan = [&](const uint32_t(&v)[32], const float(&m3)[11], uint32_t cbase, bool hit) {
      if (hit) {
        auto take = [&](int i) {
          const float d = __uint_as_float(v[i]) + qoff;
          const uint32_t col = cbase + i;
          if (d <= tau_f && col < P.n && col != self_c) {
            const uint64_t key = make_key(fmaxf(d, 0.0f), col * P.col_stride);
#if !CAGRA_TC_STAGED_APPEND
            if (kmode == 1) {  // straight into the row's global buffer
              if (gcnt < P.capg) row_buf[gcnt] = key;
              ++gcnt;
              return;
            }
#endif
            mypend[(pbase + cnt) * ROWS + rl] = key;
            ++cnt;
          }
        };
#pragma unroll
        for (int g = 0; g < 10; ++g) {
          if (m3[g] <= tau_e) {
            take(3 * g);
            take(3 * g + 1);
            take(3 * g + 2);
          }
        }
        if (m3[10] <= tau_e) {
          take(30);
          take(31);
        }
      }
      if (kmode == 2) {
        if (cnt) drain();
      } else if ((!(CAGRA_TC_STAGED_APPEND == 0) || kmode == 0) &&
                 __any_sync(0xffffffffu, cnt > P.pend_cap - 32)) {
        if (kmode == 0) flush(TC_PEND / 4);
        else spill();
      }
    };
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t acc = t % ACC, aph = (t / ACC) & 1;
      mbar_wait(tfull0 + 8 * acc, aph);
      tc_fence_after();
      const uint32_t tbase = tmem + ((q4 * 32) << 16) + (hv * ACC + acc) * W;
      // two 32-column chunks per step: both TMEM loads in flight behind one
      // wait, two independent FMNMX3 trees, one vote
#pragma unroll 1
      for (uint32_t c = 0; c < c_hi; c += 2) {
        uint32_t va[32], vb[32];
        tmem_ld32_nowait(tbase + c * 32, va);
        tmem_ld32_nowait(tbase + c * 32 + 32, vb);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + 2 == c_hi) {
          // release the accumulator: one arrival per warp, at the leader for a pair
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR) mbar_arrive_remote(tempty0 + 8 * acc, 0);
            else mbar_arrive(tempty0 + 8 * acc);
          }
        }
        float ma[11], mb[11];
        const float mna = chunk_min(va, ma), mnb = chunk_min(vb, mb);
        const bool ok = live && gcnt <= P.capg;
        const bool hita = ok && mna <= tau_e, hitb = ok && mnb <= tau_e;
        if (!__any_sync(0xffffffffu, hita || hitb)) continue;
        const uint32_t cbase = tile_of(t) * W + c * 32;
        scan(va, ma, cbase, hita);
        scan(vb, mb, cbase + 32, hitb);
      }
    }
    if (kmode == 0) {
      flush(0);
    } else if (kmode == 2) {
#if CAGRA_TC_MAXLIST
      if (live && tmax != P.KC - 1) {  // the maximum goes last
        const uint64_t a = mypend[tmax * ROWS + rl];
        mypend[tmax * ROWS + rl] = mypend[(P.KC - 1) * ROWS + rl];
        mypend[(P.KC - 1) * ROWS + rl] = a;
      }
#endif
      if (live)
        for (uint32_t i = 0; i < P.KC; ++i)
          lists[(size_t)row * P.KC + i] = mypend[i * ROWS + rl];
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

// FP16 single-term split (the default filter).  With x' = fl(x - mu) and a
// power of two s chosen so that s |x'| < 2^13 for every data and query row:
//   query side P = [-2 h(s q') | sig sig | 0..]
//   data side  R = [ h(s x')   | n0  n1  | 0..]     sig = 2^14,
// h = round-to-nearest fp16, n0 + n1 = h-split of s^2 |x'|^2 / sig, so the GEMM
// yields e = s^2 (|x'|^2 - 2 q'.x') up to the fp16 rounding of the operands
// (relative 2^-11 each: |2 q.x - 2 h(q).h(x)| <= 2 (2^-10 + 2^-22) |q||x|) and
// the epilogue adds the row constant s^2 |q'|^2.  K = dim + 2 instead of the
// bf16x3 split's 3 dim + 6: 2.5x fewer MMA steps and B-tile bytes at 96-d.
// Pass 1: |x'|^2 per row (the same fmaf chain as tc_split_kernel) + its max.
__global__ void tc_norm_kernel(const float* __restrict__ src, uint32_t rows, uint32_t ld,
                               uint32_t dim, const float* __restrict__ mu,
                               float* __restrict__ norms, uint32_t* __restrict__ maxnorm_bits) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = src + (size_t)row * ld;
  float ss = 0.0f;
  for (uint32_t i = lane; i < dim; i += 32) {
    const float v = x[i] - mu[i];
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    norms[row] = ss;
    atomicMax(maxnorm_bits, __float_as_uint(ss));
  }
}
constexpr float kSplit16Sigma = 16384.0f;
// Pass 2: the fp16 rows (P and/or R) of `rows` rows, scale s (exact power of 2).
__global__ void tc_split16_kernel(const float* __restrict__ src, uint32_t rows, uint32_t ld,
                                  uint32_t dim, uint32_t Kp, const float* __restrict__ mu, float sc,
                                  const float* __restrict__ norms, __half* __restrict__ P,
                                  __half* __restrict__ R) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = src + (size_t)row * ld;
  __half* p = P ? P + (size_t)row * Kp : nullptr;
  __half* r = R ? R + (size_t)row * Kp : nullptr;
  for (uint32_t i = lane; i < dim; i += 32) {
    const __half h = __float2half_rn((x[i] - mu[i]) * sc);
    if (p) p[i] = __float2half_rn(-2.0f * __half2float(h));  // exact
    if (r) r[i] = h;
  }
  const float nn = norms[row] * (sc * sc) * (1.0f / kSplit16Sigma);  // exact scaling
  const __half n0 = __float2half_rn(nn);
  const __half n1 = __float2half_rn(nn - __half2float(n0));
  const __half zero = __float2half_rn(0.0f), sig = __float2half_rn(kSplit16Sigma);
  for (uint32_t i = dim + lane; i < Kp; i += 32) {
    const uint32_t j = i - dim;
    if (p) p[i] = j < 2 ? sig : zero;
    if (r) r[i] = j == 0 ? n0 : (j == 1 ? n1 : zero);
  }
}

// --------------------------------------------------------------- rerank ----
// One warp per query row: band selection on d~, exact sequential-chain
// distances, (dist, id) sort, first k.  Rows whose band overflows the KC keys
// are queued for the exact SIMT kernel.
__global__ void tc_rerank_kernel(const uint64_t* __restrict__ lists, uint32_t nq, uint32_t KC,
                                 uint32_t K, const float* __restrict__ qnorm, float xm,
                                 float dscale, float eps_rel,
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
  // delta in distance units; d~ keys are in GEMM units (x dscale = s^2)
  const float delta = eps_rel * sqrtf(qn) * sqrtf(xm) + eps_norm * (qn + xm);
  const float bound = key_dist(kth) + 2.0f * delta * dscale;
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
      const float acc = seq_dist(x, q, dim);
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

// Sort the first c (<= 32 E) keys of b ascending, warp-wide, in place.
template <int E>
__device__ __forceinline__ void sort_keys_inplace(uint64_t* b, uint32_t c, int lane) {
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
}

// Append-mode rerank: one warp per row.  The buffer holds EVERY point with
// d~ <= tau* (tau* from the sample pass).  Valid iff K <= count <= capg and
// d~_(K) + 2 delta <= tau* (then every point that can be a true top-K member
// is in the buffer); otherwise the row is queued for the list-mode pass.
// Two instantiations keep the common case light on registers (occupancy is
// what hides the row gathers): ES = 16 sorts rows of <= 512 keys and queues
// larger ones on `big`; ES = 32 then runs over the `big` rows only.
struct AppendRerank {
  uint64_t* bufs;
  const uint32_t* bcount;
  uint32_t capg;
  const uint64_t* tau_keys;
  uint32_t tau_ld, nq, K;
  const float* qnorm;
  float xm, dscale, eps_rel, eps_norm;
  const float* data;
  uint32_t ld;
  const float* queries;
  uint32_t qld, dim;
  uint32_t* out_ids;
  float* out_dists;
  uint32_t* fail_rows;
  uint32_t* fail_cnt;
  uint32_t* big_rows;  // [0] = count, rows from [1]
  unsigned long long* reranked;
};

template <int ES>
__device__ __forceinline__ void rerank_append_row(const AppendRerank& A, uint32_t row, int lane) {
  uint64_t* __restrict__ bufs = A.bufs;
  const uint32_t capg = A.capg, K = A.K, ld = A.ld, qld = A.qld, dim = A.dim;
  const float xm = A.xm, dscale = A.dscale, eps_rel = A.eps_rel, eps_norm = A.eps_norm;
  const float* __restrict__ data = A.data;
  const float* __restrict__ queries = A.queries;
  const uint32_t c = A.bcount[row];
  const float tau_star = key_dist(A.tau_keys[(size_t)row * A.tau_ld + A.tau_ld - 1]);
  uint64_t* b = bufs + (size_t)row * capg;
  bool ok = c >= K && c <= capg;
  float bound = 0.0f;
  if (ok) {
    // the smallest warp sort that holds the row's keys (typically ~430)
    if (c <= 256) {
      sort_keys_inplace<8>(b, c, lane);
    } else if (c <= 512) {
      sort_keys_inplace<16>(b, c, lane);
    } else if (ES == 32) {
      sort_keys_inplace<32>(b, c, lane);
    } else {
      if (lane == 0) A.big_rows[1 + atomicAdd(A.big_rows, 1u)] = row;
      return;
    }
    const float qn = A.qnorm[row];
    const float delta = eps_rel * sqrtf(qn) * sqrtf(xm) + eps_norm * (qn + xm);
    bound = key_dist(b[K - 1]) + 2.0f * delta * dscale;
    ok = bound <= tau_star;
  }
  if (!ok) {
    if (lane == 0) A.fail_rows[atomicAdd(A.fail_cnt, 1u)] = row;
    return;
  }
  // exact sequential-chain distances for the band, cyclic over lanes: slot
  // e * 32 + lane of the sorted buffer; 4 slots' chains interleaved, and a
  // group is skipped once no lane's slot is in the band (the buffer is sorted)
  constexpr int E2 = 8, G = 4;
  uint64_t w[E2];
  const float* q = queries + (size_t)row * qld;
  uint32_t nre = 0;
  bool over = false;
#pragma unroll
  for (int e0 = 0; e0 < E2; e0 += G) {
    uint32_t id[G];
    bool in[G];
    const float* xs[G];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const uint32_t i = (e0 + u) * 32 + lane;
      const uint64_t key = i < c ? b[i] : kDummyKey;
      in[u] = !key_is_dummy(key) && key_dist(key) <= bound;
      id[u] = in[u] ? key_id(key) : key_id(b[0]);  // out of band: a cached row
      xs[u] = data + (size_t)id[u] * ld;
    }
    if (!__any_sync(0xffffffffu, in[0])) {
#pragma unroll
      for (int u = 0; u < G; ++u) w[e0 + u] = kDummyKey;
      continue;
    }
    float acc[G];
    seq_dist_multi<G>(xs, q, dim, acc);
#pragma unroll
    for (int u = 0; u < G; ++u) {
      w[e0 + u] = in[u] ? make_key(acc[u], id[u]) : kDummyKey;
      nre += in[u] ? 1u : 0u;
    }
  }
  // the band must fit the 256 re-rank slots
  if (c > 32 * E2 && key_dist(b[32 * E2]) <= bound) over = true;
  if (__any_sync(0xffffffffu, over)) {
    if (lane == 0) A.fail_rows[atomicAdd(A.fail_cnt, 1u)] = row;
    return;
  }
  warp_sort_regs<E2>(w, lane);
#pragma unroll
  for (int e = 0; e < E2; ++e) {
    const uint32_t i = lane * E2 + e;
    if (i < K) {
      A.out_ids[(size_t)row * K + i] = key_id(w[e]);
      A.out_dists[(size_t)row * K + i] = key_dist(w[e]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nre += __shfl_xor_sync(0xffffffffu, nre, o);
  if (lane == 0 && A.reranked) atomicAdd(A.reranked, (unsigned long long)nre);
}

// ES = 16: every row (grid covers nq warps); ES = 32: the queued big rows
template <int ES>
__global__ void __launch_bounds__(256, ES == 16 ? 3 : 1) tc_rerank_append_kernel(const AppendRerank A) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (ES == 16) {
    if (w < A.nq) rerank_append_row<16>(A, w, lane);
  } else {
    const uint32_t nb = *(volatile const uint32_t*)A.big_rows;
    for (uint32_t i = w; i < nb; i += gridDim.x * (blockDim.x / 32))
      rerank_append_row<32>(A, A.big_rows[1 + i], lane);
  }
}

// Column-split list passes: per row, merge groups of up to m sorted KC-key
// lists (slabs [g][nq][KC]) into one sorted KC-key list (m * KC <= 1024).
__global__ void merge_lists_kernel(const uint64_t* __restrict__ in, uint32_t g_in, uint32_t m,
                                   uint32_t nq, uint32_t KC, uint64_t* __restrict__ out) {
  const uint32_t row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  const uint32_t grp = blockIdx.y;
  if (row >= nq) return;
  const uint32_t g0 = grp * m, gn = min(m, g_in - g0);
  constexpr int E = 32;
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e, g = i / KC, j = i - g * KC;
    v[e] = g < gn ? in[((size_t)(g0 + g) * nq + row) * KC + j] : kDummyKey;
  }
  warp_sort_regs<E>(v, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e;
    if (i < KC) out[((size_t)grp * nq + row) * KC + i] = v[e];
  }
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
// Stream-ordered scratch of the occasional paths (small-batch list pass,
// retried rows): cudaMallocAsync from the device pool, whose release threshold
// is raised once so freed blocks stay mapped — a plain cudaMalloc/cudaFree
// pair here was measured stalling the host for up to ~350 ms between passes.
void keep_pool_mapped() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || done[dev & 63]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev & 63] = true;
}
struct Dev {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  Dev(size_t b, cudaStream_t st) : s(st) {
    keep_pool_mapped();
    CAGRA_CUDA_TRY(cudaMallocAsync(&p, b ? b : 16, s));
  }
  ~Dev() {
    if (p) cudaFreeAsync(p, s);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// Grow-only per-device scratch of the main kNN path (operand rows, norms,
// candidate buffers).  A cold 4 GB cudaMalloc costs tens to hundreds of ms of
// host time inside the build; repeated builds (shards, ground truth, benches)
// reuse the same memory.  cagra_trim_scratch() releases it.  Builds on one
// device are serialised by that device's g_knn_mu (they share its arena);
// builds on different devices run concurrently (row-sharded multi-GPU build).
enum ArenaSlot { kSlotP, kSlotR, kSlotQn, kSlotXn, kSlotMax, kSlotMu, kSlotPart, kSlotLists,
                 kSlotBufs, kSlotBcount, kSlotFails, kSlotRer, kSlotCount };
struct Arena {
  void* p[kSlotCount] = {};
  size_t cap[kSlotCount] = {};
};
std::mutex g_knn_mu[64];
Arena g_arena[64];
struct View {  // non-owning view of an arena slot
  void* p;
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};
void* arena(int slot, size_t bytes) {
  int dev = 0;
  CAGRA_CUDA_TRY(cudaGetDevice(&dev));
  Arena& a = g_arena[dev & 63];
  if (bytes == 0) bytes = 16;
  if (a.cap[slot] < bytes) {
    if (a.p[slot]) cudaFree(a.p[slot]);
    a.p[slot] = nullptr;
    a.cap[slot] = 0;
    CAGRA_CUDA_TRY(cudaMalloc(&a.p[slot], bytes));
    a.cap[slot] = bytes;
  }
  return a.p[slot];
}

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
                     uint32_t box_rows, bool f16) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {Kp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * 2 * row_step};
  cuuint32_t box[2] = {TC_BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tm, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed");
  return tm;
}

// the query tile is streamed (SA) when it cannot stay resident
bool tc_streamed(uint32_t kblocks) { return kblocks > TC_MAX_KB; }

size_t tc_smem_bytes(uint32_t kblocks, uint32_t stages, uint32_t pend_cap = TC_PEND,
                     bool pair = false, uint32_t hv = 1) {
  const bool sa = tc_streamed(kblocks);
  const bool ts = CAGRA_KNN_TS && !pair && !sa && hv == 1;
  const bool w64 = hv == 2 && CAGRA_TC_W64;
  const size_t stage = sa ? 3 * TILE_BYTES : (pair || w64 ? TILE_BYTES / 2 : TILE_BYTES);
  const uint32_t acc = ts || sa ? 2 : (hv == 2 ? (w64 ? 4 : 2) : 4);
  return 1024 + (ts || sa ? 0 : (size_t)hv * kblocks * TILE_BYTES) + stages * stage +
         sizeof(uint64_t) * (pend_cap * TC_BM * hv + 2 * stages + 1 + 2 * acc) + 16;
}

constexpr size_t kSmemLimit = 227 * 1024;

// deepest B ring that fits next to the resident query tile
uint32_t tc_stages(uint32_t kblocks, uint32_t pend_cap = TC_PEND, bool pair = false,
                   uint32_t hv = 1) {
  uint32_t s = pair || (hv == 2 && CAGRA_TC_W64) ? 2 * TC_STAGES : TC_STAGES;  // half tiles
  while (s > 2 && tc_smem_bytes(kblocks, s, pend_cap, pair, hv) > kSmemLimit) --s;
  return s;
}

// two 128-row halves per CTA when A (both halves) + a >= 3-deep B ring fits
uint32_t tc_halves(uint32_t kblocks, uint32_t pend_cap) {
  const char* e = std::getenv("CAGRA_TC_HALVES");
  if (e && e[0] == '1') return 1;
  if (tc_streamed(kblocks)) return 1;
  return tc_smem_bytes(kblocks, 3, pend_cap, false, 2) <= kSmemLimit ? 2 : 1;
}

}  // namespace

KnnTcStats g_knn_tc_stats;

void knn_trim_scratch(int device) {
  for (int d = 0; d < 64; ++d) {
    if (device >= 0 && d != device) continue;
    std::lock_guard<std::mutex> lk(g_knn_mu[d]);
    Arena& a = g_arena[d];
    for (int i = 0; i < kSlotCount; ++i) {
      if (!a.p[i]) continue;
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(d);
      cudaFree(a.p[i]);
      cudaSetDevice(cur);
      a.p[i] = nullptr;
      a.cap[i] = 0;
    }
  }
}

namespace {
// Filter split: 1 = fp16 single term (default), 3 = bf16x3 (CAGRA_KNN_SPLIT=3).
uint32_t split_terms() {
  const char* e = std::getenv("CAGRA_KNN_SPLIT");
  return e && e[0] == '3' ? 3u : 1u;
}
uint32_t split_k(uint32_t dim, uint32_t terms) { return terms == 1 ? dim + 2 : 3 * dim + 6; }
}  // namespace

bool knn_tc_eligible(uint32_t dim, uint32_t K) {
  const char* env = std::getenv("CAGRA_KNN_PATH");
  if (env && std::strcmp(env, "simt") == 0) return false;
  uint32_t Kp = round_up_u32(split_k(dim, split_terms()), TC_BK);
  const uint32_t kb = Kp / TC_BK;
  if (kb > TC_MAX_KB_STREAM || K + 32 + TC_PEND > 256) return false;
  if (tc_streamed(kb)) return tc_smem_bytes(kb, 3) <= kSmemLimit;  // >= 3-deep A+B+B ring
  return tc_smem_bytes(kb, tc_stages(kb, TC_PEND, true), TC_PEND, true) <= kSmemLimit;
}

namespace {

// CAGRA_KNN_TRACE=1: device-event and host-wall time of every build phase to
// stderr (diagnostics for the build-time spread across runs).
struct Tracer {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> wall;
  std::chrono::steady_clock::time_point t0;
  explicit Tracer(cudaStream_t st) : s(st) {
    const char* e = std::getenv("CAGRA_KNN_TRACE");
    on = e && e[0] == '1';
    if (on) t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* name) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
    wall.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
  }
  ~Tracer() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    std::fprintf(stderr, "[knn trace]");
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      std::fprintf(stderr, " %s %.2fms(host %.1f)", ev[i].first, ms, wall[i]);
    }
    std::fprintf(stderr, "\n");
    for (auto& p : ev) cudaEventDestroy(p.second);
  }
};

// Everything one kNN / top-k call shares between its passes.
struct TcCall {
  const float* data;
  uint32_t n, ld, dim, K, Kp, kblocks, stages;
  bool exclude_self;
  uint32_t self_base;  // kNN rows [self_base, self_base + nq) of the graph (row-sharded builds)
  float eps_rel, eps_norm;
  float xm;            // max |x'|^2 the error bound uses
  uint32_t terms;      // 1: fp16 single-term split, 3: bf16x3
  float dscale;        // s^2 (1 for bf16x3): d~ keys are in GEMM units
  uint32_t ksteps_last;
  const void* R;  // n x Kp 16-bit operand rows
  cudaStream_t stream;
};

// CTA pairs (cluster of 2, cta_group::2 MMA) with CAGRA_TC_PAIR=1.
bool tc_pair_enabled() {
  const char* e = std::getenv("CAGRA_TC_PAIR");  // measured slower than single CTAs: opt-in
  return e && e[0] == '1';
}

void run_tc_kernel(const TcCall& c, const void* Pq, const CUtensorMap& tmA,
                   const CUtensorMap& tmB, TcArgs a, uint32_t nq, uint32_t splits = 1) {
  const bool sa = tc_streamed(c.kblocks);
  const bool pair = tc_pair_enabled() && !sa;
  a.kblocks = c.kblocks;
  a.prow = reinterpret_cast<const uint32_t*>(Pq);
  a.ab_fmt = c.terms == 1 ? 0u : 1u;
  a.ksteps_last = c.ksteps_last;
  a.dscale = c.dscale;
  a.pend_cap = a.mode == 1 ? TC_PEND_APPEND : (a.mode == 2 ? a.KC + 32 : TC_PEND);
  const uint32_t hv = pair ? 1 : tc_halves(c.kblocks, a.pend_cap);
  a.stages = tc_stages(c.kblocks, a.pend_cap, pair, hv);
  a.exclude_self = c.exclude_self ? 1 : 0;
  a.nq = nq;
  const size_t smem = tc_smem_bytes(c.kblocks, a.stages, a.pend_cap, pair, hv);
  if (!sa && !pair && hv == 2) {
    // one instantiation per epilogue mode: the hot full pass carries no
    // list/insertion code (registers and code size)
    auto fn = a.mode == 1 ? knn_tc_kernel<false, false, 2, 1>
                          : (a.mode == 2 ? knn_tc_kernel<false, false, 2, 2>
                                         : knn_tc_kernel<false, false, 2, 0>);
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<dim3((nq + 2 * TC_BM - 1) / (2 * TC_BM), splits), 64 + 2 * TC_BM, smem, c.stream>>>(
        tmA, tmB, a);
    CAGRA_LAUNCH_CHECK();
    return;
  }
  if (sa) {
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<false, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    knn_tc_kernel<false, true>
        <<<dim3((nq + TC_BM - 1) / TC_BM, splits), TC_THREADS, smem, c.stream>>>(tmA, tmB, a);
    CAGRA_LAUNCH_CHECK();
    return;
  }
  if (!pair) {
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    knn_tc_kernel<false>
        <<<dim3((nq + TC_BM - 1) / TC_BM, splits), TC_THREADS, smem, c.stream>>>(tmA, tmB, a);
    CAGRA_LAUNCH_CHECK();
    return;
  }
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(knn_tc_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * ((nq + 2 * TC_BM - 1) / (2 * TC_BM)), splits);
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
  // column splits: enough CTAs to cover the SMs when the batch is small
  int dev = 0, sms = 148;
  CAGRA_CUDA_TRY(cudaGetDevice(&dev));
  CAGRA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint32_t row_ctas = (nq + 2 * TC_BM - 1) / (2 * TC_BM);
  const uint32_t ntiles = (c.n + TC_BN - 1) / TC_BN;
  // (only when the row CTAs leave most SMs idle: every split re-fills its
  // own list from scratch, which costs more than it saves on a half-full GPU)
  uint32_t splits = row_ctas * 2 >= (uint32_t)sms
                        ? 1u
                        : std::min<uint32_t>((2u * (uint32_t)sms + row_ctas - 1) / row_ctas,
                                             std::max<uint32_t>(1, ntiles / 8));
  if (std::getenv("CAGRA_TC_NOSPLIT")) splits = 1;
  Dev lists(8ull * nq * KC * splits, c.stream), fails(4ull * nq + 4, c.stream), rer(8, c.stream);
  CAGRA_CUDA_TRY(cudaMemsetAsync(fails.p, 0, 4ull * nq + 4, c.stream));
  CAGRA_CUDA_TRY(cudaMemsetAsync(rer.p, 0, 8, c.stream));
  const uint32_t brows = BOX_ROWS;  // every B load is one or more 64-point boxes
  const bool f16 = c.terms == 1;
  CUtensorMap tmA = make_map(P, nq, c.Kp, 1, TC_BN, f16),
              tmB = make_map(c.R, c.n, c.Kp, 1, brows, f16);
  TcArgs a{};
  a.qnorm = f16 ? qnorm : nullptr;
  a.n = c.n;
  a.KC = KC;
  a.mode = KC <= 48 ? 2 : 0;  // short lists: per-row insertion lists in smem
  a.col_stride = 1;
  a.lists = lists.as<uint64_t>();
  a.self_ids = self_ids;
  a.self_base = self_ids ? 0 : c.self_base;
  run_tc_kernel(c, P, tmA, tmB, a, nq, splits);
  if (splits > 1) {
    // merge the split lists in rounds of m per row until one remains
    const uint32_t m = std::max<uint32_t>(2, 1024 / KC);
    uint32_t g = splits;
    uint64_t* src = lists.as<uint64_t>();
    Dev tmp(8ull * nq * KC * ((splits + m - 1) / m), c.stream);
    uint64_t* dst = tmp.as<uint64_t>();
    while (g > 1) {
      const uint32_t go = (g + m - 1) / m;
      merge_lists_kernel<<<dim3((nq + 7) / 8, go), 256, 0, c.stream>>>(src, g, m, nq, KC, dst);
      CAGRA_LAUNCH_CHECK();
      std::swap(src, dst);
      g = go;
    }
    if (src != lists.as<uint64_t>())
      CAGRA_CUDA_TRY(cudaMemcpyAsync(lists.p, src, 8ull * nq * KC, cudaMemcpyDeviceToDevice,
                                     c.stream));
  }
  uint32_t* fail_cnt = fails.as<uint32_t>();
  uint32_t* fail_rows = fail_cnt + 1;
  tc_rerank_kernel<<<(nq + 7) / 8, 256, 0, c.stream>>>(
      lists.as<uint64_t>(), nq, KC, c.K, qnorm, c.xm, c.dscale, c.eps_rel, c.eps_norm, c.data, c.ld,
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
  Dev q((size_t)nf * qld * 4, c.stream), sid(4ull * nf, c.stream), sc(8ull * nf * c.K, c.stream),
      fi(4ull * nf * c.K, c.stream), fd(4ull * nf * c.K, c.stream);
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
  int lk_dev = 0;
  CAGRA_CUDA_TRY(cudaGetDevice(&lk_dev));
  std::lock_guard<std::mutex> lk(g_knn_mu[lk_dev & 63]);
  Tracer tr(stream);
  tr.mark("start");
  TcCall c;
  c.self_base = exclude_self ? self_base : 0;
  c.data = d_data;
  c.n = n;
  c.ld = ld;
  c.dim = dim;
  c.K = K;
  c.terms = split_terms();
  const uint32_t kv = round_up_u32(split_k(dim, c.terms), 16);  // K in 16-wide MMA steps
  c.Kp = round_up_u32(kv, TC_BK);
  c.kblocks = c.Kp / TC_BK;
  c.ksteps_last = (kv - (c.kblocks - 1) * TC_BK) / 16;
  c.stages = tc_stages(c.kblocks);
  c.exclude_self = exclude_self;
  c.stream = stream;
  // error bound of d~ (file header): |d~ - d| <= eps_rel |q| max|x| +
  // eps_norm (|q|^2 + max|x|^2), norms of the centred rows x' = fl(x - mu).
  //  * split: bf16x3 omits 3.1*2^-16 of sum|q_i||x_i| <= |q||x|; the fp16
  //    single term rounds both operands (2^-10 + 2^-22), both doubled by -2;
  //  * fp32 accumulation over Kp terms of total magnitude 2|q||x| + |q|^2 +
  //    |x|^2 (counted with 2^-23 per term: no assumption on the tensor core's
  //    rounding), the fp32 norms (dim + 8 terms), the epilogue's row-offset
  //    add (2 u), the centring rounding (|d - |x'-q'|^2| <= 2u (|x'| + |q'|)^2);
  //  * fp16 only: the 2-term norm split (2^-22, counted 2^-21) and operands
  //    below the fp16 normal range (absolute 2^-25 in GEMM units <= 2^-35
  //    max|x'|^2 per element; counted 2^-28 for any dim <= 2^12).
  const float u23 = 1.1920929e-07f;
  if (c.terms == 1) {
    c.eps_rel = 2.0f * (9.765625e-04f + 2.3841858e-07f) + 2.0f * (float)c.Kp * u23 + 4.0f * u23;
    c.eps_norm = (float)c.Kp * u23 + (float)(dim + 8) * u23 + 4.0f * u23 + 4.76837158e-07f +
                 3.7252903e-09f;
  } else {
    c.eps_rel = 2.0f * 3.1f * 1.52587890625e-05f + 2.0f * (float)c.Kp * u23 + 4.0f * u23;
    c.eps_norm = (float)c.Kp * u23 + (float)(dim + 8) * u23 + 2.0f * u23;
  }

  // kNN graph: the queries are data rows [self_base, self_base + nq), so the
  // data split also yields their query-side rows
  const bool same = exclude_self;
  View dP{arena(kSlotP, (size_t)(same ? n : nq) * c.Kp * 2)},
      dR{arena(kSlotR, (size_t)n * c.Kp * 2)}, dqn{arena(kSlotQn, 4ull * nq)},
      dxn{arena(kSlotXn, 4ull * n)}, dmax{arena(kSlotMax, 8)};
  CAGRA_CUDA_TRY(cudaMemsetAsync(dmax.p, 0, 8, stream));
  View dmu{arena(kSlotMu, 4ull * dim)}, dpart{arena(kSlotPart, 8ull * kMeanChunks * dim)};
  col_mean_partial_kernel<<<dim3((dim + 31) / 32, kMeanChunks), 256, 0, stream>>>(
      d_data, n, ld, dim, dpart.as<double>());
  col_mean_final_kernel<<<(dim + 127) / 128, 128, 0, stream>>>(dpart.as<double>(), n, dim,
                                                               dmu.as<float>());
  CAGRA_LAUNCH_CHECK();
  uint32_t* dmaxx = dmax.as<uint32_t>();
  uint32_t* dmaxq = dmaxx + 1;
  if (c.terms == 1) {
    tc_norm_kernel<<<(n + 7) / 8, 256, 0, stream>>>(d_data, n, ld, dim, dmu.as<float>(),
                                                    dxn.as<float>(), dmaxx);
    if (!same)
      tc_norm_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(d_queries, nq, qld, dim, dmu.as<float>(),
                                                       dqn.as<float>(), dmaxq);
    CAGRA_LAUNCH_CHECK();
    uint32_t hm[2] = {0, 0};
    CAGRA_CUDA_TRY(cudaMemcpyAsync(hm, dmax.p, 8, cudaMemcpyDeviceToHost, stream));
    CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    float mx;
    uint32_t mb = std::max(hm[0], hm[1]);
    std::memcpy(&mx, &mb, 4);
    // s = 2^(13 - E) with sqrt(mx) = f 2^E, f in [0.5, 1): s |x'| < 2^13
    int E = 0;
    if (mx > 0.0f) std::frexp(std::sqrt((double)mx), &E);
    const int se = mx > 0.0f ? 13 - E : 0;
    if (se < -60 || se > 60) {
      c.terms = 3;  // outside the exponent range the fp16 scaling can represent
    } else {
      const float sc = std::ldexp(1.0f, se);
      c.dscale = sc * sc;
      c.xm = mx;
      tc_split16_kernel<<<(n + 7) / 8, 256, 0, stream>>>(
          d_data, n, ld, dim, c.Kp, dmu.as<float>(), sc, dxn.as<float>(),
          same ? dP.as<__half>() : nullptr, dR.as<__half>());
      if (!same)
        tc_split16_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(d_queries, nq, qld, dim, c.Kp,
                                                            dmu.as<float>(), sc, dqn.as<float>(),
                                                            dP.as<__half>(), nullptr);
      CAGRA_LAUNCH_CHECK();
    }
    if (c.terms == 3) {  // re-derive the bf16x3 layout (rare: extreme magnitudes)
      const uint32_t kv3 = round_up_u32(split_k(dim, 3), 16);
      if (round_up_u32(kv3, TC_BK) / TC_BK > TC_MAX_KB_STREAM)
        throw CudaErr("knn_tc: dimension beyond the bf16x3 path");
      c.Kp = round_up_u32(kv3, TC_BK);
      c.kblocks = c.Kp / TC_BK;
      c.ksteps_last = (kv3 - (c.kblocks - 1) * TC_BK) / 16;
      c.stages = tc_stages(c.kblocks);
      c.eps_rel = 2.0f * 3.1f * 1.52587890625e-05f + 2.0f * (float)c.Kp * u23 + 4.0f * u23;
      c.eps_norm = (float)c.Kp * u23 + (float)(dim + 8) * u23 + 2.0f * u23;
      dP.p = arena(kSlotP, (size_t)(same ? n : nq) * c.Kp * 2);
      dR.p = arena(kSlotR, (size_t)n * c.Kp * 2);
      CAGRA_CUDA_TRY(cudaMemsetAsync(dmax.p, 0, 8, stream));
    }
  }
  if (c.terms == 3) {
    c.dscale = 1.0f;
    // data side: R (and P when the queries are the data), norms, max norm
    tc_split_kernel<<<(n + 7) / 8, 256, 0, stream>>>(d_data, n, ld, dim, c.Kp, dmu.as<float>(),
                                                     same ? dP.as<__nv_bfloat16>() : nullptr,
                                                     dR.as<__nv_bfloat16>(), dxn.as<float>(),
                                                     dmaxx);
    CAGRA_LAUNCH_CHECK();
    if (!same) {
      tc_split_kernel<<<(nq + 7) / 8, 256, 0, stream>>>(d_queries, nq, qld, dim, c.Kp,
                                                        dmu.as<float>(), dP.as<__nv_bfloat16>(),
                                                        nullptr, dqn.as<float>(), nullptr);
      CAGRA_LAUNCH_CHECK();
    }
    uint32_t hm = 0;
    CAGRA_CUDA_TRY(cudaMemcpyAsync(&hm, dmaxx, 4, cudaMemcpyDeviceToHost, stream));
    CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    std::memcpy(&c.xm, &hm, 4);
  }
  tr.mark("prep");
  const float* qnorm_all = same ? dxn.as<float>() + c.self_base : dqn.as<float>();
  const uint16_t* Pq_all = dP.as<uint16_t>() + (same ? (size_t)c.self_base * c.Kp : 0);
  c.R = dR.p;
  uint64_t reranked = 0, fallback = 0, retried = 0;

  const char* onepass = std::getenv("CAGRA_TC_ONEPASS");
  // two passes need enough query rows to fill the SMs (and enough points for
  // a meaningful sample); small batches (ground truth, retries) take the
  // column-split list pass instead
  int cur_dev = 0, n_sms = 148;
  CAGRA_CUDA_TRY(cudaGetDevice(&cur_dev));
  CAGRA_CUDA_TRY(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, cur_dev));
  const bool two_pass = n / kSampleStride >= 4096 && nq >= (uint32_t)n_sms * 2 * TC_BM &&
                        !(onepass && onepass[0] == '1');
  if (!two_pass) {
    list_pass(c, Pq_all, nq, qnorm_all, d_queries, qld, nullptr, d_ids, d_dists, reranked,
              fallback);
  } else {
    // Rows in chunks of <= 512k so every row keeps a 1024-key append buffer
    // (4 GB per chunk): a smaller buffer overflowed for ~15% of the rows at
    // 10M points (the count of d~ <= tau* has a standard deviation of ~80).
    constexpr uint32_t kChunk = 512u * 1024u;
    const uint32_t ns = n / kSampleStride;
    // r-th smallest of the sample: ~16 r points per row pass tau* (>= K plus
    // the band with margin: 16 x 24 = 384, standard deviation ~80); r <= 24
    // keeps the sample pass's smem lists next to two A halves
    uint32_t r = std::min<uint32_t>(
        24, std::max<uint32_t>(8, (3 * (K + 16) + kSampleStride - 1) / kSampleStride));
    if (const char* er = std::getenv("CAGRA_TC_SAMPLE_R"))  // A/B: sample rank (8..24)
      r = std::min<uint32_t>(24, std::max<uint32_t>(8, (uint32_t)std::atoi(er)));
    const uint32_t capg = 1024;
    const uint32_t cmax = std::min(nq, kChunk);
    View lists1{arena(kSlotLists, 8ull * r * cmax)}, bufs{arena(kSlotBufs, 8ull * cmax * capg)},
        bcount{arena(kSlotBcount, 4ull * cmax)}, fails{arena(kSlotFails, 8ull * cmax + 8)},
        rer{arena(kSlotRer, 8)};
    const uint32_t brows = BOX_ROWS;  // every B load is one or more 64-point boxes
    const bool f16 = c.terms == 1;
    CUtensorMap tmS = make_map(dR.p, ns, c.Kp, kSampleStride, brows, f16);
    CUtensorMap tmB = make_map(dR.p, n, c.Kp, 1, brows, f16);
    for (uint32_t q0 = 0; q0 < nq; q0 += kChunk) {
      const uint32_t cq = std::min(kChunk, nq - q0);
      const uint16_t* Pq = Pq_all + (size_t)q0 * c.Kp;
      const float* qnorm = qnorm_all + q0;
      const float* cqueries = d_queries + (size_t)q0 * qld;
      uint32_t* cids = d_ids + (size_t)q0 * K;
      float* cdists = d_dists + (size_t)q0 * K;
      TcCall cc = c;
      cc.self_base = c.self_base + q0;
      CAGRA_CUDA_TRY(cudaMemsetAsync(fails.p, 0, 4, stream));  // the fail count
      CAGRA_CUDA_TRY(cudaMemsetAsync(fails.as<uint32_t>() + 1 + cmax, 0, 4, stream));  // big count
      CAGRA_CUDA_TRY(cudaMemsetAsync(rer.p, 0, 8, stream));
      CAGRA_CUDA_TRY(cudaMemsetAsync(bcount.p, 0, 4ull * cq, stream));  // append counters
      CUtensorMap tmA = make_map(Pq, cq, c.Kp, 1, TC_BN, f16);
      // pass 1: every 16th point; the r-th smallest d~ over the sample is an
      // upper bound of the r-th smallest over all points (valid for ANY r).
      TcArgs a{};
      a.n = ns;
      a.KC = r;
      a.mode = 2;  // r <= 48: per-row insertion lists in shared memory
      a.col_stride = kSampleStride;
      a.lists = lists1.as<uint64_t>();
      a.self_base = cc.self_base;
      a.qnorm = f16 ? qnorm : nullptr;
      tr.mark("setup");
      run_tc_kernel(cc, Pq, tmA, tmS, a, cq);
      tr.mark("sample");
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
      b.self_base = cc.self_base;
      b.qnorm = a.qnorm;
      run_tc_kernel(cc, Pq, tmA, tmB, b, cq);
      tr.mark("full");
      uint32_t* fail_cnt = fails.as<uint32_t>();
      uint32_t* fail_rows = fail_cnt + 1;
      AppendRerank ar;
      ar.bufs = bufs.as<uint64_t>();
      ar.bcount = bcount.as<uint32_t>();
      ar.capg = capg;
      ar.tau_keys = lists1.as<uint64_t>();
      ar.tau_ld = r;
      ar.nq = cq;
      ar.K = K;
      ar.qnorm = qnorm;
      ar.xm = c.xm;
      ar.dscale = c.dscale;
      ar.eps_rel = c.eps_rel;
      ar.eps_norm = c.eps_norm;
      ar.data = d_data;
      ar.ld = ld;
      ar.queries = cqueries;
      ar.qld = qld;
      ar.dim = dim;
      ar.out_ids = cids;
      ar.out_dists = cdists;
      ar.fail_rows = fail_rows;
      ar.fail_cnt = fail_cnt;
      ar.big_rows = fail_rows + cmax;  // [count, rows...] after the fail list
      ar.reranked = rer.as<unsigned long long>();
      tc_rerank_append_kernel<16><<<(cq + 7) / 8, 256, 0, stream>>>(ar);
      tc_rerank_append_kernel<32><<<std::min<uint32_t>((cq + 7) / 8, 148 * 8), 256, 0, stream>>>(ar);
      CAGRA_LAUNCH_CHECK();
      uint32_t nf = 0;
      unsigned long long nre = 0;
      CAGRA_CUDA_TRY(cudaMemcpyAsync(&nf, fail_cnt, 4, cudaMemcpyDeviceToHost, stream));
      CAGRA_CUDA_TRY(cudaMemcpyAsync(&nre, rer.p, 8, cudaMemcpyDeviceToHost, stream));
      CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
      reranked += nre;
      retried += nf;
      tr.mark("rerank");
      if (!nf) continue;
      // the rows whose threshold did not bracket their band: single-pass list
      // mode on just those rows
      Dev P2((size_t)nf * c.Kp * 2, stream), qn2(4ull * nf, stream),
          q2((size_t)nf * qld * 4, stream), ids2(4ull * nf * K, stream), d2(4ull * nf * K, stream);
      gather_u16_rows_kernel<<<nf, 128, 0, stream>>>(Pq, c.Kp, fail_rows, nf, P2.as<uint16_t>());
      gather_f32_kernel<<<(nf + 255) / 256, 256, 0, stream>>>(qnorm, fail_rows, nf,
                                                              qn2.as<float>());
      gather_rows_kernel<<<nf, 128, 0, stream>>>(cqueries, qld, fail_rows, nf, q2.as<float>());
      CAGRA_LAUNCH_CHECK();
      // the retried rows' data ids (their self columns)
      Dev sid2(4ull * nf, stream);
      const uint32_t* self2 = nullptr;
      if (exclude_self) {
        offset_ids_kernel<<<(nf + 255) / 256, 256, 0, stream>>>(fail_rows, nf, cc.self_base,
                                                                sid2.as<uint32_t>());
        CAGRA_LAUNCH_CHECK();
        self2 = sid2.as<uint32_t>();
      }
      list_pass(cc, P2.p, nf, qn2.as<float>(), q2.as<float>(), qld, self2, ids2.as<uint32_t>(),
                d2.as<float>(), reranked, fallback);
      scatter_rows_kernel<<<nf, 128, 0, stream>>>(fail_rows, nf, K, ids2.as<uint32_t>(),
                                                  d2.as<float>(), cids, cdists);
      CAGRA_LAUNCH_CHECK();
      CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    }
  }
  tr.mark("retry/end");
  g_knn_tc_stats.rows = nq;
  g_knn_tc_stats.fallback_rows = fallback;
  g_knn_tc_stats.reranked = reranked;
  g_knn_tc_stats.retried_rows = retried;
  g_knn_tc_stats.split_terms = c.terms;
  g_knn_tc_stats.gemm_k = (c.kblocks - 1) * TC_BK + 16 * c.ksteps_last;
}

}  // namespace cagra
