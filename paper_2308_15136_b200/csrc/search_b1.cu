// Batch-1 shared mode (shared_query_search, engine.cpp:38-78) as one small CTA
// per team with every phase of an iteration fused, and the team merge
// (merge_team_results, engine.cpp:12-36) done by the query's last team CTA:
// ONE kernel launch per batch.
//
// Each team is a 128-thread CTA (4 warps); the T teams of a query share the
// query's visited set — a bitmap of hcap * 32 bits in L2 (reference sizing
// next_pow2(2 (I_max + 1) T d) slots, 32 bits each).  A candidate is a first
// visit when its bit is clear; the bit is then set with a fire-and-forget
// atomic OR, so no atomic round trip sits on the iteration's critical path.
// Within a team this is exact (the CTA barrier orders a team's marks before its
// next test); across the racing teams a node may be evaluated twice when two
// teams test it in the same iteration, and a hash collision (<~1% of the bits
// at the reference's sizing) skips a node — the lockstep reference order is
// not kept by any racing multi-CTA scheme anyway (±0.04 pp measured for claim
// order, SURVEY §8(c'); parity is checked on recall, tests and bench).
// The bitmap has two regions used by alternate calls: a call tests region
// (tag & 1) and clears region ((tag + 1) & 1) for the next call, so no memset
// precedes the kernel.  One iteration of a team:
//   * expansion: candidate c of the parent's graph row (or of the team's init
//     samples) is owned by an 8-lane group; every lane loads its id, lane
//     `sub` < 4 of each group the bitmap word of pass `sub`, then every lane
//     its V float4 of the 4 rows (all in flight together);
//   * distance: per-lane partial sums + 3 xor shuffles (fast mode; the final k
//     are re-scored with the sequential chain);
//   * survivors (first visit and key < the M-th key) are written to the
//     candidate's fixed shared slot (dummy otherwise; three slot sets rotate
//     over the iterations), no atomics;
//   * ONE barrier; then every warp merges the survivors into its own copy of
//     the team's sorted top-M (M <= 32, one entry per lane) by ranks: each
//     key's position = the number of keys before it, counted with pipelined
//     shuffle broadcasts, then one scatter through shared memory; every warp
//     selects the same next parent (first unflagged entry) and warp 0
//     prefetches the graph row of the entry after it into L2 (the likely
//     parent of the following iteration).
// The dependent chain per iteration is parent -> graph row -> data rows.
//
// Semantics per team follow Traversal (search.cpp:147-259) with p = 1, k = M,
// the standard policy and team seeds mix_seed(qseed + 0x7ea4 (t + 1))
// (engine.cpp:56): init samples with replacement (duplicates are sentinels),
// update_topm order (dist, stripped id), first-unflagged parent, I_max, the
// final flush.  The last team CTA of a query merges the teams' lists: only the
// first k entries of each (sorted, unique) team list can be in the global
// top-k, so it sorts T * k keys (one 256-key warp sort per quarter of the
// teams, then one 128-key sort), drops duplicate ids, re-scores the k winners
// with the sequential fp32 chain of squared_l2 and re-sorts — the reported
// distances are the reference's bits.
#include <cstdio>

#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int B1_THREADS = 128;

// 1: the visited test is an atomic claim (fetch-OR in flight with the row
// loads: exact across teams, no separate mark); 0: a plain L2 load of the
// bitmap word, then a fire-and-forget OR for first visits (racy across teams)
#ifndef CAGRA_B1_CLAIM
#define CAGRA_B1_CLAIM 1
#endif

// Phase profiler (tools/build_variant.sh b1prof -DCAGRA_B1_PROF search_b1):
// team 0, thread 0 accumulates cycles per phase; printed by the launcher.
#ifdef CAGRA_B1_PROF
__device__ unsigned long long g_b1_prof[8];
#define B1_T(v) const long long v = clock64()
#define B1_ADD(i, a, b) \
  do { if (item == 0 && tid == 0) g_b1_prof[i] += (unsigned long long)((b) - (a)); } while (0)
#else
#define B1_T(v)
#define B1_ADD(i, a, b) do { } while (0)
#endif
constexpr uint64_t kStrip = ~(1ull << 31);  // key without the parent flag

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
#if !CAGRA_B1_CLAIM
__device__ __forceinline__ uint32_t ldcg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
#endif
#if CAGRA_B1_CLAIM
// atomic OR returning the old word (the visited claim), issued like a load
__device__ __forceinline__ uint32_t atom_or_u32(uint32_t* p, uint32_t bit) {
  uint32_t v;
  asm volatile("atom.global.or.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "r"(bit) : "memory");
  return v;
}
#endif
__device__ __forceinline__ float4 ldg_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

struct B1Params {
  const float* data;
  const uint32_t* graph;
  const float* queries;
  uint32_t n, ld, dim, degree, T, M, k, max_iter, min_iter;
  uint64_t seed, query_offset;
  uint32_t seed_mode, hcap, tag;
  uint32_t direct;                 // bit = node id (hcap * 32 >= n), else hash_id
  uint32_t* tab;                   // [2][nq][hcap] u32 words of the visited bitmaps
  unsigned long long* team_out;    // [nq * T][M]
  void* team_stats;                // [nq * T] DevStats-compatible
  uint32_t* done_ctr;              // [nq] teams finished (reset by the merging CTA)
  uint32_t* out_ids;
  float* out_dists;
  uint32_t* out_counts;
  void* stats;                     // [nq] DevStats-compatible, may be null
};

struct B1Stats {
  uint32_t iterations, hash_resets;
  unsigned long long distance_evals;
  uint32_t converged, pad;
};

// unique keys (adjacent equal keys dropped) of a warp-sorted register array,
// compacted in order into dst[0, limit); returns the number of unique keys
template <int E>
__device__ __forceinline__ uint32_t compact_unique(const uint64_t (&v)[E], int lane,
                                                   uint64_t* dst, uint32_t limit) {
  uint64_t prev = __shfl_up_sync(0xffffffffu, v[E - 1], 1);
  if (lane == 0) prev = ~0ull;
  uint32_t keep = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool u = !key_is_dummy(v[e]) && v[e] != prev;
    keep |= (u ? 1u : 0u) << e;
    prev = v[e];
  }
  const uint32_t cnt = __popc(keep);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  uint32_t pos = incl - cnt;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if ((keep >> e) & 1u) {
      if (pos < limit) dst[pos] = v[e];
      ++pos;
    }
  return __shfl_sync(0xffffffffu, incl, 31);
}

// warp w: the first k entries of teams w, w + 4, ... (32 E keys at most) ->
// sort -> unique -> first k at dst (dummy padded)
template <int E>
__device__ __forceinline__ void b1_merge_quarter(const unsigned long long* lists, uint32_t T,
                                                 uint32_t M, uint32_t k, int warp, int lane,
                                                 uint64_t* dst) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e;
    const uint32_t tl = i / k, j = i - tl * k, team = warp + 4 * tl;
    v[e] = team < T ? cmp_key(__ldcg(lists + (size_t)team * M + j)) : kDummyKey;
  }
  warp_sort_regs<E>(v, lane);
  const uint32_t tot = compact_unique<E>(v, lane, dst, k);
  __syncwarp();
  for (uint32_t i = tot + lane; i < k; i += 32) dst[i] = kDummyKey;
}

// The query's final top-k from its T team lists (run by its last CTA).
__device__ void b1_merge(const B1Params& P, uint32_t q, uint64_t* sm) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t T = P.T, M = P.M, k = P.k;
  const unsigned long long* lists = P.team_out + (size_t)q * T * M;
  // 1) per warp: a quarter of the teams' first-k entries
  if (((T + 3) / 4) * k <= 256) b1_merge_quarter<8>(lists, T, M, k, warp, lane, sm + warp * 32);
  else b1_merge_quarter<16>(lists, T, M, k, warp, lane, sm + warp * 32);
  __syncthreads();
  if (warp != 0) return;
  // 2) the 4 warps' lists -> sort -> unique -> first k at sm[128 ...]
  uint64_t v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t i = lane * 4 + e, w = i / 32, j = i - w * 32;
    v[e] = j < k ? sm[w * 32 + j] : kDummyKey;
  }
  __syncwarp();
  warp_sort_regs<4>(v, lane);
  const uint32_t live = min(k, compact_unique<4>(v, lane, sm + 128, k));
  __syncwarp();
  // 3) sequential-chain re-score (dataset.hpp:33-43), one lane per winner,
  //    then (dist, id) order
  uint64_t one[1] = {kDummyKey};
  if ((uint32_t)lane < live) {
    const uint32_t id = key_id(sm[128 + lane]);
    const float* x = P.data + (size_t)id * P.ld;
    const float* qv = P.queries + (size_t)q * P.ld;
    float acc = 0.0f;
    for (uint32_t d = 0; d < P.dim; ++d) acc = seq_step(acc, __ldg(x + d), __ldg(qv + d));
    one[0] = make_key(acc, id);
  }
  warp_sort_regs<1>(one, lane);
  if ((uint32_t)lane < k) {
    const bool ok = (uint32_t)lane < live;
    P.out_ids[(size_t)q * k + lane] = ok ? key_id(one[0]) : kInvalidId;
    P.out_dists[(size_t)q * k + lane] = ok ? key_dist(one[0]) : __int_as_float(0x7f800000);
  }
  if (lane == 0) {
    P.out_counts[q] = live;
    if (P.stats) {
      const B1Stats* ts = reinterpret_cast<const B1Stats*>(P.team_stats) + (size_t)q * T;
      B1Stats st;
      unsigned long long ev = 0;
      uint32_t it = 0, cv = 1;
      for (uint32_t t = 0; t < T; ++t) {
        ev += __ldcg(&ts[t].distance_evals);
        it = max(it, __ldcg(&ts[t].iterations));
        cv = cv && __ldcg(&ts[t].converged);
      }
      st.iterations = it;
      st.hash_resets = 0;
      st.distance_evals = ev;
      st.converged = cv;
      st.pad = 0;
      reinterpret_cast<B1Stats*>(P.stats)[q] = st;
    }
  }
}

template <int V>
__global__ void __launch_bounds__(B1_THREADS, 1) team_b1_kernel(const B1Params P) {
  const uint32_t item = blockIdx.x, q = item / P.T, t = item - q * P.T;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, grp = lane >> 3, sub = lane & 7;
  __shared__ uint32_t s_ids[64];
  __shared__ uint64_t s_surv[3][64];   // candidate c of iteration i at [i % 3][c]
                                       // (its key if it survived, else a dummy)
  __shared__ uint64_t s_comp[4][64];   // per warp: the survivors, compacted
  __shared__ uint64_t s_tops[4][32];   // per warp: its top-M before the merge
  __shared__ uint64_t s_stage[4][32];  // per warp: the merged top-M
  __shared__ __align__(16) uint64_t s_state[160];  // init chain, then the merge's staging
  __shared__ uint32_t s_evals, s_last;
  const uint32_t deg = P.degree, nv4 = P.ld >> 2;
  const uint32_t bmask = P.hcap * 32u - 1u;  // visited bitmap: hcap words of 32 bits
  const size_t region = (size_t)(gridDim.x / P.T) * P.hcap;  // one call's tables (all queries)
  uint32_t* bits = P.tab + (P.tag & 1u) * region + (size_t)q * P.hcap;

  // the query slice of this lane (float4 sub + 8 v), zero beyond the row
  float4 qv[V];
  {
    const float4* Q = reinterpret_cast<const float4*>(P.queries + (size_t)q * P.ld);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t i = sub + 8 * v;
      qv[v] = i < nv4 ? __ldg(Q + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  {
    // clear this CTA's share of the OTHER region (the next call's tables)
    uint4* other = reinterpret_cast<uint4*>(P.tab + ((P.tag + 1) & 1u) * region);
    const size_t n16 = region / 4, per = (n16 + gridDim.x - 1) / gridDim.x;
    const size_t b = (size_t)blockIdx.x * per, e = min(n16, b + per);
    for (size_t i = b + tid; i < e; i += B1_THREADS) other[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) {
    // engine.cpp:108 (batch_search seed) / search.cpp:163 (search_one), team
    // seed engine.cpp:56, init samples search.cpp:192-201
    const uint64_t qseed =
        P.seed_mode == 0 ? mix_seed(P.seed ^ (0x0badull + P.query_offset + q)) : P.seed;
    const uint64_t tseed = mix_seed(qseed + 0x7ea4ull * (t + 1));
    uint64_t state = mix_seed(tseed ^ 0x5eedull);
    for (uint32_t c = 0; c < deg; ++c) {  // the chain is sequential; the modulo is not
      state = mix_seed(state);
      s_state[c] = state;
    }
    s_evals = 0;
  }
  __syncthreads();
  if ((uint32_t)tid < deg) s_ids[tid] = (uint32_t)(s_state[tid] % P.n);
  __syncthreads();
  // a repeated init sample is a sentinel (search.cpp:192-201: the visited
  // insert of the later copy fails)
  if ((uint32_t)tid < deg) {
    const uint32_t id = s_ids[tid];
    bool dup = false;
    for (uint32_t j = 0; j < (uint32_t)tid; ++j) dup |= s_ids[j] == id;
    s_surv[2][tid] = dup ? 1u : 0u;  // applied after every thread has read s_ids
  }
  __syncthreads();
  if ((uint32_t)tid < deg && s_surv[2][tid]) s_ids[tid] = kInvalidId;
  __syncthreads();

  // Every warp keeps its own copy of the team's top-M (entry `lane`) and runs
  // the same update_topm / select_parents on the shared survivors, so one
  // barrier per iteration suffices.  (A team never evaluates an id twice —
  // its own marks are ordered by that barrier and the init samples are
  // de-duplicated — so survivors never duplicate a top-M entry.)
  uint64_t top = kDummyKey, mth = kDummyKey;
  uint32_t iter = 0, parent = 0, slot = 0, evals = 0;
  bool from_graph = false, finish = false, converged = false;
  for (;;) {
    B1_T(p0);
    // ---------------- expansion: 16 candidates per warp, 4 per pass
    // (loads are asm volatile so the compiler issues all of them before any
    // use: left alone it recycled registers and serialised the 4 passes into
    // 4 dependent memory round trips)
    uint32_t cid[4];
    if (from_graph) {
      const uint32_t* row = P.graph + (size_t)parent * deg;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        cid[j] = ldg_u32(row + min((uint32_t)(warp * 16 + j * 4 + grp), deg - 1));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) cid[j] = s_ids[min((uint32_t)(warp * 16 + j * 4 + grp), deg - 1)];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((uint32_t)(warp * 16 + j * 4 + grp) >= deg) cid[j] = kInvalidId;
    // visited test: lane `sub` < 4 of each group reads the bitmap word of the
    // group's candidate of pass `sub` (an L2 load issued with the row loads)
    const uint32_t my_id =
        sub == 0 ? cid[0]
                 : (sub == 1 ? cid[1] : (sub == 2 ? cid[2] : (sub == 3 ? cid[3] : kInvalidId)));
    const uint32_t bi = my_id == kInvalidId ? 0u : (P.direct ? my_id : hash_id(my_id, bmask));
    B1_T(p1);
#if CAGRA_B1_CLAIM
    // claim: atomic OR returning the old word, in flight with the row loads;
    // exactly one team wins a node
    const uint32_t word = my_id != kInvalidId ? atom_or_u32(bits + (bi >> 5), 1u << (bi & 31)) : ~0u;
#else
    const uint32_t word = ldcg_u32(bits + (bi >> 5));
#endif
    float4 xv[4][V];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4* X = reinterpret_cast<const float4*>(
          P.data + (size_t)(cid[j] == kInvalidId ? 0u : cid[j]) * P.ld);
#pragma unroll
      for (int v = 0; v < V; ++v) xv[j][v] = ldg_f4(X + min((uint32_t)(sub + 8 * v), nv4 - 1));
    }
    // lanes past the row (V * 8 > ld / 4) or invalid candidates contribute 0
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (cid[j] == kInvalidId || (uint32_t)(sub + 8 * v) >= nv4) xv[j][v] = qv[v];
    float dist[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float acc = 0.0f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float a = xv[j][v].x - qv[v].x, b = xv[j][v].y - qv[v].y;
        const float c = xv[j][v].z - qv[v].z, d = xv[j][v].w - qv[v].w;
        acc = fmaf(a, a, acc);
        acc = fmaf(b, b, acc);
        acc = fmaf(c, c, acc);
        acc = fmaf(d, d, acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      dist[j] = acc;
    }
    B1_T(p2);
    // first visit = bit clear; mark it (fire-and-forget atomic OR, never
    // waited on: the barrier below orders it for this team's next tests)
    const bool mine_first = my_id != kInvalidId && !((word >> (bi & 31)) & 1u) && sub < 4;
#if !CAGRA_B1_CLAIM
    if (mine_first) atomicOr(bits + (bi >> 5), 1u << (bi & 31));
#endif
    const unsigned fb = __ballot_sync(0xffffffffu, mine_first);
    const uint32_t firstm = (fb >> (lane & ~7)) & 0xfu;
    // survivors: candidate c's fixed slot holds its key, or a dummy (the
    // evaluation count stays in registers until the end)
    uint32_t nev = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool first = (firstm >> j) & 1u;
      const uint64_t key = make_key(dist[j], cid[j]);
      if (sub == 0)
        s_surv[slot][warp * 16 + j * 4 + grp] = first && key < mth ? key : kDummyKey;
      nev += (sub == 0 && first) ? 1u : 0u;
    }
    evals += nev;
    B1_T(p3);
    __syncthreads();
    B1_T(p4);
    // ---------------- every warp: update_topm + select_parents
    // update_topm as a rank merge: every key's final position = the number of
    // top-M entries and survivors before it (distinct ids: distinct keys).
    // The survivors are compacted into shared memory, the counting loops read
    // them and the old top-M back with broadcast loads (independent, so they
    // pipeline), and one scatter through shared memory places every key.
    const uint64_t c0 = s_surv[slot][lane], c1 = s_surv[slot][lane + 32];
    const unsigned m0 = __ballot_sync(0xffffffffu, !key_is_dummy(c0));
    const unsigned m1 = __ballot_sync(0xffffffffu, !key_is_dummy(c1));
    const uint32_t n0 = __popc(m0), ns = n0 + __popc(m1);
    if (ns) {
      const unsigned below = (1u << lane) - 1u;
      uint64_t* cs = s_comp[warp];
      uint64_t* ts = s_tops[warp];
      uint64_t* st = s_stage[warp];
      if (!key_is_dummy(c0)) cs[__popc(m0 & below)] = c0;
      if (!key_is_dummy(c1)) cs[n0 + __popc(m1 & below)] = c1;
      ts[lane] = top;
      __syncwarp();
      const uint64_t s0 = (uint32_t)lane < ns ? cs[lane] : kDummyKey;
      const uint64_t s1 = (uint32_t)lane + 32 < ns ? cs[lane + 32] : kDummyKey;
      const uint64_t tk = top & kStrip, k0 = s0 & kStrip, k1 = s1 & kStrip;
      uint32_t tr = 0, r0 = 0, r1 = 0;
      uint32_t k = 0;
      for (; k + 4 <= ns; k += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t x = cs[k + u];  // survivors carry no flag
          tr += x < tk;
          r0 += x < k0;
          r1 += x < k1;
        }
      }
      for (; k < ns; ++k) {
        const uint64_t x = cs[k];
        tr += x < tk;
        r0 += x < k0;
        r1 += x < k1;
      }
#pragma unroll 8
      for (uint32_t j = 0; j < P.M; ++j) {
        const uint64_t x = ts[j] & kStrip;
        r0 += x < k0;
        r1 += x < k1;
      }
      if ((uint32_t)lane < P.M && lane + tr < P.M) st[lane + tr] = top;
      if ((uint32_t)lane < ns && r0 < P.M) st[r0] = s0;
      if ((uint32_t)lane + 32 < ns && r1 < P.M) st[r1] = s1;
      __syncwarp();
      top = (uint32_t)lane < P.M ? st[lane] : kDummyKey;
      __syncwarp();
    }
    B1_ADD(5, 0, ns);   // survivors
    if ((uint32_t)lane >= P.M) top = kDummyKey;
    bool done = finish;
    if (!done) {
      ++iter;  // search.cpp:225
      const bool cand = (uint32_t)lane < P.M && !key_is_dummy(top) &&
                        !(static_cast<uint32_t>(top) & kParentFlag);
      const unsigned b = __ballot_sync(0xffffffffu, cand);
      if (!b) {  // no parent: converged (search.cpp:225-231)
        done = true;
        converged = iter >= P.min_iter;
      } else {
        const int pl = __ffs(b) - 1;
        parent = __shfl_sync(0xffffffffu, static_cast<uint32_t>(top), pl);
        if (lane == pl) top |= kParentFlag;
        finish = iter >= P.max_iter;  // the expansion below is flushed, then stop
        // the next two unflagged entries are the likely parents after this
        // one: pull their graph rows into L2 while this expansion runs
        unsigned b2 = b & ~(1u << pl);
        const unsigned b3 = b2 ? b2 & (b2 - 1) : 0u;
        b2 = b2 & ~b3;  // lowest remaining bit
        const unsigned pre = b2 | (b3 & (0u - b3));
        if (warp == 0 && ((pre >> lane) & 1u)) {
          const uint32_t* row = P.graph + (size_t)static_cast<uint32_t>(top) * deg;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
          if (deg * 4 > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + 32));
        }
      }
    }
    B1_T(p5);
    B1_ADD(0, p0, p1);  // graph-row ids
    B1_ADD(1, p1, p2);  // bitmap word + data rows + distances
    B1_ADD(2, p2, p3);  // first-visit marks + survivor appends
    B1_ADD(3, p3, p4);  // barrier
    B1_ADD(4, p4, p5);  // update_topm + select_parents
    B1_ADD(6, 0, 1);    // iterations
    if (done) break;
    const uint64_t m = __shfl_sync(0xffffffffu, top, P.M - 1) & kStrip;
    mth = key_is_dummy(m) ? kDummyKey : m;
    from_graph = true;
    slot = (slot + 1) % 3;
  }
  evals += __shfl_xor_sync(0xffffffffu, evals, 16);
  evals += __shfl_xor_sync(0xffffffffu, evals, 8);
  if (lane == 0 && evals) atomicAdd(&s_evals, evals);
  __syncthreads();
  if (warp == 0) {
    if ((uint32_t)lane < P.M) P.team_out[(size_t)item * P.M + lane] = top;
    if (lane == 0) {
      B1Stats st;
      st.iterations = iter;
      st.hash_resets = 0;
      st.distance_evals = s_evals;
      st.converged = converged ? 1u : 0u;
      st.pad = 0;
      reinterpret_cast<B1Stats*>(P.team_stats)[item] = st;
    }
    // last team of the query merges (the threadFenceReduction pattern)
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      const uint32_t prev = atomicAdd(&P.done_ctr[q], 1u);
      s_last = prev == P.T - 1 ? 1u : 0u;
      if (s_last) P.done_ctr[q] = 0;  // ready for the next call
    }
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    b1_merge(P, q, s_state);
  }
}

}  // namespace

bool team_b1_eligible(uint32_t M, uint32_t k, uint32_t T, uint32_t degree, uint32_t ld) {
  // the fused merge: each warp's share of the teams' first-k entries fits one
  // 512-key warp sort, and the 4 warps' first-k lists one 128-key sort
  const uint32_t share = ((T + 3) / 4) * k;
  return M >= 1 && M <= 32 && k <= 32 && share <= 512 && degree >= 1 && degree <= 64 &&
         ld <= 128;
}

void launch_team_b1(const float* data, const uint32_t* graph, uint32_t n, uint32_t ld,
                    uint32_t dim, uint32_t degree, const float* queries, uint32_t nq, uint32_t T,
                    uint32_t M, uint32_t k, uint32_t max_iter, uint32_t min_iter, uint64_t seed,
                    uint64_t query_offset, uint32_t seed_mode, uint32_t* tab, uint32_t hcap,
                    uint32_t tag, uint32_t direct, unsigned long long* team_out, void* team_stats,
                    uint32_t* done_ctr, uint32_t* out_ids, float* out_dists,
                    uint32_t* out_counts, void* stats, cudaStream_t stream) {
  B1Params P;
  P.data = data;
  P.graph = graph;
  P.queries = queries;
  P.n = n;
  P.ld = ld;
  P.dim = dim;
  P.degree = degree;
  P.T = T;
  P.M = M;
  P.k = k;
  P.max_iter = max_iter;
  P.min_iter = min_iter;
  P.seed = seed;
  P.query_offset = query_offset;
  P.seed_mode = seed_mode;
  P.hcap = hcap;
  P.tag = tag;
  P.direct = direct;
  P.tab = tab;
  P.team_out = team_out;
  P.team_stats = team_stats;
  P.done_ctr = done_ctr;
  P.out_ids = out_ids;
  P.out_dists = out_dists;
  P.out_counts = out_counts;
  P.stats = stats;
  const uint32_t v = (ld / 4 + 7) / 8;
  const dim3 grid(nq * T);
#ifdef CAGRA_B1_PROF
  unsigned long long zero[8] = {};
  CAGRA_CUDA_TRY(cudaMemcpyToSymbolAsync(g_b1_prof, zero, sizeof(zero), 0,
                                         cudaMemcpyHostToDevice, stream));
#endif
  switch (v) {
    case 1: team_b1_kernel<1><<<grid, B1_THREADS, 0, stream>>>(P); break;
    case 2: team_b1_kernel<2><<<grid, B1_THREADS, 0, stream>>>(P); break;
    case 3: team_b1_kernel<3><<<grid, B1_THREADS, 0, stream>>>(P); break;
    default: team_b1_kernel<4><<<grid, B1_THREADS, 0, stream>>>(P); break;
  }
  CAGRA_LAUNCH_CHECK();
#ifdef CAGRA_B1_PROF
  unsigned long long h[8];
  CAGRA_CUDA_TRY(cudaMemcpyFromSymbolAsync(h, g_b1_prof, sizeof(h), 0, cudaMemcpyDeviceToHost,
                                           stream));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
  const double it = h[6] ? (double)h[6] : 1.0;
  fprintf(stderr, "b1 prof per iteration (cycles, team 0 thread 0, %llu iterations): ids %.0f "
                  "rows+dist %.0f marks %.0f barrier %.0f merge+select %.0f | survivors %.1f\n",
          h[6], h[0] / it, h[1] / it, h[2] / it, h[3] / it, h[4] / it, h[5] / it);
#endif
}

}  // namespace cagra
