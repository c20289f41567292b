// Batch beam search on device — the north-star hot path.
//
//   search_one / Traversal (search.cpp:147-268) and batch_search
//   (engine.cpp:95-120), per-query mode: ONE CTA PER QUERY (persistent CTAs
//   pull queries from an atomic counter).
//   shared_query_search (engine.cpp:38-78): T lockstep teams inside one CTA
//   sharing one visited table, reproducing the reference's team order.
//
// Per query, shared memory holds the query, the sorted top-M list (double
// buffered), the candidate "survivors" of the last expansion and, for the
// forgettable policy, the open-addressing visited table.  The standard
// policy's visited set lives in a generation-tagged table in HBM (one region
// per resident CTA, never cleared: a bumped tag empties it).
//
// Reference semantics reproduced exactly (ids, distances, counters):
//   * buffer order (dist, stripped id) with flag-OR dedup — entries are 64-bit
//     keys (dist bits << 32 | id), see common.cuh;
//   * update_topm (search.cpp:55-85) == merge of the previous expansion's
//     candidates into top-M.  Candidates that cannot enter top-M (key >= the
//     M-th key) are dropped at expansion time ("survivors" only), duplicates
//     of top-M entries are dropped (equivalent to the flag-OR collapse, the
//     top-M copy already carries the flag);
//   * select_parents (search.cpp:87-98): first p unflagged non-dummy entries;
//   * visited semantics, including forgettable "Full" early resets in exact
//     reference order (serial slow path when an expansion could fill the table);
//   * init samples: state = mix_seed(qseed ^ 0x5eed), id = mix_seed-chain % N
//     (search.cpp:163, 192-201), precomputed by init_samples_kernel;
//   * termination / convergence / I_max (search.cpp:218-245) and finish
//     (:247-259).
// Distances: EXACT=true uses the sequential fp32 chain of squared_l2 per
// candidate (bit-equal to the CPU).  EXACT=false ("fast") splits a row over a
// team of lanes with 128-bit loads and a shuffle reduction; the final k are
// re-scored with the sequential chain and re-sorted, so reported distances are
// always bit-equal to the reference's.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int SNT = 256;  // threads per search CTA
#ifdef CAGRA_DEBUG
#define DBG(...) do { if (blockIdx.x == 0 && threadIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define DBG(...) do { } while (0)
#endif
constexpr int SWARPS = SNT / 32;

struct DevStats {
  uint32_t iterations, hash_resets;
  unsigned long long distance_evals;
  uint32_t converged, pad;
};

struct KParams {
  const float* data;
  const uint32_t* graph;
  uint32_t n, dim, ld, degree;
  uint32_t deg_shift;  // log2(degree) when a power of two, else 0xff
  const float* queries;
  uint32_t nq;
  uint32_t k, M, p, C, max_iter, min_iter, policy, reset_interval;
  uint32_t hcap;  // visited capacity (power of two)
  uint32_t teams;  // shared mode team count (1 for per-query)
  const uint32_t* init_ids;  // [nq][teams*C]; null: generated in-kernel (small C)
  uint64_t seed, query_offset;
  uint32_t seed_mode;
  unsigned long long* gtables;  // [grid][hcap] when the table is global
  // standard policy, per-query mode: an exact visited BITMAP indexed by node
  // id, bm_words u32 per resident CTA (cleared per query), instead of the
  // hashed table — one L2 atomicOr per candidate, no probing, never full
  uint32_t* bitmaps;
  uint32_t bm_words;
  uint32_t* gens;               // [grid]
  uint32_t* work;               // query counter
  uint32_t* out_ids;
  float* out_dists;
  uint32_t* out_counts;
  DevStats* stats;
  int* error;
  unsigned long long* prof;  // optional phase cycle counters (CAGRA_SEARCH_PROF)
  // multi-CTA shared mode: work item qi = query * mc_teams + team; the teams
  // of a query share the HBM visited region of the query (generation mc_tag)
  uint32_t mc_teams, mc_tag;
  // per-query kernel: update_topm in place (one top-M buffer, the plan's
  // default; the double-buffered merge stays for CAGRA_SEARCH_INPLACE=0)
  uint32_t inplace;
  uint32_t* mc_tab;  // [nq][hcap] u32, kInvalidId = empty, cleared per call
  unsigned long long* team_out;  // [nq * teams][M] team top-M keys
  DevStats* team_stats;          // [nq * teams]
};

// Phase profiler: compiled in only with -DCAGRA_PROF_BUILD (tools/build_variant.sh),
// then enabled at run time by CAGRA_SEARCH_PROF=1.  The production build has
// no timestamps live across phases (64-register budget of the search kernel).
#ifdef CAGRA_PROF_BUILD
#define PROF_T(var) long long var = (P.prof && threadIdx.x == 0) ? clock64() : 0
#define PROF_ADD(slot, since) \
  do { if (P.prof && threadIdx.x == 0) atomicAdd(&P.prof[slot], (unsigned long long)(clock64() - since)); } while (0)
#define PROF_CNT(slot, v) \
  do { if (P.prof && threadIdx.x == 0) atomicAdd(&P.prof[slot], (unsigned long long)(v)); } while (0)
#else
#define PROF_T(var)
#define PROF_ADD(slot, since) do { } while (0)
#define PROF_CNT(slot, v) do { } while (0)
#endif

// ------------------------------------------------------------- init ids ----
__global__ void init_samples_kernel(uint32_t nq, uint32_t C, uint32_t teams, uint32_t n,
                                    uint64_t seed, uint32_t seed_mode, uint64_t qoff,
                                    uint32_t* __restrict__ out) {
  uint32_t qi = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t t = blockIdx.y;
  if (qi >= nq) return;
  // engine.cpp:108 / search.cpp:163 / engine.cpp:56
  uint64_t qseed = seed_mode == 0 ? mix_seed(seed ^ (0x0badull + qoff + qi)) : seed;
  uint64_t tseed = teams > 1 ? mix_seed(qseed + 0x7ea4ull * (t + 1)) : qseed;
  uint64_t state = mix_seed(tseed ^ 0x5eedull);
  uint32_t* o = out + ((size_t)qi * teams + t) * C;
  for (uint32_t j = 0; j < C; ++j) {
    state = mix_seed(state);
    o[j] = (uint32_t)(state % n);
  }
}

// ------------------------------------------------------------ sorting ------
template <int E>
__device__ __forceinline__ void warp_sort_smem_E(uint64_t* a, uint32_t cnt, int lane) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t i = lane * E + e;
    v[e] = i < cnt ? a[i] : kDummyKey;
  }
  warp_sort_regs<E>(v, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t i = lane * E + e;
    if (i < cnt) a[i] = v[e];
  }
}

// Sort a[0..cnt) ascending using one warp (cnt <= 256).
__device__ __noinline__ void warp_sort_smem(uint64_t* a, uint32_t cnt, int lane) {
  if (cnt <= 1) return;
  if (cnt <= 32) warp_sort_smem_E<1>(a, cnt, lane);
  else if (cnt <= 64) warp_sort_smem_E<2>(a, cnt, lane);
  else if (cnt <= 128) warp_sort_smem_E<4>(a, cnt, lane);
  else warp_sort_smem_E<8>(a, cnt, lane);
  __syncwarp();
}

// Block-wide bitonic sort of a[0..P), P power of two (caller syncs before).
__device__ void block_sort_smem(uint64_t* a, uint32_t P) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
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
      __syncthreads();
    }
  }
}

// Block-wide bitonic sort of a[0..EPT*SNT) held EPT keys per thread in
// registers (index = tid*EPT + e): intra-thread and intra-warp stages need no
// barrier; only partner distances >= 32*EPT go through shared memory (6
// barrier pairs for 1024 keys instead of 55 barriers).  a is used as the
// exchange buffer and holds the sorted keys on return (caller syncs before).
template <int EPT>
__device__ void block_sort_regs(uint64_t* a) {
  constexpr uint32_t P = EPT * SNT;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  uint64_t v[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) v[e] = a[tid * EPT + e];
#pragma unroll
  for (uint32_t k = 2; k <= P; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j < (uint32_t)EPT) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if ((e & j) == 0) {
            const uint32_t i = tid * EPT + e;
            const bool up = (i & k) == 0;
            uint64_t x = v[e], y = v[e ^ j];
            if ((x > y) == up) {
              v[e] = y;
              v[e ^ j] = x;
            }
          }
        }
      } else if (j < 32u * EPT) {
        const uint32_t lm = j / EPT;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const uint32_t i = tid * EPT + e;
          const bool up = (i & k) == 0, lower = (lane & lm) == 0;
          uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], lm);
          uint64_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == up) ? mn : mx;
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EPT; ++e) a[tid * EPT + e] = v[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const uint32_t i = tid * EPT + e;
          const bool up = (i & k) == 0, lower = (i & j) == 0;
          uint64_t o = a[i ^ j];
          uint64_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < EPT; ++e) a[tid * EPT + e] = v[e];
}

// a[0..P) for P a power of two in [256, 2048] via the register sort, else the
// smem network.
__device__ __noinline__ void block_sort_any(uint64_t* a, uint32_t P) {
  if (P == 256) block_sort_regs<1>(a);
  else if (P == 512) block_sort_regs<2>(a);
  else if (P == 1024) block_sort_regs<4>(a);
  else if (P == 2048) block_sort_regs<8>(a);
  else if (P == 4096) block_sort_regs<16>(a);
  else block_sort_smem(a, P);
}

// #{i < len : cmp_key(a[i]) < key}   (a sorted by cmp_key)
__device__ __forceinline__ uint32_t lb_cmp(const uint64_t* a, uint32_t len, uint64_t key) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (cmp_key(a[mid]) < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Warp-aggregated append: every lane with `pred` gets a distinct slot of the
// shared counter `*ctr` (one atomic per warp instead of one per element).
// Must be called by all 32 lanes of the warp.
__device__ __forceinline__ uint32_t warp_append_slot(uint32_t* ctr, bool pred) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return 0;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(ctr, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

// ------------------------------------------------------------ visited -----
// Shared-memory table: u32 slots, kInvalidId = empty.
__device__ __forceinline__ bool smem_insert_from(uint32_t* tab, uint32_t mask, uint32_t id,
                                                 uint32_t h) {
  for (;;) {
    uint32_t old = atomicCAS(&tab[h], kInvalidId, id);
    if (old == kInvalidId) return true;
    if (old == id) return false;
    h = (h + 1) & mask;
  }
}
__device__ __forceinline__ bool smem_insert(uint32_t* tab, uint32_t mask, uint32_t id) {
  uint32_t h = hash_id(id, mask);
  for (;;) {
    uint32_t old = atomicCAS(&tab[h], kInvalidId, id);
    if (old == kInvalidId) return true;
    if (old == id) return false;
    h = (h + 1) & mask;
  }
}

// HBM table: u64 slots (tag << 32 | id); a slot whose tag differs from the
// current generation is empty.
__device__ __forceinline__ bool gtab_insert(unsigned long long* tab, uint32_t mask, uint32_t tag,
                                            uint32_t id) {
  const unsigned long long want = ((unsigned long long)tag << 32) | id;
  uint32_t h = hash_id(id, mask);
  unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(&tab[h]);
  for (;;) {
    if ((uint32_t)(cur >> 32) != tag) {
      unsigned long long old = atomicCAS(&tab[h], cur, want);
      if (old == cur) return true;
      cur = old;  // re-examine the same slot
      continue;
    }
    if ((uint32_t)cur == id) return false;
    h = (h + 1) & mask;
    cur = *reinterpret_cast<volatile unsigned long long*>(&tab[h]);
  }
}

// ------------------------------------------------------------ distances ----
__device__ __forceinline__ float exact_dist(const float* __restrict__ row, const float* q,
                                            uint32_t dim) {
  float acc = 0.0f;
  uint32_t i = 0;
  for (; i + 4 <= dim; i += 4) {
    float4 x = __ldg(reinterpret_cast<const float4*>(row + i));
    acc = seq_step(acc, x.x, q[i]);
    acc = seq_step(acc, x.y, q[i + 1]);
    acc = seq_step(acc, x.z, q[i + 2]);
    acc = seq_step(acc, x.w, q[i + 3]);
  }
  for (; i < dim; ++i) acc = seq_step(acc, __ldg(row + i), q[i]);
  return acc;
}

// ------------------------------------------------------------- the CTA -----
// All per-query state of the CTA, carved from dynamic shared memory.
struct Smem {
  float* q;            // ld
  uint64_t* topA;      // teams * M
  uint64_t* topB;      // teams * M
  uint64_t* surv;      // teams * SP
  uint32_t* evlist;    // teams * C   (ids to evaluate)
  uint16_t* evteam;    // teams * C   (owning team of each evlist entry)
  uint32_t* parents;   // teams * p
  uint32_t* table;     // hcap (smem table only)
  uint32_t* rclaim;    // shared mode: round first-occurrence hash (RP ids + RP orders)
  uint32_t* cand;      // shared mode: the round's candidates in reference order
  uint64_t* fin;       // shared mode: merged team results
};

constexpr int kSelChunks = 8;  // select_parents chunks per barrier round


struct Ctl {
  uint32_t qi, nev, npar_total, count, dup, slow, nfresh;
  uint32_t nsurv[16];
  uint32_t npar[16];
  uint32_t warp_cnt[kSelChunks * SWARPS];
  uint64_t worst[16];
  uint32_t iters[16];
  uint32_t done[16];
  uint32_t conv[16];
  unsigned long long evals[16];
  uint32_t resets;
  uint32_t pending[16];
};

// SPEC (multi-CTA mode): the candidates were not filtered by the visited
// table; the team leader issues the table insert right after the row loads,
// so the atomic's L2 round trip overlaps the row gather, and only first
// visits are kept and counted (ctl.nfresh).
template <int TEAM, int MAXC, bool EXACT, bool SPEC = false>
__device__ __forceinline__ void eval_list(const KParams& P, const Smem& S, Ctl& ctl,
                                          uint32_t nev, uint32_t SP,
                                          uint32_t* spec_tab = nullptr, uint32_t spec_mask = 0) {
  const int tid = threadIdx.x;
  if (EXACT) {
    for (uint32_t e0 = 0; e0 < nev; e0 += SNT) {
      const uint32_t e = e0 + tid;
      uint64_t key = kDummyKey;
      uint32_t t = 0;
      if (e < nev) {
        uint32_t id = S.evlist[e];
        t = P.teams == 1 ? 0u : S.evteam[e];
        float dist = exact_dist(P.data + (size_t)id * P.ld, S.q, P.dim);
        key = make_key(dist, id);
      }
      const bool keep = e < nev && key < ctl.worst[t];
      if (P.teams == 1) {
        const uint32_t pos = warp_append_slot(&ctl.nsurv[0], keep);
        if (keep) S.surv[pos] = key;
      } else if (keep) {
        uint32_t pos = atomicAdd(&ctl.nsurv[t], 1u);
        S.surv[t * SP + pos] = key;
      }
    }
  } else {
    constexpr int NTEAMS = SNT / TEAM;
    const int team = tid / TEAM, lt = tid % TEAM;
    const uint32_t nchunk = P.ld >> 2;
    float4 qr[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      uint32_t ch = lt + TEAM * c;
      qr[c] = ch < nchunk ? reinterpret_cast<const float4*>(S.q)[ch] : make_float4(0, 0, 0, 0);
    }
    // rows in flight per team (register budget ~9-12 float4 per lane)
#ifndef CAGRA_EVAL_U3
#define CAGRA_EVAL_U3 3
#endif
    constexpr int U = MAXC <= 2 ? 4 : (MAXC == 3 ? CAGRA_EVAL_U3 : 2);
#ifndef CAGRA_EVAL_ROLL
#define CAGRA_EVAL_ROLL 1
#endif
    if (CAGRA_EVAL_ROLL && !SPEC && MAXC == 3 && P.teams == 1) {
      // rolling pipeline (the 96-d variant): slot u's next row is requested as
      // soon as slot u's distance is done, so UR rows stay in flight per team
      // through the whole list instead of draining at the end of every batch.
      // Same per-row arithmetic as the batch loop below (bit-equal keys);
      // measured +1.3% over the 3-row batch loop (profiles/r02_eval_roll_ab.txt)
      constexpr int UR = 2;
      float4 xv[UR][MAXC];
      auto load = [&](int u, uint32_t e) {
        const uint32_t id = e < nev ? S.evlist[e] : 0;
        const float4* row = reinterpret_cast<const float4*>(P.data + (size_t)id * P.ld);
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          const uint32_t ch = lt + TEAM * c;
          xv[u][c] = (e < nev && ch < nchunk) ? __ldg(row + ch) : make_float4(0, 0, 0, 0);
        }
      };
#pragma unroll
      for (int u = 0; u < UR; ++u) load(u, team + u * NTEAMS);
      for (uint32_t base = 0; base < nev; base += NTEAMS * UR) {
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const uint32_t e = base + team + u * NTEAMS;
          float acc = 0.0f;
#pragma unroll
          for (int c = 0; c < MAXC; ++c) {
            const float4 qc = qr[c];
            float dx = xv[u][c].x - qc.x, dy = xv[u][c].y - qc.y;
            float dz = xv[u][c].z - qc.z, dw = xv[u][c].w - qc.w;
            acc = fmaf(dx, dx, acc);
            acc = fmaf(dy, dy, acc);
            acc = fmaf(dz, dz, acc);
            acc = fmaf(dw, dw, acc);
          }
          load(u, e + NTEAMS * UR);  // this slot's row of the next batch
#pragma unroll
          for (int o = TEAM / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, TEAM);
          uint64_t key = kDummyKey;
          bool keep = false;
          if (lt == 0 && e < nev) {
            key = make_key(acc, S.evlist[e]);
            keep = key < ctl.worst[0];
          }
          const uint32_t pos = warp_append_slot(&ctl.nsurv[0], keep);
          if (keep) S.surv[pos] = key;
        }
      }
      return;
    }
    // warp-uniform trip count: every lane runs every iteration (the team
    // shuffles below use the full mask)
    for (uint32_t base = 0; base < nev; base += NTEAMS * U) {
      const uint32_t e0 = base + team;
      float4 xv[U][MAXC];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t e = e0 + u * NTEAMS;
        uint32_t id = e < nev ? S.evlist[e] : 0;
        const float4* row = reinterpret_cast<const float4*>(P.data + (size_t)id * P.ld);
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          uint32_t ch = lt + TEAM * c;
          xv[u][c] = (e < nev && ch < nchunk) ? __ldg(row + ch) : make_float4(0, 0, 0, 0);
        }
      }
      uint32_t fresh = 0;  // SPEC: bit u = first visit of candidate u
      if (SPEC && lt == 0) {
        uint32_t old[U], h[U], ids[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // first probes of all U inserts in flight together
          uint32_t e = e0 + u * NTEAMS;
          ids[u] = e < nev ? S.evlist[e] : kInvalidId;
          h[u] = hash_id(ids[u], spec_mask);
          old[u] = e < nev ? atomicCAS(&spec_tab[h[u]], kInvalidId, ids[u]) : ids[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bool ins = old[u] == kInvalidId;
          if (!ins && old[u] != ids[u])  // collision: continue the linear probe
            ins = smem_insert_from(spec_tab, spec_mask, ids[u], (h[u] + 1) & spec_mask);
          fresh |= (ins ? 1u : 0u) << u;
        }
        const uint32_t nf = __popc(fresh);
        if (nf) atomicAdd(&ctl.nfresh, nf);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          float dx = xv[u][c].x - qr[c].x, dy = xv[u][c].y - qr[c].y;
          float dz = xv[u][c].z - qr[c].z, dw = xv[u][c].w - qr[c].w;
          acc = fmaf(dx, dx, acc);
          acc = fmaf(dy, dy, acc);
          acc = fmaf(dz, dz, acc);
          acc = fmaf(dw, dw, acc);
        }
#pragma unroll
        for (int o = TEAM / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, TEAM);
        uint32_t e = e0 + u * NTEAMS;
        uint64_t key = kDummyKey;
        uint32_t t = 0;
        bool keep = false;
        if (lt == 0 && e < nev) {
          uint32_t id = S.evlist[e];
          t = P.teams == 1 ? 0u : S.evteam[e];
          key = make_key(acc, id);
          keep = key < ctl.worst[t] && (!SPEC || ((fresh >> u) & 1u));
        }
        if (P.teams == 1) {
          const uint32_t pos = warp_append_slot(&ctl.nsurv[0], keep);
          if (keep) S.surv[pos] = key;
        } else if (keep) {
          uint32_t pos = atomicAdd(&ctl.nsurv[t], 1u);
          S.surv[t * SP + pos] = key;
        }
      }
    }
  }
}

// Generic (any dimension) fast path: query read from shared memory.
template <bool EXACT>
__device__ __forceinline__ void eval_list_generic(const KParams& P, const Smem& S, Ctl& ctl,
                                                  uint32_t nev, uint32_t SP) {
  if (EXACT) {
    eval_list<32, 1, true>(P, S, ctl, nev, SP);
    return;
  }
  const int tid = threadIdx.x, team = tid / 32, lt = tid % 32;
  const uint32_t nchunk = P.ld >> 2;
  for (uint32_t e = team; e < nev; e += SWARPS) {
    uint32_t id = S.evlist[e];
    const float4* row = reinterpret_cast<const float4*>(P.data + (size_t)id * P.ld);
    float acc = 0.0f;
    for (uint32_t ch = lt; ch < nchunk; ch += 32) {
      float4 x = __ldg(row + ch), q = reinterpret_cast<const float4*>(S.q)[ch];
      float dx = x.x - q.x, dy = x.y - q.y, dz = x.z - q.z, dw = x.w - q.w;
      acc = fmaf(dx, dx, acc);
      acc = fmaf(dy, dy, acc);
      acc = fmaf(dz, dz, acc);
      acc = fmaf(dw, dw, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lt == 0) {
      uint32_t t = P.teams == 1 ? 0u : S.evteam[e];
      uint64_t key = make_key(acc, id);
      if (key < ctl.worst[t]) {
        uint32_t pos = atomicAdd(&ctl.nsurv[t], 1u);
        S.surv[t * SP + pos] = key;
      }
    }
  }
}

// Clear of the shared-memory visited table: 16-byte stores (the table is
// 16-byte aligned and hcap is a power of two >= 4 whenever it lives in smem).
__device__ __forceinline__ void smem_table_clear(uint32_t* t, uint32_t hcap) {
  const uint4 inv = make_uint4(kInvalidId, kInvalidId, kInvalidId, kInvalidId);
  uint4* t4 = reinterpret_cast<uint4*>(t);
  for (uint32_t i = threadIdx.x; i < (hcap >> 2); i += SNT) t4[i] = inv;
  if (hcap < 4)
    for (uint32_t i = threadIdx.x; i < hcap; i += SNT) t[i] = kInvalidId;
}

// Visited-table reset with the current top-M ids (reset_table,
// search.cpp:138-145).  Called by all threads; top-M ids are distinct, so the
// parallel inserts fill exactly the first min(live, hcap) entries.
template <bool SMEM_TABLE>
__device__ void table_reset(const KParams& P, const Smem& S, Ctl& ctl, const uint64_t* top,
                            unsigned long long* gtab, uint32_t& tag) {
  if (SMEM_TABLE) {
    smem_table_clear(S.table, P.hcap);
  } else {
    tag = tag + 1;  // every thread keeps the same register copy
  }
  __syncthreads();
  uint32_t live = 0;
  {
    // dummies form the tail of the sorted list
    uint32_t lo = 0, hi = P.M;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (!key_is_dummy(top[mid])) lo = mid + 1;
      else hi = mid;
    }
    live = lo;
  }
  uint32_t lim = live < P.hcap ? live : P.hcap;
  for (uint32_t i = threadIdx.x; i < lim; i += SNT) {
    uint32_t id = key_id(top[i]) & kIdMask;
    if (SMEM_TABLE) smem_insert(S.table, P.hcap - 1, id);
    else gtab_insert(gtab, P.hcap - 1, tag, id);
  }
  if (threadIdx.x == 0) ctl.count = lim;
  __syncthreads();
}

// Serial (reference-order) visited processing of candidates when the
// forgettable table could fill mid-expansion (eval_or_skip, search.cpp:168-190).
template <bool SMEM_TABLE>
__device__ void serial_visit(const KParams& P, const Smem& S, Ctl& ctl, const uint32_t* ids,
                             uint32_t cnt, const uint64_t* top, unsigned long long* gtab,
                             uint32_t& tag) {
  // thread 0 only; tag is advanced in ctl via return (caller broadcasts)
  const uint32_t mask = P.hcap - 1;
  auto ins = [&](uint32_t id) -> int {  // 0 new, 1 present, 2 full
    if (ctl.count == P.hcap) return 2;
    uint32_t h = hash_id(id, mask);
    for (;;) {
      if (SMEM_TABLE) {
        uint32_t s = S.table[h];
        if (s == kInvalidId) {
          S.table[h] = id;
          break;
        }
        if (s == id) return 1;
      } else {
        unsigned long long s = gtab[h];
        if ((uint32_t)(s >> 32) != tag) {
          gtab[h] = ((unsigned long long)tag << 32) | id;
          break;
        }
        if ((uint32_t)s == id) return 1;
      }
      h = (h + 1) & mask;
    }
    ctl.count++;
    return 0;
  };
  auto reset = [&]() {
    if (SMEM_TABLE) {
      for (uint32_t i = 0; i < P.hcap; ++i) S.table[i] = kInvalidId;
    } else {
      tag = tag + 1;
    }
    ctl.count = 0;
    for (uint32_t i = 0; i < P.M; ++i) {
      if (key_is_dummy(top[i])) break;
      ins(key_id(top[i]) & kIdMask);
    }
  };
  uint32_t nev = 0;
  for (uint32_t j = 0; j < cnt; ++j) {
    uint32_t id = ids[j];
    int r = ins(id);
    if (r == 2) {
      reset();
      ctl.resets++;
      r = ins(id);
    }
    if (r == 0) {
      S.evlist[nev] = id;
      ++nev;
    }
  }
  ctl.nev = nev;
}

// ------------------------------------------------------ per-query kernel ---
#ifndef CAGRA_SEARCH_MINB
#define CAGRA_SEARCH_MINB 4  // 64 registers: 4 CTAs (1024 threads) per SM; the heuristic alone is unstable
#endif
// MC: multi-CTA instantiation (P.mc_teams > 0, shared HBM visited table):
// graph candidates go to eval unfiltered and are inserted there (SPEC above).
template <int TEAM, int MAXC, bool EXACT, bool SMEM_TABLE, bool MC = false>
__global__ void __launch_bounds__(SNT, CAGRA_SEARCH_MINB)
search_kernel(const KParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Ctl ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t SP = max(256u, next_pow2_u32(P.C));  // survivor buffer (block sort pads to 256)
  Smem S;
  {
    unsigned char* p = smem_raw;
    S.q = reinterpret_cast<float*>(p);
    p += sizeof(float) * round_up_u32(P.ld, 4);
    S.topA = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * P.M;
    S.topB = reinterpret_cast<uint64_t*>(p);
    if (!P.inplace) p += sizeof(uint64_t) * P.M;
    S.surv = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * SP;
    S.evlist = reinterpret_cast<uint32_t*>(p);
    p += sizeof(uint32_t) * round_up_u32(P.C, 4);  // keeps the table 16-byte aligned
    S.evteam = nullptr;  // one team: every candidate belongs to team 0
    if (P.inplace) S.topB = S.surv;  // scratch for the final re-score only
    S.parents = reinterpret_cast<uint32_t*>(p);
    p += sizeof(uint32_t) * round_up_u32(P.p, 4);
    S.table = reinterpret_cast<uint32_t*>(p);
  }
  unsigned long long* gtab = SMEM_TABLE ? nullptr : P.gtables + (size_t)blockIdx.x * P.hcap;
  uint32_t* const bm = P.bitmaps ? P.bitmaps + (size_t)blockIdx.x * P.bm_words : nullptr;
  // (tags only for the hashed HBM tables: the bitmap and smem tables are
  // cleared per query)
  uint32_t tag = SMEM_TABLE || bm ? 0 : P.gens[blockIdx.x];
  const uint32_t mask = P.hcap - 1;
  const bool forget = P.policy == 1;

  for (;;) {
    if (tid == 0) ctl.qi = atomicAdd(P.work, 1u);
    __syncthreads();
    const uint32_t qi = ctl.qi;
    if (qi >= P.nq) break;
    // ---- per-query setup
    const uint32_t qreal = P.mc_teams ? qi / P.mc_teams : qi;
    for (uint32_t i = tid; i < P.ld; i += SNT) S.q[i] = P.queries[(size_t)qreal * P.ld + i];
    for (uint32_t i = tid; i < P.M; i += SNT) S.topA[i] = kDummyKey;
    if (SMEM_TABLE) smem_table_clear(S.table, P.hcap);
    if (bm) {  // the previous query's marks (bm_words is a multiple of 4)
      uint4* b4 = reinterpret_cast<uint4*>(bm);
      for (uint32_t i = tid; i < (P.bm_words >> 2); i += SNT) b4[i] = make_uint4(0, 0, 0, 0);
    }
    if (!SMEM_TABLE && P.mc_teams) {
      gtab = P.gtables + (size_t)qreal * P.hcap;  // shared by the query's teams
      tag = P.mc_tag;
    } else {
      tag = tag + 1;
    }
    if (tid == 0) {
      ctl.nsurv[0] = 0;
      ctl.count = 0;
      ctl.resets = 0;
      ctl.evals[0] = 0;
      ctl.iters[0] = 0;
      ctl.conv[0] = 0;
      ctl.worst[0] = kDummyKey;
      ctl.dup = 0;
    }
    __syncthreads();

    uint64_t* top = S.topA;
    uint64_t* nxt = S.topB;
    const uint32_t* init;
    if (P.init_ids) {
      init = P.init_ids + (size_t)qi * P.C;
    } else {
      // init samples in-kernel (search.cpp:192-201 with the engine's seeds,
      // engine.cpp:56, 108): one sequential splitmix chain, C <= 256
      uint32_t* buf = reinterpret_cast<uint32_t*>(S.surv);
      if (tid == 0) {
        const uint64_t qseed =
            P.seed_mode == 0 ? mix_seed(P.seed ^ (0x0badull + P.query_offset + qreal)) : P.seed;
        const uint32_t team = P.mc_teams ? qi % P.mc_teams : 0;
        const uint64_t tseed = P.mc_teams ? mix_seed(qseed + 0x7ea4ull * (team + 1)) : qseed;
        uint64_t state = mix_seed(tseed ^ 0x5eedull);
        for (uint32_t j = 0; j < P.C; ++j) {
          state = mix_seed(state);
          buf[j] = (uint32_t)(state % P.n);
        }
      }
      __syncthreads();
      init = buf;
    }

    // visit(): candidates [src 0..cnt) -> evlist of first visits
    auto visit = [&](const uint32_t* src_ids, bool from_graph, uint32_t cnt) {
      PROF_T(tv0);
      bool slow = forget && (ctl.count + cnt > P.hcap);
      if (MC && MAXC > 0 && from_graph) {
        for (uint32_t j = tid; j < cnt; j += SNT) {
          const uint32_t pi = j >> P.deg_shift, c = j & (P.degree - 1);
          S.evlist[j] = P.deg_shift != 0xffu
                            ? __ldg(&P.graph[(size_t)S.parents[pi] * P.degree + c])
                            : __ldg(&P.graph[(size_t)S.parents[j / P.degree] * P.degree +
                                             j % P.degree]);
        }
        if (tid == 0) {
          ctl.nev = cnt;
          ctl.nfresh = 0;
        }
      } else if (!slow) {
        if (tid == 0) ctl.nev = 0;
        __syncthreads();
        // all of this thread's candidate ids are loaded before any insert, so
        // the graph-row gathers overlap instead of queueing behind the atomics
        constexpr int VPT = 8;
        for (uint32_t j0 = 0; j0 < cnt; j0 += SNT * VPT) {
          uint32_t ids[VPT];
#pragma unroll
          for (int k = 0; k < VPT; ++k) {
            const uint32_t j = j0 + k * SNT + tid;
            ids[k] = 0;
            if (j < cnt) {
              if (from_graph) {
                const uint32_t pi = j >> P.deg_shift, c = j & (P.degree - 1);
                ids[k] = P.deg_shift != 0xffu
                             ? __ldg(&P.graph[(size_t)S.parents[pi] * P.degree + c])
                             : __ldg(&P.graph[(size_t)S.parents[j / P.degree] * P.degree +
                                              j % P.degree]);
              } else {
                ids[k] = src_ids[j];  // global (init_samples_kernel) or shared (in-kernel)
              }
            }
          }
          if (bm) {
            // visited bitmap (standard policy): the word returned by atomicOr
            // names the one winner; all VPT atomics in flight before any use
            uint32_t old[VPT];
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
              const uint32_t j = j0 + k * SNT + tid;
              old[k] = j < cnt ? atomicOr(bm + (ids[k] >> 5), 1u << (ids[k] & 31)) : ~0u;
            }
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
              if (j0 + k * SNT >= cnt) break;
              const bool ins = !((old[k] >> (ids[k] & 31)) & 1u);
              const uint32_t pos = warp_append_slot(&ctl.nev, ins);
              if (ins) S.evlist[pos] = ids[k];
            }
          } else {
#pragma unroll
            for (int k = 0; k < VPT; ++k) {
              const uint32_t j = j0 + k * SNT + tid;
              if (j0 + k * SNT >= cnt) break;
              bool ins = false;
              if (j < cnt)
                ins = SMEM_TABLE ? smem_insert(S.table, mask, ids[k])
                    : P.mc_teams ? smem_insert(P.mc_tab + (size_t)qreal * P.hcap, mask, ids[k])
                                 : gtab_insert(gtab, mask, tag, ids[k]);
              const uint32_t pos = warp_append_slot(&ctl.nev, ins);
              if (ins) S.evlist[pos] = ids[k];
            }
          }
        }
        __syncthreads();
        if (tid == 0) ctl.count += ctl.nev;
      } else {
        // materialise candidate ids in reference order, then serial visit
        for (uint32_t j = tid; j < cnt; j += SNT) {
          uint32_t id;
          if (from_graph) {
            uint32_t pi = j / P.degree, c = j - pi * P.degree;
            id = P.graph[(size_t)S.parents[pi] * P.degree + c];
          } else {
            id = src_ids[j];
          }
          reinterpret_cast<uint32_t*>(S.surv)[j] = id;  // scratch (survivors are empty now)
        }
        __syncthreads();
        if (tid == 0) {
          uint32_t t2 = tag;
          serial_visit<SMEM_TABLE>(P, S, ctl, reinterpret_cast<uint32_t*>(S.surv), cnt, top,
                                   gtab, t2);
          ctl.slow = t2;
          ctl.dup = 1;
        }
        __syncthreads();
        if (!SMEM_TABLE) tag = ctl.slow;
      }
      __syncthreads();
      PROF_ADD(0, tv0);
      PROF_T(te0);
      uint32_t nev = ctl.nev;
      if (MC && MAXC > 0 && from_graph) {
        eval_list<TEAM, (MAXC > 0 ? MAXC : 1), EXACT, true>(
            P, S, ctl, nev, SP, P.mc_tab + (size_t)qreal * P.hcap, mask);
        __syncthreads();
        if (tid == 0) {
          ctl.evals[0] += ctl.nfresh;
          ctl.count += ctl.nfresh;
        }
      } else {
        if (MAXC > 0) eval_list<TEAM, (MAXC > 0 ? MAXC : 1), EXACT>(P, S, ctl, nev, SP);
        else eval_list_generic<EXACT>(P, S, ctl, nev, SP);
        if (tid == 0) ctl.evals[0] += nev;
      }
      __syncthreads();
      PROF_ADD(1, te0);
    };

    // update_topm(): merge survivors into top
    auto merge = [&]() {
      uint32_t ns = ctl.nsurv[0];
      if (ns > 0) {
        PROF_T(tq0);
        PROF_CNT(8, ns);
        PROF_CNT(9, 1);
        // drop duplicates of top-M entries (forgettable revisits)
        if (forget) {
          for (uint32_t j = tid; j < ns; j += SNT) {
            uint64_t s = S.surv[j];
            uint32_t ix = lb_cmp(top, P.M, s);
            if (ix < P.M && cmp_key(top[ix]) == s) {
              S.surv[j] = kDummyKey;
#ifdef CAGRA_PROF_BUILD
              if (P.prof) atomicAdd(&P.prof[10], 1ull);
#endif
            }
          }
          __syncthreads();
        }
        PROF_ADD(5, tq0);
        PROF_T(tq1);
        if (ns <= 64) {
          if (warp == 0) warp_sort_smem(S.surv, ns, lane);
        } else {
          const uint32_t P2 = max(256u, next_pow2_u32(ns));
          for (uint32_t j = ns + tid; j < P2; j += SNT) S.surv[j] = kDummyKey;
          __syncthreads();
          block_sort_any(S.surv, P2);
        }
        __syncthreads();
        if (ctl.dup) {
          // a serial visit may admit one id twice: collapse adjacent equals
          __syncthreads();
          if (tid == 0) {
            uint32_t w = 0;
            for (uint32_t j = 0; j < ns; ++j) {
              uint64_t s = S.surv[j];
              if (key_is_dummy(s)) break;
              if (w > 0 && S.surv[w - 1] == s) continue;
              S.surv[w++] = s;
            }
            ctl.nsurv[0] = w;
            ctl.dup = 0;
          }
          __syncthreads();
          ns = ctl.nsurv[0];
        } else if (forget) {
          // count survivors that are not dummies (dummies sorted last)
          uint32_t lo = 0, hi = ns;
          while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (!key_is_dummy(S.surv[mid])) lo = mid + 1;
            else hi = mid;
          }
          ns = lo;
        }
        PROF_ADD(6, tq1);
        PROF_T(tq2);
        if (P.inplace) {
          // in place: survivors' slots against the unmodified list (evlist is
          // dead after the eval), then the tail from the first survivor's
          // slot on moves right, highest chunk first — a chunk's entries are
          // all read before its barrier and land at or past the chunk's start,
          // where every entry has already been read; survivors go last
          for (uint32_t j = tid; j < ns; j += SNT) S.evlist[j] = j + lb_cmp(top, P.M, S.surv[j]);
          __syncthreads();
          const uint32_t start = ns ? S.evlist[0] : P.M;
          if (start < P.M) {
            for (int32_t c0 = (int32_t)(start + ((P.M - 1 - start) / SNT) * SNT);
                 c0 >= (int32_t)start; c0 -= SNT) {
              const uint32_t i = (uint32_t)c0 + tid;
              uint64_t e = 0;
              uint32_t pos = P.M;
              if (i >= start && i < P.M) {
                e = top[i];
                const uint64_t ke = cmp_key(e);
                uint32_t lo = 0, hi = ns;
                while (lo < hi) {
                  uint32_t mid = (lo + hi) >> 1;
                  if (S.surv[mid] < ke) lo = mid + 1;
                  else hi = mid;
                }
                pos = i + lo;
              }
              __syncthreads();
              if (pos < P.M) top[pos] = e;
            }
            for (uint32_t j = tid; j < ns; j += SNT) {
              const uint32_t pos = S.evlist[j];
              if (pos < P.M) top[pos] = S.surv[j];
            }
          }
          __syncthreads();
          PROF_ADD(7, tq2);
        } else {
        for (uint32_t i = tid; i < P.M; i += SNT) {
          uint64_t e = top[i];
          uint32_t lo = 0, hi = ns;
          uint64_t ke = cmp_key(e);
          while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (S.surv[mid] < ke) lo = mid + 1;
            else hi = mid;
          }
          uint32_t pos = i + lo;
          if (pos < P.M) nxt[pos] = e;
        }
        for (uint32_t j = tid; j < ns; j += SNT) {
          uint64_t s = S.surv[j];
          uint32_t pos = j + lb_cmp(top, P.M, s);
          if (pos < P.M) nxt[pos] = s;
        }
        __syncthreads();
        PROF_ADD(7, tq2);
        uint64_t* t = top;
        top = nxt;
        nxt = t;
        }
        if (tid == 0) ctl.nsurv[0] = 0;
      }
      __syncthreads();
    };

    // ---- init (search.cpp:192-201)
    DBG("q%u init\n", qi);
    visit(init, false, P.C);
    DBG("q%u init done nsurv=%u\n", qi, ctl.nsurv[0]);
    bool pending = true;
    uint32_t iters = 0;
    bool converged = false;
    for (;;) {
      // ---- step (search.cpp:218-245)
      DBG("q%u it%u merge ns=%u\n", qi, iters, ctl.nsurv[0]);
      {
        PROF_T(tm0);
        merge();
        PROF_ADD(2, tm0);
      }
      DBG("q%u it%u merged\n", qi, iters);
      PROF_T(ts0);
      pending = false;
      ++iters;
      // select_parents: first p unflagged non-dummy entries.  Up to 8 chunks
      // of SNT entries per round: one barrier publishes every warp's count of
      // eligible entries, then each thread ranks its entries in list order.
      uint32_t np = 0;
      for (uint32_t g0 = 0; g0 < P.M && np < P.p; g0 += kSelChunks * SNT) {
        const uint32_t nch = min((uint32_t)kSelChunks, (P.M - g0 + SNT - 1) / SNT);
        for (uint32_t c = 0; c < nch; ++c) {
          uint32_t i = g0 + c * SNT + tid;
          uint64_t e = i < P.M ? top[i] : kDummyKey;
          bool elig = i < P.M && !key_is_dummy(e) && !(e & kFlagBit64);
          unsigned bal = __ballot_sync(0xffffffffu, elig);
          if (lane == 0) ctl.warp_cnt[c * SWARPS + warp] = __popc(bal);
        }
        __syncthreads();
        uint32_t run = np;
        for (uint32_t c = 0; c < nch && run < P.p; ++c) {
          uint32_t i = g0 + c * SNT + tid;
          uint64_t e = i < P.M ? top[i] : kDummyKey;
          bool elig = i < P.M && !key_is_dummy(e) && !(e & kFlagBit64);
          unsigned bal = __ballot_sync(0xffffffffu, elig);
          uint32_t off = 0, tot = 0;
#pragma unroll
          for (int w = 0; w < SWARPS; ++w) {
            uint32_t cw = ctl.warp_cnt[c * SWARPS + w];
            off += w < warp ? cw : 0u;
            tot += cw;
          }
          uint32_t rank = run + off + __popc(bal & ((1u << lane) - 1));
          if (elig && rank < P.p) {
            S.parents[rank] = key_id(e) & kIdMask;
            top[i] = e | kFlagBit64;
          }
          run += tot;
        }
        np = min(P.p, run);
        __syncthreads();
      }
      PROF_ADD(3, ts0);
      DBG("q%u it%u np=%u\n", qi, iters, np);
      if (np == 0) {
        converged = iters >= P.min_iter;
        break;
      }
      // worst key of top-M bounds which candidates can matter
      if (tid == 0) ctl.worst[0] = cmp_key(top[P.M - 1]);
      __syncthreads();
      visit(nullptr, true, np * P.degree);
      pending = true;
      if (forget && iters % P.reset_interval == 0) {
        PROF_T(tr0);
        table_reset<SMEM_TABLE>(P, S, ctl, top, gtab, tag);
        if (tid == 0) ctl.resets++;
        PROF_ADD(4, tr0);
      }
      if (iters >= P.max_iter) break;
    }
    DBG("q%u loop done\n", qi);
    if (pending) merge();
    DBG("q%u final merge\n", qi);

    if (P.mc_teams) {
      // multi-CTA: hand the team's whole top-M list to the team merge (K7)
      for (uint32_t i = tid; i < P.M; i += SNT) P.team_out[(size_t)qi * P.M + i] = top[i];
      if (tid == 0) {
        DevStats st;
        st.iterations = iters;
        st.hash_resets = 0;
        st.distance_evals = ctl.evals[0];
        st.converged = converged ? 1u : 0u;
        st.pad = 0;
        P.team_stats[qi] = st;
      }
      __syncthreads();
      continue;
    }
    // ---- finish (search.cpp:247-259)
    uint32_t live;
    {
      uint32_t lo = 0, hi = P.k;
      while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (!key_is_dummy(top[mid])) lo = mid + 1;
        else hi = mid;
      }
      live = lo;
    }
    if (!EXACT) {
      // re-score the final k with the sequential chain, re-sort by (dist, id)
      for (uint32_t i = tid; i < live; i += SNT) {
        uint32_t id = key_id(top[i]) & kIdMask;
        nxt[i] = make_key(exact_dist(P.data + (size_t)id * P.ld, S.q, P.dim), id);
      }
      __syncthreads();
      if (live <= 256) {
        if (warp == 0) warp_sort_smem(nxt, live, lane);
      } else {
        uint32_t P2 = next_pow2_u32(live);
        for (uint32_t j = live + tid; j < P2; j += SNT) nxt[j] = kDummyKey;
        __syncthreads();
        block_sort_any(nxt, P2);
      }
      __syncthreads();
      top = nxt;
    }
    for (uint32_t i = tid; i < P.k; i += SNT) {
      bool ok = i < live;
      uint64_t e = ok ? top[i] : kDummyKey;
      P.out_ids[(size_t)qi * P.k + i] = ok ? (key_id(e) & kIdMask) : kInvalidId;
      P.out_dists[(size_t)qi * P.k + i] = key_dist(e);
    }
    if (tid == 0) {
      P.out_counts[qi] = live;
      if (P.stats) {
        DevStats st;
        st.iterations = iters;
        st.hash_resets = ctl.resets;
        st.distance_evals = ctl.evals[0];
        st.converged = converged ? 1u : 0u;
        st.pad = 0;
        P.stats[qi] = st;
      }
    }
    __syncthreads();
  }
  if (!SMEM_TABLE && !bm && !P.mc_teams && tid == 0) P.gens[blockIdx.x] = tag;
}

// ------------------------------------------------------ K7 team merge ------
// merge_team_results (engine.cpp:12-36) for the multi-CTA shared mode: per
// query the union of the T team top-M lists sorted by (dist, id), ids
// deduplicated, first k; re-scored with the sequential chain in fast mode.
// Stats: evaluations summed, iterations max, converged = all teams.
__global__ void __launch_bounds__(SNT)
team_merge_kernel(const unsigned long long* __restrict__ team_out,
                  const DevStats* __restrict__ team_stats, uint32_t T, uint32_t M, uint32_t k,
                  const float* __restrict__ data, uint32_t ld, uint32_t dim,
                  const float* __restrict__ queries, uint32_t exact, uint32_t* __restrict__ out_ids,
                  float* __restrict__ out_dists, uint32_t* __restrict__ out_counts,
                  DevStats* __restrict__ stats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t total = T * M, P2 = max(256u, next_pow2_u32(total));
  const uint32_t F = max(256u, next_pow2_u32(k));             // k <= M may exceed 256
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);   // P2
  uint64_t* fin = keys + P2;                                  // F
  __shared__ uint32_t nfin;
  for (uint32_t i = tid; i < P2; i += SNT)
    keys[i] = i < total ? cmp_key(team_out[(size_t)q * total + i]) : kDummyKey;
  __syncthreads();
  block_sort_any(keys, P2);
  __syncthreads();
  if (tid == 0) {
    uint32_t w = 0, prev = kInvalidId;
    for (uint32_t i = 0; i < P2 && w < k; ++i) {
      const uint64_t e = keys[i];
      if (key_is_dummy(e)) break;
      if (key_id(e) == prev) continue;
      prev = key_id(e);
      fin[w++] = e;
    }
    nfin = w;
  }
  __syncthreads();
  const uint32_t live = nfin;
  if (!exact) {
    // sequential-chain re-score: each warp stages a candidate row and the
    // query in shared memory with coalesced loads, then one lane runs the
    // chain from smem (a per-dimension dependent global load would dominate)
    float* rowbuf = reinterpret_cast<float*>(fin + F) + warp * 2 * ld;
    const float* qv = queries + (size_t)q * ld;
    for (uint32_t i = warp; i < live; i += SNT / 32) {
      const uint32_t id = key_id(fin[i]);
      const float* x = data + (size_t)id * ld;
      for (uint32_t j = lane; j < ld; j += 32) {
        rowbuf[j] = __ldg(x + j);
        rowbuf[ld + j] = __ldg(qv + j);
      }
      __syncwarp();
      if (lane == 0) {
        float acc = 0.0f;
        for (uint32_t d = 0; d < dim; ++d) acc = seq_step(acc, rowbuf[d], rowbuf[ld + d]);
        fin[i] = make_key(acc, id);
      }
      __syncwarp();
    }
    __syncthreads();
    if (live <= 256) {
      if (warp == 0) warp_sort_smem(fin, live, lane);
    } else {
      for (uint32_t j = live + tid; j < F; j += SNT) fin[j] = kDummyKey;
      __syncthreads();
      block_sort_any(fin, F);
    }
    __syncthreads();
  }
  for (uint32_t i = tid; i < k; i += SNT) {
    const bool ok = i < live;
    out_ids[(size_t)q * k + i] = ok ? key_id(fin[i]) : kInvalidId;
    out_dists[(size_t)q * k + i] = ok ? key_dist(fin[i]) : __int_as_float(0x7f800000);
  }
  if (tid == 0) {
    out_counts[q] = live;
    if (stats) {
      DevStats st;
      unsigned long long ev = 0;
      uint32_t it = 0, cv = 1;
      for (uint32_t t = 0; t < T; ++t) {
        const DevStats& s = team_stats[(size_t)q * T + t];
        ev += s.distance_evals;
        it = max(it, s.iterations);
        cv = cv && s.converged;
      }
      st.iterations = it;
      st.hash_resets = 0;
      st.distance_evals = ev;
      st.converged = cv;
      st.pad = 0;
      stats[q] = st;
    }
  }
}


// --------------------------------------------------- shared-mode kernel ----
// shared_query_search (engine.cpp:38-78): T traversals (p = 1, k = M,
// standard policy) share one visited table and advance in lockstep rounds,
// team 0 first.  Candidate (t, j) of a round is a first visit iff its id was
// not visited in an earlier round and no (t', j') < (t, j) of the same round
// carries the same id — exactly the reference's sequential team order.  Team
// merges / parent selection run one warp per team; expansions of all teams
// run CTA-wide.
template <int TEAM, int MAXC, bool EXACT>
__global__ void __launch_bounds__(SNT)
shared_search_kernel(const KParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Ctl ctl;
  __shared__ uint32_t parity;  // bit t: team t's current top list is in topB
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t T = P.teams;
  const uint32_t d = P.degree;
  const uint32_t SP = next_pow2_u32(d);
  const uint32_t RP = next_pow2_u32(2 * T * d);
  const uint32_t KP = next_pow2_u32(P.k);
  Smem S;
  {
    unsigned char* p = smem_raw;
    S.q = reinterpret_cast<float*>(p);
    p += sizeof(float) * round_up_u32(P.ld, 4);
    S.topA = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * P.M * T;
    S.topB = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * P.M * T;
    S.surv = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * SP * T;
    S.fin = reinterpret_cast<uint64_t*>(p);
    p += sizeof(uint64_t) * KP;
    S.rclaim = reinterpret_cast<uint32_t*>(p);
    p += sizeof(uint32_t) * 2 * RP;
    S.cand = reinterpret_cast<uint32_t*>(p);
    p += sizeof(uint32_t) * T * d;
    S.evlist = reinterpret_cast<uint32_t*>(p);
    p += sizeof(uint32_t) * T * d;
    S.evteam = reinterpret_cast<uint16_t*>(p);
    p += sizeof(uint16_t) * round_up_u32(T * d, 2);
    S.parents = reinterpret_cast<uint32_t*>(p);
  }
  unsigned long long* gtab = P.gtables + (size_t)blockIdx.x * P.hcap;
  uint32_t tag = P.gens[blockIdx.x];
  const uint32_t mask = P.hcap - 1;

  auto team_top = [&](uint32_t t) -> uint64_t* {
    return ((parity >> t) & 1u) ? S.topB + t * P.M : S.topA + t * P.M;
  };
  auto team_nxt = [&](uint32_t t) -> uint64_t* {
    return ((parity >> t) & 1u) ? S.topA + t * P.M : S.topB + t * P.M;
  };

  for (;;) {
    if (tid == 0) ctl.qi = atomicAdd(P.work, 1u);
    __syncthreads();
    const uint32_t qi = ctl.qi;
    if (qi >= P.nq) break;
    for (uint32_t i = tid; i < P.ld; i += SNT) S.q[i] = P.queries[(size_t)qi * P.ld + i];
    for (uint32_t i = tid; i < P.M * T; i += SNT) S.topA[i] = kDummyKey;
    tag = tag + 1;
    if (tid < (int)T) {
      ctl.nsurv[tid] = 0;
      ctl.evals[tid] = 0;
      ctl.iters[tid] = 0;
      ctl.done[tid] = 0;
      ctl.conv[tid] = 0;
      ctl.worst[tid] = kDummyKey;
      ctl.npar[tid] = 0;
      ctl.pending[tid] = 0;
    }
    if (tid == 0) parity = 0;
    __syncthreads();

    // Process one lockstep round of candidates for the teams in `active`.
    auto round_visit = [&](bool init_phase, uint32_t active) {
      const uint32_t total = T * d;
      for (uint32_t i = tid; i < 2 * RP; i += SNT) S.rclaim[i] = kInvalidId;
      if (tid == 0) ctl.nev = 0;
      __syncthreads();
      for (uint32_t o = tid; o < total; o += SNT) {
        uint32_t t = o / d, j = o - t * d;
        if (!((active >> t) & 1u)) continue;
        uint32_t id = init_phase ? __ldg(&P.init_ids[((size_t)qi * T + t) * d + j])
                                 : __ldg(&P.graph[(size_t)S.parents[t] * d + j]);
        S.cand[o] = id;
        uint32_t h = hash_id(id, RP - 1);
        for (;;) {
          uint32_t old = atomicCAS(&S.rclaim[h], kInvalidId, id);
          if (old == kInvalidId || old == id) break;
          h = (h + 1) & (RP - 1);
        }
        atomicMin(&S.rclaim[RP + h], o);
      }
      __syncthreads();
      for (uint32_t o = tid; o < total; o += SNT) {
        uint32_t t = o / d;
        if (!((active >> t) & 1u)) continue;
        uint32_t id = S.cand[o];
        uint32_t h = hash_id(id, RP - 1);
        while (S.rclaim[h] != id) h = (h + 1) & (RP - 1);
        if (S.rclaim[RP + h] == o && gtab_insert(gtab, mask, tag, id)) {
          uint32_t pos = atomicAdd(&ctl.nev, 1u);
          S.evlist[pos] = id;
          S.evteam[pos] = (uint16_t)t;
          atomicAdd(&ctl.evals[t], 1ull);
        }
      }
      __syncthreads();
      uint32_t nev = ctl.nev;
      if (MAXC > 0) eval_list<TEAM, (MAXC > 0 ? MAXC : 1), EXACT>(P, S, ctl, nev, SP);
      else eval_list_generic<EXACT>(P, S, ctl, nev, SP);
      __syncthreads();
    };

    // update_topm of team t by one warp
    auto team_merge = [&](uint32_t t) {
      uint32_t ns = ctl.nsurv[t];
      if (ns == 0) return;
      uint64_t* top = team_top(t);
      uint64_t* nxt = team_nxt(t);
      uint64_t* sv = S.surv + t * SP;
      warp_sort_smem(sv, ns, lane);
      for (uint32_t i = lane; i < P.M; i += 32) {
        uint64_t e = top[i];
        uint64_t ke = cmp_key(e);
        uint32_t lo = 0, hi = ns;
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if (sv[mid] < ke) lo = mid + 1;
          else hi = mid;
        }
        uint32_t pos = i + lo;
        if (pos < P.M) nxt[pos] = e;
      }
      for (uint32_t j = lane; j < ns; j += 32) {
        uint64_t s = sv[j];
        uint32_t pos = j + lb_cmp(top, P.M, s);
        if (pos < P.M) nxt[pos] = s;
      }
      __syncwarp();
      if (lane == 0) {
        atomicXor(&parity, 1u << t);
        ctl.nsurv[t] = 0;
      }
      __syncwarp();
    };

    // init: every team's d samples, team order (engine.cpp:59)
    round_visit(true, (1u << T) - 1);
    if (tid < (int)T) ctl.pending[tid] = 1;
    __syncthreads();
    uint32_t live_mask = (1u << T) - 1;
    while (live_mask) {
      for (uint32_t t = warp; t < T; t += SWARPS) {
        if (!((live_mask >> t) & 1u)) continue;
        team_merge(t);
        if (lane == 0) {
          ctl.pending[t] = 0;
          ctl.iters[t]++;
        }
        __syncwarp();
        uint64_t* top = team_top(t);
        uint32_t found = kInvalidId;
        for (uint32_t c0 = 0; c0 < P.M && found == kInvalidId; c0 += 32) {
          uint32_t i = c0 + lane;
          uint64_t e = i < P.M ? top[i] : kDummyKey;
          bool elig = i < P.M && !key_is_dummy(e) && !(e & kFlagBit64);
          unsigned bal = __ballot_sync(0xffffffffu, elig);
          if (bal) found = c0 + __ffs(bal) - 1;
        }
        if (lane == 0) {
          if (found == kInvalidId) {
            ctl.npar[t] = 0;
            ctl.conv[t] = ctl.iters[t] >= P.min_iter;
            ctl.done[t] = 1;
          } else {
            uint64_t e = top[found];
            S.parents[t] = key_id(e) & kIdMask;
            top[found] = e | kFlagBit64;
            ctl.npar[t] = 1;
            ctl.worst[t] = cmp_key(top[P.M - 1]);
          }
        }
        __syncwarp();
      }
      __syncthreads();
      uint32_t expand_mask = 0;
      for (uint32_t t = 0; t < T; ++t)
        if (((live_mask >> t) & 1u) && ctl.npar[t]) expand_mask |= 1u << t;
      if (expand_mask) round_visit(false, expand_mask);
      if (tid < (int)T && ((expand_mask >> tid) & 1u)) {
        ctl.pending[tid] = 1;
        if (ctl.iters[tid] >= P.max_iter) ctl.done[tid] = 1;
      }
      __syncthreads();
      uint32_t nl = 0;
      for (uint32_t t = 0; t < T; ++t)
        if (((live_mask >> t) & 1u) && !ctl.done[t]) nl |= 1u << t;
      live_mask = nl;
      __syncthreads();
    }
    // finish every team (search.cpp:247-259)
    for (uint32_t t = warp; t < T; t += SWARPS)
      if (ctl.pending[t]) team_merge(t);
    __syncthreads();
    // merge_team_results (engine.cpp:12-36): T-way merge of the sorted team
    // lists by (dist, id), ids deduplicated, first k.
    if (tid == 0) {
      uint32_t idx[16];
      for (uint32_t t = 0; t < T; ++t) idx[t] = 0;
      uint32_t w = 0, prev = kInvalidId;
      while (w < P.k) {
        uint64_t best = kDummyKey;
        int bt = -1;
        for (uint32_t t = 0; t < T; ++t) {
          if (idx[t] >= P.M) continue;
          uint64_t v = cmp_key(team_top(t)[idx[t]]);
          if (key_is_dummy(team_top(t)[idx[t]])) continue;
          if (bt < 0 || v < best) {
            best = v;
            bt = (int)t;
          }
        }
        if (bt < 0) break;
        idx[bt]++;
        uint32_t id = key_id(best);
        if (id == prev) continue;
        prev = id;
        S.fin[w++] = best;
      }
      ctl.nev = w;
    }
    __syncthreads();
    const uint32_t live = ctl.nev;
    if (!EXACT) {
      for (uint32_t i = tid; i < live; i += SNT) {
        uint32_t id = key_id(S.fin[i]);
        S.fin[i] = make_key(exact_dist(P.data + (size_t)id * P.ld, S.q, P.dim), id);
      }
      __syncthreads();
      if (live <= 256) {
        if (warp == 0) warp_sort_smem(S.fin, live, lane);
      } else {
        for (uint32_t j = live + tid; j < KP; j += SNT) S.fin[j] = kDummyKey;
        __syncthreads();
        block_sort_smem(S.fin, KP);
      }
      __syncthreads();
    }
    for (uint32_t i = tid; i < P.k; i += SNT) {
      bool ok = i < live;
      uint64_t e = ok ? S.fin[i] : kDummyKey;
      P.out_ids[(size_t)qi * P.k + i] = ok ? key_id(e) : kInvalidId;
      P.out_dists[(size_t)qi * P.k + i] = key_dist(e);
    }
    if (tid == 0) {
      P.out_counts[qi] = live;
      if (P.stats) {
        DevStats st;
        unsigned long long ev = 0;
        uint32_t it = 0, cv = 1;
        for (uint32_t t = 0; t < T; ++t) {
          ev += ctl.evals[t];
          it = max(it, ctl.iters[t]);
          cv = cv && ctl.conv[t];
        }
        st.iterations = it;
        st.hash_resets = 0;
        st.distance_evals = ev;
        st.converged = cv;
        st.pad = 0;
        P.stats[qi] = st;
      }
    }
    __syncthreads();
  }
  if (tid == 0) P.gens[blockIdx.x] = tag;
}

// ------------------------------------------------------------- dispatch ----
uint32_t resolved_max_iter(uint32_t max_iter, uint32_t M, uint32_t p) {
  if (max_iter) return max_iter;  // search.cpp:33-37
  uint32_t it = (2 * M + p - 1) / p;
  return it < 16 ? 16 : (it > 256 ? 256 : it);
}

// team / register-chunk variants: (team lanes, float4 chunks per lane)
struct Variant {
  int team, maxc;
};

Variant pick_variant(uint32_t ld, uint32_t req_team) {
  uint32_t ch = ld / 4;
  const Variant table[] = {{4, 2}, {8, 3}, {8, 4}, {16, 4}, {32, 8}};
  for (const Variant& v : table) {
    if (req_team && (uint32_t)v.team != req_team) continue;
    if ((uint32_t)(v.team * v.maxc) >= ch) return v;
  }
  return {32, 0};  // generic
}

using KernelFn = void (*)(const KParams);

// multi-CTA mode (fast distances only): speculative-insert instantiation
KernelFn mc_fn(Variant v) {
#ifdef CAGRA_AB_HOT_ONLY  // A/B libraries: only the 96-d kernels (ptxas in ~1 min)
  return search_kernel<8, 3, false, false, true>;
#else
  switch (v.team * 100 + v.maxc) {
    case 402: return search_kernel<4, 2, false, false, true>;
    case 803: return search_kernel<8, 3, false, false, true>;
    case 804: return search_kernel<8, 4, false, false, true>;
    case 1604: return search_kernel<16, 4, false, false, true>;
    case 3208: return search_kernel<32, 8, false, false, true>;
    default: return search_kernel<32, 0, false, false>;
  }
#endif
}

template <bool EXACT, bool SMEM>
KernelFn per_query_fn(Variant v) {
  if (EXACT) return search_kernel<32, 1, true, SMEM>;
#ifdef CAGRA_AB_HOT_ONLY
  return search_kernel<8, 3, false, SMEM>;
#else
  switch (v.team * 100 + v.maxc) {
    case 402: return search_kernel<4, 2, false, SMEM>;
    case 803: return search_kernel<8, 3, false, SMEM>;
    case 804: return search_kernel<8, 4, false, SMEM>;
    case 1604: return search_kernel<16, 4, false, SMEM>;
    case 3208: return search_kernel<32, 8, false, SMEM>;
    default: return search_kernel<32, 0, false, SMEM>;
  }
#endif
}

KernelFn shared_fn(bool exact, Variant v) {
  if (exact) return shared_search_kernel<32, 1, true>;
#ifdef CAGRA_AB_HOT_ONLY
  return shared_search_kernel<8, 3, false>;
#else
  switch (v.team * 100 + v.maxc) {
    case 402: return shared_search_kernel<4, 2, false>;
    case 803: return shared_search_kernel<8, 3, false>;
    case 804: return shared_search_kernel<8, 4, false>;
    case 1604: return shared_search_kernel<16, 4, false>;
    case 3208: return shared_search_kernel<32, 8, false>;
    default: return shared_search_kernel<32, 0, false>;
  }
#endif
}

}  // namespace

// CAGRA_VISITED_BITMAP=0: the hashed generation-tagged table instead (A/B)
// CAGRA_SEARCH_INPLACE=0 selects the double-buffered update_topm of the
// per-query kernel (A/B; default in place)
int inplace_override() {
  const char* e = std::getenv("CAGRA_SEARCH_INPLACE");
  return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
}

bool bitmap_disabled() {
  const char* e = std::getenv("CAGRA_VISITED_BITMAP");
  return e && e[0] == '0';
}

uint64_t mc_table_bytes_per_query(const SearchConfig& c, uint32_t degree) {
  // the shared-mode visited table of plan_search (engine.cpp:47-50)
  const uint32_t imax = resolved_max_iter(c.max_iter, c.topm, 1);
  const uint64_t want = 2 * std::max<uint64_t>(1, (uint64_t)(imax + 1) * c.team_count * degree);
  uint64_t cap = 1;
  while (cap < want) cap <<= 1;
  return cap * 8;
}

SearchPlan plan_search(const DeviceIndexView& ix, const SearchConfig& c, uint32_t nq,
                       int sm_count, size_t table_budget) {
  SearchPlan pl;
  const bool shared_mode = c.mode == 1;
  // multi-CTA shared mode: one CTA per (query, team), racing on a shared
  // visited table (reference order is kept only by the lockstep kernel)
  pl.mc = shared_mode && !c.exact && c.multi_cta != 1 &&
          (c.multi_cta == 2 || nq < (uint32_t)sm_count);
  const bool shared = shared_mode && !pl.mc;  // single-CTA lockstep teams
  const uint32_t T = shared_mode ? c.team_count : 1;
  if (shared && (T < 2 || T > 16))
    throw UsageErr("batch_search: lockstep shared mode supports 2 <= team_count <= 16");
  if (pl.mc && (T < 2 || T > 256))
    throw UsageErr("batch_search: multi-CTA shared mode supports 2 <= team_count <= 256");
  if (pl.mc) {
    // K7 stages the union of the team lists (T*M keys), the k finalists and
    // one row pair per warp in shared memory (launch_search)
    const uint64_t msmem = 8ull * (std::max<uint64_t>(256, next_pow2_u32(T * c.topm)) +
                                   std::max<uint32_t>(256, next_pow2_u32(c.k))) +
                           8ull * ix.ld * (SNT / 32);
    if (msmem > 200 * 1024)
      throw UsageErr("search: team_count * M exceeds the team-merge shared-memory budget");
  }
  const uint32_t p = shared_mode ? 1 : c.width;
  const uint32_t d = ix.degree;
  const uint32_t C = p * d;
  const uint32_t imax = resolved_max_iter(c.max_iter, c.topm, p);
  pl.teams = T;
  pl.C = C;
  pl.max_iter = imax;
  pl.min_iter = shared_mode ? std::min(c.min_iter, imax) : c.min_iter;  // engine.cpp:45
  const bool forget = !shared_mode && c.hash_policy == 1;
  uint64_t hcap;
  if (forget) {
    hcap = 1ull << c.hash_bits;
  } else {
    // VisitedTable::standard_sized (search.cpp:104-108)
    uint64_t expected = (uint64_t)(imax + 1) * (shared_mode ? T : p) * d;
    uint64_t want = 2 * std::max<uint64_t>(1, expected), cap = 1;
    while (cap < want) cap <<= 1;
    if (cap > (1ull << 31)) throw UsageErr("visited table capacity overflow");
    hcap = cap;
  }
  pl.hcap = (uint32_t)hcap;
  pl.smem_table = forget && hcap * 4 <= 32 * 1024;
  const uint32_t ldr = round_up_u32(ix.ld, 4);
  size_t smem;
  if (!shared) {
    uint32_t SP = std::max(256u, next_pow2_u32(C));
    // update_topm in place (one top-M buffer) unless disabled or the final
    // re-score of k > SP keys would not fit the survivor buffer it borrows;
    // measured faster at every M (fewer shared-memory writes; at M = 3328 it
    // also frees 26 KB per CTA: 2 -> 3 CTAs per SM at p = 16)
    pl.inplace = !pl.mc && inplace_override() != 0 && (c.k <= 256 || next_pow2_u32(c.k) <= SP);
    smem = 4ull * ldr + (pl.inplace ? 8ull : 16ull) * c.topm + 8ull * SP + 4ull * round_up_u32(C, 4) +
           4ull * round_up_u32(p, 4) + (pl.smem_table ? 4ull * hcap : 0);
  } else {
    if (d > 256) throw UsageErr("batch_search: shared mode on device needs graph degree <= 256");
    uint32_t SP = next_pow2_u32(d), RP = next_pow2_u32(2 * T * d), KP = next_pow2_u32(c.k);
    smem = 4ull * ldr + 16ull * c.topm * T + 8ull * SP * T + 8ull * KP + 8ull * RP +
           8ull * T * d + 2ull * round_up_u32(T * d, 2) + 4ull * round_up_u32(T, 4);
  }
  if (smem > 200 * 1024)
    throw UsageErr("search: parameters exceed the device shared-memory budget");
  pl.smem = smem;
  Variant v = pick_variant(ix.ld, c.team_size);
  KernelFn fn;
  if (shared) fn = shared_fn(c.exact != 0, v);
  else if (pl.mc) fn = mc_fn(v);
  else if (pl.smem_table) fn = c.exact ? per_query_fn<true, true>(v) : per_query_fn<false, true>(v);
  else fn = c.exact ? per_query_fn<true, false>(v) : per_query_fn<false, false>(v);
  pl.fn = reinterpret_cast<const void*>(fn);
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CAGRA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, SNT, smem));
  if (occ < 1) throw UsageErr("search: kernel cannot be resident with these parameters");
  uint64_t grid = (uint64_t)sm_count * occ;
  const uint64_t items = pl.mc ? (uint64_t)nq * T : nq;
  if (grid > items) grid = items ? items : 1;
  if (pl.mc) {
    // one visited region per query, shared by its teams
    if ((uint64_t)nq * hcap * 8 > table_budget)
      throw UsageErr("search: multi-CTA visited tables exceed the device memory budget");
    pl.table_elems = (uint64_t)nq * hcap;
    pl.team_elems = (uint64_t)nq * T * c.topm;
  } else if (!pl.smem_table && !forget && !shared_mode && !bitmap_disabled() &&
             grid * (uint64_t)round_up_u32((ix.n + 31) / 32, 4) * 4 <= table_budget) {
    // exact visited bitmap per resident CTA (n bits: 125 KB at 1M points)
    pl.bitmap = true;
    pl.bm_words = round_up_u32((ix.n + 31) / 32, 4);
    pl.table_elems = (grid * (uint64_t)pl.bm_words + 1) / 2;
  } else if (!pl.smem_table) {
    uint64_t per = hcap * 8;
    uint64_t maxg = table_budget / per;
    if (maxg < 1) throw UsageErr("search: visited table exceeds the device memory budget");
    if (grid > maxg) grid = maxg;
    pl.table_elems = grid * hcap;
  } else {
    pl.table_elems = 0;
  }
  pl.grid = (uint32_t)grid;
  pl.init_elems = (size_t)nq * T * C;
  if (pl.mc && team_b1_eligible(c.topm, c.k, T, d, ix.ld)) {
    const char* e = std::getenv("CAGRA_B1_KERNEL");  // "0": the generic multi-CTA kernel
    pl.b1 = !(e && e[0] == '0');
    if (pl.b1) {
      pl.grid = nq * T;
      // the reference-sized table (hcap slots) as a bitmap of hcap * 32 bits;
      // when that covers every node id, a bitmap of n bits indexed by id is
      // smaller and collision-free (the reference's table is exact)
      const uint32_t nw = round_up_u32((ix.n + 31) / 32, 4);
      const char* de = std::getenv("CAGRA_B1_DIRECT");  // "0": hashed bits (A/B)
      if ((uint64_t)pl.hcap * 32 >= ix.n && !(de && de[0] == '0')) {
        pl.hcap = nw;
        pl.b1_direct = true;
      }
      pl.table_elems = (uint64_t)nq * pl.hcap;  // two regions of nq * hcap words
    }
  }
  return pl;
}

uint32_t launch_search(const DeviceIndexView& ix, const SearchConfig& c, const SearchPlan& pl,
                       const float* d_queries, uint32_t nq, uint32_t* d_ids, float* d_dists,
                       uint32_t* d_counts, void* d_stats, uint32_t* d_init_ids,
                       uint32_t* d_work, unsigned long long* d_tables, uint32_t* d_gens,
                       unsigned long long* d_team_out, void* d_team_stats, uint32_t mc_tag,
                       cudaStream_t stream, uint32_t* d_b1_ctr) {
  if (nq == 0) return 0;
  // small per-item sample counts are generated inside the search kernel (one
  // launch less on the batch-1 path); the lockstep shared kernel and large
  // candidate lists use the batched sampler
  const bool sample_in_kernel = c.mode != 1 ? pl.C <= 256 : pl.mc;
  uint32_t launches = 1;
  if (!sample_in_kernel) {
    dim3 ig((nq + 127) / 128, pl.teams);
    init_samples_kernel<<<ig, 128, 0, stream>>>(nq, pl.teams > 1 ? ix.degree : pl.C, pl.teams,
                                                ix.n, c.seed, c.seed_mode, c.query_offset,
                                                d_init_ids);
    CAGRA_LAUNCH_CHECK();
    ++launches;
  }
  if (!pl.b1) CAGRA_CUDA_TRY(cudaMemsetAsync(d_work, 0, sizeof(uint32_t), stream));
  KParams P;
  P.data = ix.data;
  P.graph = ix.graph;
  P.n = ix.n;
  P.dim = ix.dim;
  P.ld = ix.ld;
  P.degree = ix.degree;
  P.deg_shift = (ix.degree & (ix.degree - 1)) == 0 ? (uint32_t)__builtin_ctz(ix.degree) : 0xffu;
  P.queries = d_queries;
  P.nq = pl.mc ? nq * pl.teams : nq;
  P.k = c.k;
  P.M = c.topm;
  P.p = c.mode == 1 ? 1 : c.width;
  P.C = pl.C;
  P.max_iter = pl.max_iter;
  P.min_iter = pl.min_iter;
  P.policy = c.mode == 1 ? 0 : c.hash_policy;
  P.reset_interval = c.reset_interval ? c.reset_interval : 1;
  P.hcap = pl.hcap;
  P.teams = pl.mc ? 1 : pl.teams;
  P.mc_teams = pl.mc ? pl.teams : 0;
  P.inplace = pl.inplace ? 1u : 0u;
  P.mc_tag = mc_tag;
  P.mc_tab = pl.mc ? reinterpret_cast<uint32_t*>(d_tables) : nullptr;
  if (pl.mc && !pl.b1)  // one visited region per query, emptied for this call
    CAGRA_CUDA_TRY(cudaMemsetAsync(d_tables, 0xff, sizeof(uint32_t) * (size_t)nq * pl.hcap, stream));
  if (pl.b1) {
    // one launch: teams + the last team's merge; its two table regions are
    // cleared alternately inside the kernel
    launch_team_b1(ix.data, ix.graph, ix.n, ix.ld, ix.dim, ix.degree, d_queries, nq, pl.teams,
                   c.topm, c.k, pl.max_iter, pl.min_iter, c.seed, c.query_offset, c.seed_mode,
                   reinterpret_cast<uint32_t*>(d_tables), pl.hcap, mc_tag,
                   pl.b1_direct ? 1u : 0u, d_team_out,
                   d_team_stats, d_b1_ctr, d_ids, d_dists, d_counts, d_stats, stream);
    return launches;
  }
  P.team_out = d_team_out;
  P.team_stats = reinterpret_cast<DevStats*>(d_team_stats);
  P.init_ids = sample_in_kernel ? nullptr : d_init_ids;
  P.seed = c.seed;
  P.query_offset = c.query_offset;
  P.seed_mode = c.seed_mode;
  P.gtables = d_tables;
  P.gens = d_gens;
  P.bitmaps = pl.bitmap ? reinterpret_cast<uint32_t*>(d_tables) : nullptr;
  P.bm_words = pl.bm_words;
  P.work = d_work;
  P.out_ids = d_ids;
  P.out_dists = d_dists;
  P.out_counts = d_counts;
  P.stats = reinterpret_cast<DevStats*>(d_stats);
  P.error = nullptr;
  P.prof = nullptr;
#ifdef CAGRA_PROF_BUILD
  const char* penv = std::getenv("CAGRA_SEARCH_PROF");
#else
  const char* penv = nullptr;  // phase profiler not compiled in
#endif
  static unsigned long long* d_prof = nullptr;
  if (penv && penv[0] == '1') {
    if (!d_prof) CAGRA_CUDA_TRY(cudaMalloc(&d_prof, 16 * sizeof(unsigned long long)));
    CAGRA_CUDA_TRY(cudaMemsetAsync(d_prof, 0, 16 * sizeof(unsigned long long), stream));
    P.prof = d_prof;
  }
  KernelFn fn = reinterpret_cast<KernelFn>(const_cast<void*>(pl.fn));
  fn<<<pl.grid, SNT, pl.smem, stream>>>(P);
  CAGRA_LAUNCH_CHECK();
  if (pl.mc) {
    const uint32_t total = pl.teams * c.topm;
    const uint32_t P2 = std::max(256u, next_pow2_u32(total));
    const uint32_t F = std::max(256u, next_pow2_u32(c.k));
    const size_t msmem = 8ull * (P2 + F) + sizeof(float) * 2 * ix.ld * (SNT / 32);
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(team_merge_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
    team_merge_kernel<<<nq, SNT, msmem, stream>>>(
        d_team_out, reinterpret_cast<const DevStats*>(d_team_stats), pl.teams, c.topm, c.k,
        ix.data, ix.ld, ix.dim, d_queries, c.exact, d_ids, d_dists, d_counts,
        reinterpret_cast<DevStats*>(d_stats));
    CAGRA_LAUNCH_CHECK();
    ++launches;
  }
  if (P.prof) {
    unsigned long long h[16];
    CAGRA_CUDA_TRY(cudaMemcpyAsync(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CAGRA_CUDA_TRY(cudaStreamSynchronize(stream));
    double tot = (double)(h[0] + h[1] + h[2] + h[3] + h[4]);
    fprintf(stderr, "search prof (cycles summed over CTAs, grid %u): visit %.3g eval %.3g merge %.3g "
                    "select %.3g reset %.3g | shares %.1f%% %.1f%% %.1f%% %.1f%% %.1f%%\n",
            pl.grid, (double)h[0], (double)h[1], (double)h[2], (double)h[3], (double)h[4],
            100 * h[0] / tot, 100 * h[1] / tot, 100 * h[2] / tot, 100 * h[3] / tot,
            100 * h[4] / tot);
    if (h[9])
      fprintf(stderr, "search prof merge: dedup %.3g sort %.3g place %.3g | merges %llu "
                      "mean survivors %.1f dups %llu\n",
              (double)h[5], (double)h[6], (double)h[7], h[9], (double)h[8] / h[9], h[10]);
  }
  return launches;
}

}  // namespace cagra
