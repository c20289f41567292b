// NN-descent on the device (nn_descent, knn_build.cpp:96-231; the paper's
// initial-graph builder): random initial rows, then
// rounds of neighbour-of-neighbour joins over sampled "new"/"old" entries
// until the rows change less than delta * N * k times in a round or
// max_rounds is reached.
//
// B200 formulation — deterministic for a fixed seed, independent of timing:
//   * rows: N x k 64-bit keys (dist bits << 32 | id), sorted by (dist, id),
//     bit 31 of the id half = "fresh" (inserted since last sampled);
//   * sampling (one warp per node): new(v) = the <= S fresh forward entries
//     with the smallest hash(seed, round, v, id) — those become stale, as in
//     the reference; old(v) = the <= S stale entries of smallest hash;
//     rev(v) = the first S reverse neighbours in (rank, source) order (the
//     device build_reverse_graph, K3);
//   * join, PULL form (one warp per node, writing only its own row — no
//     proposal buffers, no atomics on rows): the candidates of v are
//     new(u) u old(u) for u in new(v) u rev(v), and new(u) for u in old(v) —
//     the pairs the reference's push-form local join at u would propose to v
//     (knn_build.cpp:186-201); v itself and ids already in row(v) are
//     skipped (shared-memory hash), the rest get 8-lane-team distances
//     (fast filter) then the sequential fp32 chain of squared_l2 for those
//     that can enter the row, and the row becomes the k smallest (dist, id)
//     of row u accepted — the set a sequential bounded insertion of the same
//     proposals leaves (try_insert, knn_build.cpp:29-38);
//   * the round's insertion count (entries new to a row) decides termination.
// Lists: new = ceil(sample_rate k) fresh entries, old = every stale entry,
// reverse = k sources, each capped at 16 (the reference joins all its stale
// entries; the cap bounds a node's candidates at (16 + 16) 32 + 16 16 = 1280).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "host_util.hpp"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr uint32_t kFresh = 0x80000000u;  // in the id half of a row key
constexpr uint64_t kStripKey = ~(uint64_t)kFresh;
constexpr int ND_WARPS = 4;               // warps (nodes in flight) per CTA
constexpr uint32_t ND_CAND = 2560;        // candidate list capacity per node
constexpr uint32_t ND_HASH = 4096;        // dedup hash slots per node
constexpr uint32_t ND_ACC = 512;          // accepted-candidate capacity per node
constexpr uint32_t ND_MAX_S = 16;

__device__ __forceinline__ uint32_t nd_hash(uint64_t seed, uint32_t round, uint32_t v,
                                            uint32_t id) {
  // 30 bits: (hash << 32 | slot) keys stay below the dummy key in sorts
  return (uint32_t)(mix_seed(seed ^ ((uint64_t)round << 40) ^ ((uint64_t)v << 20) ^
                             (0x51ed27ull * id)) >> 34);
}

__device__ __forceinline__ float seq_l2(const float* __restrict__ a, const float* __restrict__ b,
                                        uint32_t dim) {
  float acc = 0.0f;
  for (uint32_t d = 0; d < dim; ++d) acc = seq_step(acc, __ldg(a + d), __ldg(b + d));
  return acc;
}

// Warp-wide ascending sort of up to 32 * E keys held in registers (index
// lane * E + e); E is a power of two <= 16 chosen from the count.
template <int E>
__device__ __forceinline__ void sort_into(uint64_t* buf, uint32_t cnt, int lane) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e;
    v[e] = i < cnt ? buf[i] : kDummyKey;
  }
  warp_sort_regs<E>(v, lane);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t i = lane * E + e;
    if (i < cnt) buf[i] = v[e];
  }
  __syncwarp();
}
__device__ void warp_sort_buf(uint64_t* buf, uint32_t cnt, int lane) {
  if (cnt <= 32) sort_into<1>(buf, cnt, lane);
  else if (cnt <= 64) sort_into<2>(buf, cnt, lane);
  else if (cnt <= 128) sort_into<4>(buf, cnt, lane);
  else if (cnt <= 256) sort_into<8>(buf, cnt, lane);
  else sort_into<16>(buf, cnt, lane);
}

// ---- init: k distinct random non-self ids per row, exact distances, sorted
__global__ void nd_init_kernel(const float* __restrict__ data, uint32_t n, uint32_t ld,
                               uint32_t dim, uint32_t k, uint64_t seed,
                               unsigned long long* __restrict__ rows) {
  __shared__ uint32_t acc_s[ND_WARPS][256];
  __shared__ uint64_t key_s[ND_WARPS][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t v = blockIdx.x * ND_WARPS + warp; v < n; v += gridDim.x * ND_WARPS) {
    uint32_t* acc = acc_s[warp];
    uint32_t count = 0;
    for (uint64_t t = 0; count < k; t += 32) {
      const uint32_t cand = (uint32_t)(mix_seed(seed ^ (0x1234567ull + v) ^
                                                ((t + lane + 1) * 0x9e3779b97f4a7c15ull)) %
                                       n);
      bool ok = cand != v;
      for (uint32_t j = 0; j < count && ok; ++j) ok = acc[j] != cand;
      // the first of equal candidates in this step wins
      for (int o = 0; o < 32; ++o) {
        const uint32_t c = __shfl_sync(0xffffffffu, cand, o);
        if (o < lane && c == cand) ok = false;
      }
      const unsigned b = __ballot_sync(0xffffffffu, ok);
      const uint32_t pos = count + __popc(b & ((1u << lane) - 1u));
      if (ok && pos < k) acc[pos] = cand;
      count = min(k, count + (uint32_t)__popc(b));
      __syncwarp();
    }
    const float* x = data + (size_t)v * ld;
    for (uint32_t j = lane; j < k; j += 32) {
      const uint32_t id = acc[j];
      key_s[warp][j] = make_key(seq_l2(x, data + (size_t)id * ld, dim), id);
    }
    __syncwarp();
    warp_sort_buf(key_s[warp], k, lane);
    for (uint32_t j = lane; j < k; j += 32)
      rows[(size_t)v * k + j] = key_s[warp][j] | kFresh;
    __syncwarp();
  }
}

__global__ void nd_ids_kernel(const unsigned long long* __restrict__ rows, uint64_t total,
                              uint32_t* __restrict__ ids) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x)
    ids[i] = key_id(rows[i]) & ~kFresh;
}

// ---- sampling: new(v), old(v) (S each, smallest hash), sampled fresh -> stale
__global__ void nd_sample_kernel(unsigned long long* __restrict__ rows, uint32_t n, uint32_t k,
                                 uint32_t Sn, uint32_t So, uint64_t seed, uint32_t round,
                                 uint32_t* __restrict__ new_list, uint32_t* __restrict__ old_list) {
  __shared__ uint64_t h_s[ND_WARPS][256];
  __shared__ uint32_t e_s[ND_WARPS][256];  // the row's ids + flags before this round
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t v = blockIdx.x * ND_WARPS + warp; v < n; v += gridDim.x * ND_WARPS) {
    unsigned long long* row = rows + (size_t)v * k;
    for (uint32_t j = lane; j < k; j += 32) e_s[warp][j] = key_id(row[j]);
    __syncwarp();
    for (int pass = 0; pass < 2; ++pass) {  // 0: fresh -> new, 1: stale -> old
      uint64_t* hb = h_s[warp];
      for (uint32_t j = lane; j < k; j += 32) {
        const uint32_t e = e_s[warp][j];
        const bool fresh = (e & kFresh) != 0;
        const uint32_t id = e & ~kFresh;
        hb[j] = (fresh == (pass == 0)) ? ((uint64_t)nd_hash(seed, round, v, id) << 32) | j
                                        : kDummyKey;
      }
      __syncwarp();
      warp_sort_buf(hb, k, lane);
      const uint32_t S = pass == 0 ? Sn : So;
      uint32_t* out = (pass == 0 ? new_list : old_list) + (size_t)v * S;
      for (uint32_t i = lane; i < S; i += 32) {
        const uint64_t hk = i < k ? hb[i] : kDummyKey;
        uint32_t id = kInvalidId;
        if (!key_is_dummy(hk)) {
          const uint32_t j = (uint32_t)hk;
          id = e_s[warp][j] & ~kFresh;
          if (pass == 0) row[j] &= kStripKey;  // sampled: no longer fresh
        }
        out[i] = id;
      }
      __syncwarp();
    }
  }
}

// ---- join: pull candidates from the neighbours' samples, update own row
template <int MAXC>
__global__ void __launch_bounds__(ND_WARPS * 32)
nd_join_kernel(const float* __restrict__ data, uint32_t n, uint32_t ld, uint32_t dim, uint32_t k,
               uint32_t Sn, uint32_t So, unsigned long long* __restrict__ rows,
               const uint32_t* __restrict__ new_list, const uint32_t* __restrict__ old_list,
               const uint32_t* __restrict__ rev_counts, const uint32_t* __restrict__ rev_ids,
               uint32_t rev_cap, unsigned long long* __restrict__ inserted) {
  extern __shared__ __align__(16) unsigned char nd_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = lane >> 3, lt = lane & 7;
  uint32_t* cand = reinterpret_cast<uint32_t*>(nd_smem) + warp * ND_CAND;
  uint32_t* hash = reinterpret_cast<uint32_t*>(nd_smem) + ND_WARPS * ND_CAND + warp * ND_HASH;
  uint64_t* acc = reinterpret_cast<uint64_t*>(reinterpret_cast<uint32_t*>(nd_smem) +
                                              ND_WARPS * (ND_CAND + ND_HASH)) +
                  warp * (ND_ACC + 256);
  uint64_t* rowk = acc + ND_ACC;  // the row's keys (<= 256)
  unsigned long long local_ins = 0;
  const uint32_t nchunk = ld >> 2;
  for (uint32_t v = blockIdx.x * ND_WARPS + warp; v < n; v += gridDim.x * ND_WARPS) {
    unsigned long long* row = rows + (size_t)v * k;
    for (uint32_t i = lane; i < ND_HASH; i += 32) hash[i] = kInvalidId;
    for (uint32_t j = lane; j < k; j += 32) rowk[j] = row[j];
    __syncwarp();
    // v and its current neighbours are never candidates
    auto insert = [&](uint32_t id) -> bool {
      uint32_t h = hash_id(id, ND_HASH - 1);
      for (;;) {
        const uint32_t old = atomicCAS(&hash[h], kInvalidId, id);
        if (old == kInvalidId) return true;
        if (old == id) return false;
        h = (h + 1) & (ND_HASH - 1);
      }
    };
    if (lane == 0) insert(v);
    for (uint32_t j = lane; j < k; j += 32) insert(key_id(rowk[j]) & ~kFresh);
    __syncwarp();
    // candidate ids in a fixed order (deterministic): sources u in
    // new(v), rev(v), old(v); from each u its new (+ old for the first two)
    uint32_t nc = 0;
    const uint32_t nrev = min(rev_counts[v], rev_cap);
    const uint32_t nsrc = Sn + nrev + So;
    for (uint32_t si = 0; si < nsrc; ++si) {
      uint32_t u;
      bool with_old;
      if (si < Sn) {
        u = new_list[(size_t)v * Sn + si];
        with_old = true;
      } else if (si < Sn + nrev) {
        u = rev_ids[(size_t)v * rev_cap + (si - Sn)];
        with_old = true;
      } else {
        u = old_list[(size_t)v * So + (si - Sn - nrev)];
        with_old = false;
      }
      if (u == kInvalidId) continue;
      // step 0: lanes 0..Sn-1 new(u), lanes Sn..Sn+So-1 old(u);
      // step 1: lanes 0..rev_cap-1 rev(u) (u's reverse neighbours, as the
      // reference's local join at u pairs its forward AND reverse lists)
      const uint32_t nr_u = with_old ? min(rev_counts[u], rev_cap) : 0u;
      for (int step = 0; step < 2; ++step) {
        if (step == 1 && nr_u == 0) break;
        uint32_t id = kInvalidId;
        if (step == 0) {
          if ((uint32_t)lane < Sn) id = new_list[(size_t)u * Sn + lane];
          else if (with_old && (uint32_t)lane < Sn + So) id = old_list[(size_t)u * So + lane - Sn];
        } else if ((uint32_t)lane < nr_u) {
          id = rev_ids[(size_t)u * rev_cap + lane];
        }
        // equal ids in one step: the lowest lane claims (deterministic order)
        bool first_here = id != kInvalidId;
        for (int o = 0; o < 32; ++o) {
          const uint32_t c = __shfl_sync(0xffffffffu, id, o);
          if (o < lane && c == id) first_here = false;
        }
        const bool fresh_c = first_here && insert(id);
        const unsigned b = __ballot_sync(0xffffffffu, fresh_c);
        const uint32_t pos = nc + __popc(b & ((1u << lane) - 1u));
        if (fresh_c && pos < ND_CAND) cand[pos] = id;
        nc = min(ND_CAND, nc + (uint32_t)__popc(b));
      }
    }
    __syncwarp();
    // distances: 8-lane teams (fast filter), then the sequential chain for
    // the ones that can enter the row
    const uint64_t worst = rowk[k - 1] & kStripKey;
    const float worst_f = key_dist(worst);
    const float* q = data + (size_t)v * ld;
    float4 qr[MAXC > 0 ? MAXC : 1];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const uint32_t ch = lt + 8 * c;
      qr[c] = ch < nchunk ? __ldg(reinterpret_cast<const float4*>(q) + ch)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    uint32_t na = 0;
    for (uint32_t b0 = 0; b0 < nc; b0 += 4) {
      const uint32_t ci = b0 + team;
      const uint32_t id = ci < nc ? cand[ci] : v;
      const float4* x = reinterpret_cast<const float4*>(data + (size_t)id * ld);
      float a = 0.0f;
      if (MAXC > 0) {
#pragma unroll
        for (int c = 0; c < (MAXC > 0 ? MAXC : 1); ++c) {
          const uint32_t ch = lt + 8 * c;
          if (ch < nchunk) {
            const float4 xv = __ldg(x + ch);
            const float dx = xv.x - qr[c].x, dy = xv.y - qr[c].y;
            const float dz = xv.z - qr[c].z, dw = xv.w - qr[c].w;
            a = fmaf(dx, dx, a);
            a = fmaf(dy, dy, a);
            a = fmaf(dz, dz, a);
            a = fmaf(dw, dw, a);
          }
        }
      } else {
        for (uint32_t ch = lt; ch < nchunk; ch += 8) {
          const float4 xv = __ldg(x + ch), qv = __ldg(reinterpret_cast<const float4*>(q) + ch);
          const float dx = xv.x - qv.x, dy = xv.y - qv.y, dz = xv.z - qv.z, dw = xv.w - qv.w;
          a = fmaf(dx, dx, a);
          a = fmaf(dy, dy, a);
          a = fmaf(dz, dz, a);
          a = fmaf(dw, dw, a);
        }
      }
      a += __shfl_xor_sync(0xffffffffu, a, 4);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      // a candidate within a small relative margin of the row's worst gets the
      // exact distance (the team sum differs from the chain by a few ulps)
      bool maybe = lt == 0 && ci < nc && a <= worst_f * (1.0f + 1e-4f) + 1e-30f;
      uint64_t key = kDummyKey;
      if (maybe) {
        key = make_key(seq_l2(q, data + (size_t)id * ld, dim), id);
        maybe = key < worst;
      }
      const unsigned bm = __ballot_sync(0xffffffffu, maybe);
      const uint32_t pos = na + __popc(bm & ((1u << lane) - 1u));
      if (maybe && pos < ND_ACC) acc[pos] = key;
      na = min(ND_ACC, na + (uint32_t)__popc(bm));
    }
    __syncwarp();
    if (na) {
      // row := the k smallest of row u accepted (ranks: binary searches in
      // the two sorted lists, then one scatter); accepted keys enter fresh
      warp_sort_buf(acc, na, lane);
      uint64_t* out = reinterpret_cast<uint64_t*>(hash);  // hash is no longer needed
      __syncwarp();
      uint32_t ins = 0;
      for (uint32_t j = lane; j < k; j += 32) {
        const uint64_t x = rowk[j] & kStripKey;
        uint32_t lo = 0, hi = na;  // accepted keys before x
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (acc[mid] < x) lo = mid + 1;
          else hi = mid;
        }
        if (j + lo < k) out[j + lo] = rowk[j];
      }
      for (uint32_t i = lane; i < na; i += 32) {
        const uint64_t x = acc[i];
        uint32_t lo = 0, hi = k;  // row keys before x
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if ((rowk[mid] & kStripKey) < x) lo = mid + 1;
          else hi = mid;
        }
        if (i + lo < k) {
          out[i + lo] = x | kFresh;
          ++ins;
        }
      }
      __syncwarp();
      for (uint32_t j = lane; j < k; j += 32) row[j] = out[j];
      local_ins += ins;
      __syncwarp();
    }
  }
  local_ins += __shfl_xor_sync(0xffffffffu, local_ins, 16);
  local_ins += __shfl_xor_sync(0xffffffffu, local_ins, 8);
  local_ins += __shfl_xor_sync(0xffffffffu, local_ins, 4);
  local_ins += __shfl_xor_sync(0xffffffffu, local_ins, 2);
  local_ins += __shfl_xor_sync(0xffffffffu, local_ins, 1);
  if (lane == 0 && local_ins) atomicAdd(inserted, local_ins);
}

__global__ void nd_output_kernel(const unsigned long long* __restrict__ rows, uint64_t total,
                                 uint32_t* __restrict__ ids, float* __restrict__ dists) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = rows[i] & kStripKey;
    ids[i] = key_id(key);
    dists[i] = key_dist(key);
  }
}

}  // namespace

NnDescentInfo launch_nn_descent(const float* d_data, uint32_t n, uint32_t ld, uint32_t dim,
                                uint32_t k, double sample_rate, double termination_delta,
                                uint32_t max_rounds, uint64_t seed, uint32_t* d_ids,
                                float* d_dists, cudaStream_t s) {
  if (k > 256) throw UsageErr("nn_descent on device: k <= 256");
  int dev = 0, sms = 148;
  CAGRA_CUDA_TRY(cudaGetDevice(&dev));
  CAGRA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // new: ceil(sample_rate k) fresh entries; old: every stale entry; reverse:
  // k sources (the reference's reservoir bound) — each capped at 16 per list
  const uint32_t Sn = std::min<uint32_t>(
      ND_MAX_S, std::max<uint32_t>(1, (uint32_t)std::ceil(sample_rate * (double)k)));
  const uint32_t So = std::min<uint32_t>(ND_MAX_S, k), Sr = std::min<uint32_t>(ND_MAX_S, k);
  const uint64_t total = (uint64_t)n * k;
  DBuf rows(8 * total), ids(4 * total), nl(4ull * n * Sn), ol(4ull * n * So), rc(4ull * n),
      ri(4ull * n * Sr), scratch(reverse_scratch_bytes(n, k)), ins(8);
  const uint32_t grid = (uint32_t)std::min<uint64_t>((n + ND_WARPS - 1) / ND_WARPS,
                                                     (uint64_t)sms * 16);
  nd_init_kernel<<<grid, ND_WARPS * 32, 0, s>>>(d_data, n, ld, dim, k, seed,
                                                rows.as<unsigned long long>());
  CAGRA_LAUNCH_CHECK();
  const uint64_t stop_below = (uint64_t)(termination_delta * (double)n * (double)k);
  const size_t jsmem = (size_t)ND_WARPS * (4 * (ND_CAND + ND_HASH) + 8 * (ND_ACC + 256));
  const uint32_t maxc = (ld / 4 + 7) / 8;
  auto join = [&](auto kern) {
    CAGRA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)jsmem));
    kern<<<grid, ND_WARPS * 32, jsmem, s>>>(d_data, n, ld, dim, k, Sn, So,
                                            rows.as<unsigned long long>(), nl.as<uint32_t>(),
                                            ol.as<uint32_t>(), rc.as<uint32_t>(),
                                            ri.as<uint32_t>(), Sr, ins.as<unsigned long long>());
  };
  NnDescentInfo info;
  for (uint32_t round = 0; round < max_rounds; ++round) {
    nd_ids_kernel<<<grid, 256, 0, s>>>(rows.as<unsigned long long>(), total, ids.as<uint32_t>());
    CAGRA_LAUNCH_CHECK();
    // reverse neighbours: first S sources per node in (rank, source) order (K3)
    launch_reverse(ids.as<uint32_t>(), n, k, Sr, scratch.p, rc.as<uint32_t>(), ri.as<uint32_t>(),
                   s);
    nd_sample_kernel<<<grid, ND_WARPS * 32, 0, s>>>(rows.as<unsigned long long>(), n, k, Sn, So,
                                                    seed, round, nl.as<uint32_t>(),
                                                    ol.as<uint32_t>());
    CAGRA_LAUNCH_CHECK();
    CAGRA_CUDA_TRY(cudaMemsetAsync(ins.p, 0, 8, s));
    if (maxc <= 1) join(nd_join_kernel<1>);
    else if (maxc <= 2) join(nd_join_kernel<2>);
    else if (maxc <= 4) join(nd_join_kernel<4>);
    else if (maxc <= 8) join(nd_join_kernel<8>);
    else if (maxc <= 32) join(nd_join_kernel<32>);
    else join(nd_join_kernel<0>);
    CAGRA_LAUNCH_CHECK();
    unsigned long long h = 0;
    CAGRA_CUDA_TRY(cudaMemcpyAsync(&h, ins.p, 8, cudaMemcpyDeviceToHost, s));
    CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
    info.rounds = round + 1;
    info.last_inserted = h;
    if (h < stop_below) {
      info.converged = true;
      break;
    }
  }
  nd_output_kernel<<<grid, 256, 0, s>>>(rows.as<unsigned long long>(), total, d_ids, d_dists);
  CAGRA_LAUNCH_CHECK();
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
  return info;
}

}  // namespace cagra
