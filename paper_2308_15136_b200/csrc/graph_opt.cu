// Rank-mode graph optimization on device (graph_opt.cpp:45-246), bit-exact:
//   K2 detour_reorder : count_detourable_routes (:45-96) fused with
//                       reorder_and_prune (:98-124) — one CTA per node
//   K3 reverse        : build_reverse_graph (:141-160) — count, scan, scatter,
//                       per-row (rank, source) selection
//   K4 merge          : merge_graphs (:162-209) — one warp per node
// Integer work only; every output position is a pure function of the input
// rows (atomics only accumulate counts or claim bucket slots that are sorted
// afterwards), so results never depend on scheduling.
#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int OPT_NT = 128;

// ---------------------------------------------------------------- checks --
__global__ void check_sorted_kernel(const uint32_t* __restrict__ ids,
                                    const float* __restrict__ dists, uint32_t n, uint32_t deg,
                                    int* flag) {
  // graph_opt.cpp:19-31: (dist, id) strictly increasing along each row.
  uint64_t total = (uint64_t)n * deg;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    if (e % deg == 0) continue;
    float a = dists[e - 1], b = dists[e];
    bool ok = a < b || (a == b && ids[e - 1] < ids[e]);
    if (!ok) atomicOr(flag, 1);
  }
}

__global__ void check_ids_kernel(const uint32_t* __restrict__ ids, uint64_t count, uint32_t n,
                                 int* flag) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
       e += (uint64_t)gridDim.x * blockDim.x)
    if (ids[e] >= n) atomicOr(flag, 2);
}

// ------------------------------------------------------ block bitonic sort --
__device__ void block_bitonic_sort(uint64_t* a, uint32_t P) {
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

// ------------------------------------------------------------------- K2 ---
// rank_of(X) as an open-addressing table of packed (rank << 32 | id) slots,
// sized 8 deg (load <= 1/8: a miss — most probes, since most two-hop ids are
// not in X's row — costs about one 8-byte shared load), indexed by the high
// bits of a multiplicative hash.
constexpr uint64_t kSlotEmpty = ~0ull;

__device__ __forceinline__ uint32_t slot_of(uint32_t id, uint32_t hshift) {
  return (id * 2654435761u) >> hshift;
}

__device__ __forceinline__ uint32_t rank_lookup(const uint64_t* tab, uint32_t hmask,
                                                uint32_t hshift, uint32_t y) {
  uint32_t h = slot_of(y, hshift);
  for (;;) {
    const uint64_t e = tab[h];
    if (static_cast<uint32_t>(e) == y) return static_cast<uint32_t>(e >> 32);
    if (e == kSlotEmpty) return kInvalidId;
    h = (h + 1) & hmask;
  }
}

// Shared layout: tab[H] (u64, 16-byte aligned) | keys[P] (u64) | xrow[deg] | counts[deg]
__global__ void __launch_bounds__(OPT_NT)
detour_reorder_kernel(const uint32_t* __restrict__ knn, uint32_t n, uint32_t deg, uint32_t d,
                      uint32_t H, uint32_t P, const uint32_t* __restrict__ counts_in,
                      uint32_t* __restrict__ counts_out, uint32_t* __restrict__ pruned_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* keys = tab + H;
  uint32_t* xrow = reinterpret_cast<uint32_t*>(keys + P);
  uint32_t* counts = xrow + deg;
  const uint32_t hmask = H - 1, hshift = 32u - __ffs(H) + 1u;  // H = 2^b: shift 32 - b
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  for (uint32_t x = blockIdx.x; x < n; x += gridDim.x) {
    const uint32_t* xr = knn + (size_t)x * deg;
    if (counts_in == nullptr) {
      uint4* t4 = reinterpret_cast<uint4*>(tab);  // H >= 2: whole 16-byte pairs
      for (uint32_t i = tid; i < H / 2; i += blockDim.x)
        t4[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    for (uint32_t r = tid; r < deg; r += blockDim.x) {
      xrow[r] = xr[r];
      counts[r] = 0;
    }
    __syncthreads();
    if (counts_in == nullptr) {
      // rank_of: first occurrence wins (unordered_map::emplace, graph_opt.cpp:62):
      // a repeated id keeps the smaller rank (same low word -> u64 min)
      for (uint32_t r = tid; r < deg; r += blockDim.x) {
        const uint32_t id = xrow[r];
        const uint64_t e = ((uint64_t)r << 32) | id;
        uint32_t h = slot_of(id, hshift);
        for (;;) {
          const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(&tab[h]),
                                         kSlotEmpty, e);
          if (old == kSlotEmpty) break;
          if (static_cast<uint32_t>(old) == id) {
            atomicMin(reinterpret_cast<unsigned long long*>(&tab[h]), e);
            break;
          }
          h = (h + 1) & hmask;
        }
      }
      __syncthreads();
      // X -> Z (rank rz) -> Y (rank rzy in Z's row); X -> Y at rank ry.
      // Only routes with max(rz, rzy) < ry count (graph_opt.cpp:74-93), so
      // rz and rzy never need to reach deg-1.  The counts are integer sums:
      // the order of the additions does not matter.
      const uint32_t last = deg - 1;
      if ((deg & 3) == 0 && deg <= 128) {
        // Z rows as one 16-byte load per lane (lane l: ranks 4l..4l+3), R rows
        // per warp in flight together
        constexpr uint32_t R = 4;
        for (uint32_t rz0 = warp * R; rz0 < last; rz0 += nwarps * R) {
          uint4 v[R];
#pragma unroll
          for (uint32_t u = 0; u < R; ++u) {
            const uint32_t rz = rz0 + u;
            v[u] = rz < last && lane * 4 < deg
                       ? __ldg(reinterpret_cast<const uint4*>(knn + (size_t)xrow[rz] * deg) + lane)
                       : make_uint4(x, x, x, x);  // y == x: skipped
          }
#pragma unroll
          for (uint32_t u = 0; u < R; ++u) {
            const uint32_t rz = rz0 + u;
            const uint32_t ys[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (uint32_t e = 0; e < 4; ++e) {
              const uint32_t rzy = lane * 4 + e, y = ys[e];
              if (rzy >= last || y == x) continue;
              const uint32_t ry = rank_lookup(tab, hmask, hshift, y);
              if (ry == kInvalidId || ry == rz) continue;
              if ((rz > rzy ? rz : rzy) < ry) atomicAdd(&counts[ry], 1u);
            }
          }
        }
      } else {
        for (uint32_t rz = warp; rz < last; rz += nwarps) {
          const uint32_t* zr = knn + (size_t)xrow[rz] * deg;
          for (uint32_t rzy = lane; rzy < last; rzy += 32) {
            const uint32_t y = __ldg(&zr[rzy]);
            if (y == x) continue;
            const uint32_t ry = rank_lookup(tab, hmask, hshift, y);
            if (ry == kInvalidId || ry == rz) continue;
            if ((rz > rzy ? rz : rzy) < ry) atomicAdd(&counts[ry], 1u);
          }
        }
      }
      __syncthreads();
    } else {
      for (uint32_t r = tid; r < deg; r += blockDim.x) counts[r] = counts_in[(size_t)x * deg + r];
      __syncthreads();
    }
    if (counts_out)
      for (uint32_t r = tid; r < deg; r += blockDim.x) counts_out[(size_t)x * deg + r] = counts[r];
    if (pruned_out) {
      // stable sort by count == sort by (count, initial rank)
      for (uint32_t i = tid; i < P; i += blockDim.x)
        keys[i] = i < deg ? ((uint64_t)counts[i] << 32) | i : ~0ull;
      __syncthreads();
      block_bitonic_sort(keys, P);
      for (uint32_t j = tid; j < d; j += blockDim.x)
        pruned_out[(size_t)x * d + j] = xrow[(uint32_t)keys[j]];
    }
    __syncthreads();
  }
}

// Distance-mode detour counting (graph_opt.cpp:66-71, 87-93), the paper's
// comparison variant: every leg is recomputed from the vectors with the
// sequential fp32 chain (w(X->Z), w(Z->Y), w(X->Y)); a route counts when
// max(w(X->Z), w(Z->Y)) < w(X->Y).  One CTA per node X.
// Shared layout: xrow[deg] | hkey[H] | hrank[H] | counts[deg] | xdist[deg]
__global__ void __launch_bounds__(OPT_NT)
detour_distance_kernel(const uint32_t* __restrict__ knn, uint32_t n, uint32_t deg, uint32_t H,
                       const float* __restrict__ data, uint32_t ld, uint32_t dim,
                       uint32_t* __restrict__ counts_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* xrow = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* hkey = xrow + deg;
  uint32_t* hrank = hkey + H;
  uint32_t* counts = hrank + H;
  float* xdist = reinterpret_cast<float*>(counts + deg);
  const uint32_t hmask = H - 1;
  auto dist = [&](uint32_t a, uint32_t b) {
    const float* pa = data + (size_t)a * ld;
    const float* pb = data + (size_t)b * ld;
    float acc = 0.0f;
    for (uint32_t i = 0; i < dim; ++i) acc = seq_step(acc, __ldg(pa + i), __ldg(pb + i));
    return acc;
  };
  for (uint32_t x = blockIdx.x; x < n; x += gridDim.x) {
    const uint32_t* xr = knn + (size_t)x * deg;
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) {
      hkey[i] = kInvalidId;
      hrank[i] = kInvalidId;
    }
    for (uint32_t r = threadIdx.x; r < deg; r += blockDim.x) {
      xrow[r] = xr[r];
      counts[r] = 0;
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < deg; r += blockDim.x) {
      const uint32_t id = xrow[r];
      uint32_t h = hash_id(id, hmask);
      for (;;) {
        uint32_t old = atomicCAS(&hkey[h], kInvalidId, id);
        if (old == kInvalidId || old == id) break;
        h = (h + 1) & hmask;
      }
      atomicMin(&hrank[h], r);
      xdist[r] = dist(x, id);
    }
    __syncthreads();
    for (uint32_t pi = threadIdx.x; pi < deg * deg; pi += blockDim.x) {
      const uint32_t rz = pi / deg, rzy = pi - rz * deg;
      const uint32_t z = xrow[rz];
      const uint32_t y = __ldg(&knn[(size_t)z * deg + rzy]);
      if (y == x) continue;
      uint32_t h = hash_id(y, hmask), ry = kInvalidId;
      for (;;) {
        const uint32_t k = hkey[h];
        if (k == y) {
          ry = hrank[h];
          break;
        }
        if (k == kInvalidId) break;
        h = (h + 1) & hmask;
      }
      if (ry == kInvalidId || ry == rz) continue;
      const float wzy = dist(z, y);
      const float a = xdist[rz];
      if ((a < wzy ? wzy : a) < xdist[ry]) atomicAdd(&counts[ry], 1u);
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < deg; r += blockDim.x) counts_out[(size_t)x * deg + r] = counts[r];
    __syncthreads();
  }
}

size_t detour_smem(uint32_t deg, uint32_t H, uint32_t P) {
  return sizeof(uint64_t) * (P + H) + sizeof(uint32_t) * 2 * deg;
}

// ------------------------------------------------------------------- K3 ---
__global__ void indeg_kernel(const uint32_t* __restrict__ pruned, uint64_t edges,
                             uint32_t* __restrict__ indeg) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < edges;
       e += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&indeg[pruned[e]], 1u);
}

constexpr int SCAN_NT = 256;
constexpr int SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_NT * SCAN_PER;

// block-local exclusive scan of SCAN_TILE values; returns block total
__device__ unsigned long long block_scan_tile(const uint32_t* in, uint32_t n, uint32_t base,
                                              unsigned long long* out, unsigned long long carry) {
  __shared__ unsigned long long warp_tot[SCAN_NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long v[SCAN_PER];
  unsigned long long local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    uint32_t idx = base + tid * SCAN_PER + i;
    v[i] = idx < n ? in[idx] : 0;
    local += v[i];
  }
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  unsigned long long woff = 0, total = 0;
  for (int w = 0; w < SCAN_NT / 32; ++w) {
    if (w < warp) woff += warp_tot[w];
    total += warp_tot[w];
  }
  unsigned long long run = carry + woff + incl - local;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    uint32_t idx = base + tid * SCAN_PER + i;
    if (out && idx < n) out[idx] = run;
    run += v[i];
  }
  __syncthreads();
  return total;
}

__global__ void scan_partial_kernel(const uint32_t* in, uint32_t n,
                                    unsigned long long* block_sums) {
  unsigned long long t = block_scan_tile(in, n, blockIdx.x * SCAN_TILE, nullptr, 0);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = t;
}

__global__ void scan_block_sums_kernel(unsigned long long* sums, uint32_t nb) {
  // single CTA, sequential over tiles of block sums (exclusive, in place)
  __shared__ unsigned long long tile[SCAN_TILE];
  __shared__ unsigned long long carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < nb; b0 += SCAN_TILE) {
    for (int i = threadIdx.x; i < SCAN_TILE; i += SCAN_NT)
      tile[i] = b0 + i < nb ? sums[b0 + i] : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long c = carry_s;
      for (int i = 0; i < SCAN_TILE && b0 + i < nb; ++i) {
        unsigned long long t = tile[i];
        sums[b0 + i] = c;
        c += t;
      }
      carry_s = c;
    }
    __syncthreads();
  }
}

__global__ void scan_final_kernel(const uint32_t* in, uint32_t n,
                                  const unsigned long long* block_sums,
                                  unsigned long long* out) {
  block_scan_tile(in, n, blockIdx.x * SCAN_TILE, out, block_sums[blockIdx.x]);
}

__global__ void set_total_kernel(const uint32_t* in, uint32_t n, unsigned long long* out) {
  out[n] = out[n - 1] + in[n - 1];
}

__global__ void reverse_scatter_kernel(const uint32_t* __restrict__ pruned, uint32_t n,
                                       uint32_t d, const unsigned long long* __restrict__ start,
                                       uint32_t* __restrict__ fill, uint64_t* __restrict__ keys) {
  uint64_t edges = (uint64_t)n * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < edges;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)(e / d), r = (uint32_t)(e % d);
    uint32_t y = pruned[e];
    uint32_t pos = atomicAdd(&fill[y], 1u);
    keys[start[y] + pos] = ((uint64_t)r << 32) | x;  // order (rank, source)
  }
}

constexpr int REV_WARPS = 8;
constexpr int REV_BUF = 1024;  // per-warp key buffer

// Warp per target node y: the `cap` smallest (rank, source) keys of its
// bucket, processed in chunks so any in-degree works.
__global__ void __launch_bounds__(REV_WARPS * 32)
reverse_select_kernel(const unsigned long long* __restrict__ start,
                      const uint64_t* __restrict__ keys, uint32_t n, uint32_t cap,
                      uint32_t* __restrict__ rev_counts, uint32_t* __restrict__ rev_ids) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-warp key buffer: the best `cap` so far + the next chunk of in-edges
  const uint32_t capP = next_pow2_u32(cap);
  const uint32_t rev_buf = capP <= REV_BUF / 2 ? REV_BUF : 2 * capP;
  const uint32_t nwarps = blockDim.x >> 5;
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * rev_buf;
  const uint32_t chunk = rev_buf - capP;
  for (uint32_t y = blockIdx.x * nwarps + warp; y < n; y += gridDim.x * nwarps) {
    unsigned long long b = start[y], e = start[y + 1];
    uint32_t len = (uint32_t)(e - b);
    uint32_t have = 0;  // sorted best prefix in buf[0..have)
    for (uint32_t off = 0; off < len; off += chunk) {
      uint32_t take = min(chunk, len - off);
      uint32_t tot = have + take;
      uint32_t P = next_pow2_u32(tot);
      for (uint32_t i = lane; i < P; i += 32) {
        if (i >= have) buf[i] = (i < tot) ? keys[b + off + (i - have)] : ~0ull;
      }
      __syncwarp();
      for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = lane; i < P; i += 32) {
            uint32_t ixj = i ^ j;
            if (ixj > i) {
              uint64_t u = buf[i], v = buf[ixj];
              bool up = (i & k) == 0;
              if ((u > v) == up) {
                buf[i] = v;
                buf[ixj] = u;
              }
            }
          }
          __syncwarp();
        }
      have = min(tot, cap);
    }
    for (uint32_t i = lane; i < have; i += 32) rev_ids[(size_t)y * cap + i] = (uint32_t)buf[i];
    if (lane == 0) rev_counts[y] = have;
    __syncwarp();
  }
}

// ------------------------------------------------------------------- K4 ---
constexpr int MRG_WARPS = 4;

// Warp per node: the reference's sequential interleave (graph_opt.cpp:177-206),
// with the "already emitted" test done by all 32 lanes against the emitted
// prefix (ballot) instead of a serial scan.
__global__ void __launch_bounds__(MRG_WARPS * 32)
merge_kernel(const uint32_t* __restrict__ pruned, const uint32_t* __restrict__ rev_counts,
             const uint32_t* __restrict__ rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
             uint32_t* __restrict__ out, int* flag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* P = reinterpret_cast<uint32_t*>(smem_raw) + warp * (2 * d + rev_cap);
  uint32_t* R = P + d;
  uint32_t* E = R + rev_cap;
  for (uint32_t v = blockIdx.x * MRG_WARPS + warp; v < n; v += gridDim.x * MRG_WARPS) {
    uint32_t rlen = rev_counts[v];
    for (uint32_t i = lane; i < d; i += 32) P[i] = pruned[(size_t)v * d + i];
    for (uint32_t i = lane; i < rlen; i += 32) R[i] = rev_ids[(size_t)v * rev_cap + i];
    __syncwarp();
    uint32_t pi = 0, ri = 0, emitted = 0;
    bool ok = true;
    for (uint32_t slot = 0; slot < d && ok; ++slot) {
      bool got = false;
      uint32_t id = 0;
      for (int attempt = 0; attempt < 2 && !got; ++attempt) {
        bool from_p = ((slot & 1) == 0) != (attempt == 1);
        const uint32_t* src = from_p ? P : R;
        uint32_t len = from_p ? d : rlen;
        uint32_t& pos = from_p ? pi : ri;
        while (pos < len && !got) {
          uint32_t cand = src[pos++];
          bool dup = false;
          for (uint32_t j0 = 0; j0 < emitted && !dup; j0 += 32) {
            uint32_t j = j0 + lane;
            dup = __any_sync(0xffffffffu, j < emitted && E[j] == cand);
          }
          if (!dup) {
            id = cand;
            got = true;
          }
        }
      }
      if (!got) {
        ok = false;
        break;
      }
      if (lane == 0) E[emitted] = id;
      __syncwarp();
      ++emitted;
    }
    if (!ok) {
      if (lane == 0) atomicOr(flag, 4);
    } else {
      for (uint32_t i = lane; i < d; i += 32) out[(size_t)v * d + i] = E[i];
    }
    __syncwarp();
  }
}

int grid_for(uint64_t work, int nt) {
  uint64_t g = (work + nt - 1) / nt;
  return (int)(g > 148 * 64 ? 148 * 64 : (g == 0 ? 1 : g));
}

}  // namespace

void launch_check_sorted(const uint32_t* d_ids, const float* d_dists, uint32_t n, uint32_t deg,
                         int* d_flag, cudaStream_t stream) {
  uint64_t total = (uint64_t)n * deg;
  if (total == 0) return;
  check_sorted_kernel<<<grid_for(total, 256), 256, 0, stream>>>(d_ids, d_dists, n, deg, d_flag);
  CAGRA_LAUNCH_CHECK();
}

void launch_check_ids(const uint32_t* d_ids, uint64_t count, uint32_t n, int* d_flag,
                      cudaStream_t stream) {
  if (count == 0) return;
  check_ids_kernel<<<grid_for(count, 256), 256, 0, stream>>>(d_ids, count, n, d_flag);
  CAGRA_LAUNCH_CHECK();
}

static void detour_launch(const uint32_t* d_knn, const uint32_t* d_counts_in, uint32_t n,
                          uint32_t deg, uint32_t d, uint32_t* d_counts_out,
                          uint32_t* d_pruned_out, cudaStream_t stream) {
  uint32_t H = next_pow2_u32(8 * deg);  // load <= 1/8 (rank_lookup)
  uint32_t P = next_pow2_u32(deg);
  while (H > 2 * P && detour_smem(deg, H, P) > 48 * 1024) H >>= 1;  // keep 4+ CTAs per SM
  size_t smem = detour_smem(deg, H, P);
  if (smem > 200 * 1024) throw UsageErr("optimize: input degree too large for the device kernel");
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(detour_reorder_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = (int)(n < 148u * 64u ? n : 148u * 64u);
  detour_reorder_kernel<<<grid, OPT_NT, smem, stream>>>(d_knn, n, deg, d, H, P, d_counts_in,
                                                        d_counts_out, d_pruned_out);
  CAGRA_LAUNCH_CHECK();
}

void launch_detour_reorder(const uint32_t* d_knn, uint32_t n, uint32_t deg, uint32_t d,
                           uint32_t* d_counts_out, uint32_t* d_pruned_out, cudaStream_t stream) {
  detour_launch(d_knn, nullptr, n, deg, d, d_counts_out, d_pruned_out, stream);
}

void launch_detour_distance(const uint32_t* d_knn, uint32_t n, uint32_t deg, const float* d_data,
                            uint32_t ld, uint32_t dim, uint32_t* d_counts_out,
                            cudaStream_t stream) {
  const uint32_t H = next_pow2_u32(2 * deg);
  const size_t smem = sizeof(uint32_t) * (2 * (size_t)deg + 2 * H) + sizeof(float) * deg;
  if (smem > 200 * 1024) throw UsageErr("optimize: input degree too large for the device kernel");
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(detour_distance_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)(n < 148u * 64u ? n : 148u * 64u);
  detour_distance_kernel<<<grid, OPT_NT, smem, stream>>>(d_knn, n, deg, H, d_data, ld, dim,
                                                         d_counts_out);
  CAGRA_LAUNCH_CHECK();
}

void launch_reorder_from_counts(const uint32_t* d_knn, const uint32_t* d_counts, uint32_t n,
                                uint32_t deg, uint32_t d, uint32_t* d_pruned_out,
                                cudaStream_t stream) {
  detour_launch(d_knn, d_counts, n, deg, d, nullptr, d_pruned_out, stream);
}

size_t reverse_scratch_bytes(uint32_t n, uint32_t d) {
  size_t nb = (n + SCAN_TILE - 1) / SCAN_TILE + 1;
  return 256 + sizeof(uint32_t) * (size_t)n + 256 + sizeof(unsigned long long) * ((size_t)n + 1) +
         256 + sizeof(uint32_t) * (size_t)n + 256 + sizeof(uint64_t) * (size_t)n * d + 256 +
         sizeof(unsigned long long) * nb + 256;
}

static char* carve(char*& p, size_t bytes) {
  char* r = p;
  p += (bytes + 255) / 256 * 256;
  return r;
}

void launch_reverse(const uint32_t* d_pruned, uint32_t n, uint32_t d, uint32_t cap,
                    void* d_scratch, uint32_t* d_rev_counts, uint32_t* d_rev_ids,
                    cudaStream_t stream) {
  // rows never hold more than their in-degree: a cap above the largest
  // possible in-degree (n) is "no cap" (graph_opt.cpp:141-160)
  if (cap > n) cap = n;
  if (cap > 8192) throw UsageErr("build_reverse_graph: cap > 8192 unsupported on device");
  char* p = reinterpret_cast<char*>(d_scratch);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) / 256 * 256);
  uint32_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  uint32_t* indeg = reinterpret_cast<uint32_t*>(carve(p, sizeof(uint32_t) * n));
  auto* start = reinterpret_cast<unsigned long long*>(carve(p, sizeof(unsigned long long) * (n + 1)));
  uint32_t* fill = reinterpret_cast<uint32_t*>(carve(p, sizeof(uint32_t) * n));
  uint64_t* keys = reinterpret_cast<uint64_t*>(carve(p, sizeof(uint64_t) * (size_t)n * d));
  auto* bsums = reinterpret_cast<unsigned long long*>(carve(p, sizeof(unsigned long long) * (nb + 1)));
  uint64_t edges = (uint64_t)n * d;
  CAGRA_CUDA_TRY(cudaMemsetAsync(indeg, 0, sizeof(uint32_t) * n, stream));
  CAGRA_CUDA_TRY(cudaMemsetAsync(fill, 0, sizeof(uint32_t) * n, stream));
  indeg_kernel<<<grid_for(edges, 256), 256, 0, stream>>>(d_pruned, edges, indeg);
  CAGRA_LAUNCH_CHECK();
  scan_partial_kernel<<<nb, SCAN_NT, 0, stream>>>(indeg, n, bsums);
  CAGRA_LAUNCH_CHECK();
  scan_block_sums_kernel<<<1, SCAN_NT, 0, stream>>>(bsums, nb);
  CAGRA_LAUNCH_CHECK();
  scan_final_kernel<<<nb, SCAN_NT, 0, stream>>>(indeg, n, bsums, start);
  CAGRA_LAUNCH_CHECK();
  set_total_kernel<<<1, 1, 0, stream>>>(indeg, n, start);
  CAGRA_LAUNCH_CHECK();
  reverse_scatter_kernel<<<grid_for(edges, 256), 256, 0, stream>>>(d_pruned, n, d, start, fill,
                                                                   keys);
  CAGRA_LAUNCH_CHECK();
  const uint32_t capP = next_pow2_u32(cap);
  const uint32_t rev_buf = capP <= REV_BUF / 2 ? REV_BUF : 2 * capP;
  const uint32_t warps = std::max<uint32_t>(1, std::min<uint32_t>(REV_WARPS, (96u << 10) / (8u * rev_buf)));
  size_t smem = sizeof(uint64_t) * rev_buf * warps;
  CAGRA_CUDA_TRY(cudaFuncSetAttribute(reverse_select_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = (int)std::min<uint64_t>((n + warps - 1) / warps, 148ull * 16);
  reverse_select_kernel<<<grid, warps * 32, smem, stream>>>(start, keys, n, cap,
                                                                d_rev_counts, d_rev_ids);
  CAGRA_LAUNCH_CHECK();
}

void launch_merge(const uint32_t* d_pruned, const uint32_t* d_rev_counts,
                  const uint32_t* d_rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
                  uint32_t* d_out, int* d_flag, cudaStream_t stream) {
  size_t smem = sizeof(uint32_t) * (2 * d + rev_cap) * MRG_WARPS;
  if (smem > 200 * 1024) throw UsageErr("merge_graphs: degree too large for the device kernel");
  CAGRA_CUDA_TRY(
      cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = (int)std::min<uint64_t>((n + MRG_WARPS - 1) / MRG_WARPS, 148ull * 32);
  merge_kernel<<<grid, MRG_WARPS * 32, smem, stream>>>(d_pruned, d_rev_counts, d_rev_ids, n, d,
                                                       rev_cap, d_out, d_flag);
  CAGRA_LAUNCH_CHECK();
}

}  // namespace cagra
