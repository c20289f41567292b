// Shared definitions for the B200-native CAGRA engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <stdexcept>
#include <string>

namespace cagra {

// Node id layout, /root/reference/proj/core/include/fodg/common.hpp:22-27.
constexpr uint32_t kIdMask = 0x7fffffffu;
constexpr uint32_t kParentFlag = 0x80000000u;
constexpr uint32_t kInvalidId = 0xffffffffu;
constexpr uint64_t kMaxNodes = kIdMask;

// A buffer entry packed into one 64-bit word: (dist bits << 32) | id-with-flag.
// dist >= +0 always (sum of squares from +0), so the IEEE bit pattern orders
// like the float; comparing with the flag bit masked reproduces entry_less
// (search.hpp:35-38): (dist, stripped id).  The dummy {0xffffffff, +inf}
// (search.hpp:44) is the maximum key.
constexpr uint64_t kFlagBit64 = 0x80000000ull;
constexpr uint64_t kDummyKey = 0x7f800000ffffffffull;

__host__ __device__ __forceinline__ uint32_t f2u(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
__host__ __device__ __forceinline__ float u2f(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

__host__ __device__ __forceinline__ uint64_t cmp_key(uint64_t e) { return e & ~kFlagBit64; }
__host__ __device__ __forceinline__ uint64_t make_key(float dist, uint32_t id) {
  return (static_cast<uint64_t>(f2u(dist)) << 32) | id;
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t e) {
  return static_cast<uint32_t>(e);
}
__host__ __device__ __forceinline__ float key_dist(uint64_t e) {
  return u2f(static_cast<uint32_t>(e >> 32));
}
__host__ __device__ __forceinline__ bool key_is_dummy(uint64_t e) {
  return static_cast<uint32_t>(e) == kInvalidId;
}

// splitmix64 finaliser, common.hpp:34-39.
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Knuth multiplicative hash, search.cpp:21-23.
__host__ __device__ __forceinline__ uint32_t hash_id(uint32_t id, uint32_t mask) {
  return (id * 2654435761u) & mask;
}

__host__ __device__ __forceinline__ uint32_t next_pow2_u32(uint32_t x) {
  uint32_t c = 1;
  while (c < x) c <<= 1;
  return c;
}

__host__ __device__ __forceinline__ uint32_t round_up_u32(uint32_t x, uint32_t m) {
  return (x + m - 1) / m * m;
}

#ifdef __CUDACC__
// Bitonic sort of 32*E keys held blocked in registers (index = lane*E + e).
// Bitonic MERGE of a bitonic sequence of 32*E keys (ascending then
// descending) held blocked in registers: log2(32E) compare-exchange stages.
template <int E>
__device__ __forceinline__ void warp_merge_regs(uint64_t (&v)[E], int lane) {
#pragma unroll
  for (int j = 16 * E; j > 0; j >>= 1) {
    if (j < E) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if ((e & j) == 0) {
          uint64_t a = v[e], b = v[e ^ j];
          v[e] = a < b ? a : b;
          v[e ^ j] = a < b ? b : a;
        }
      }
    } else {
      const bool lower = (lane & (j / E)) == 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], j / E);
        uint64_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
        v[e] = lower ? mn : mx;
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&v)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & j) == 0) {
            int i = lane * E + e;
            bool up = (i & k) == 0;
            uint64_t a = v[e], b = v[e ^ j];
            if ((a > b) == up) {
              v[e] = b;
              v[e ^ j] = a;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          int i = lane * E + e;
          uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], j / E);
          bool up = (i & k) == 0;
          bool lower = (i & j) == 0;
          uint64_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// The reference distance, dataset.hpp:33-43: strictly sequential fp32 chain,
// separately rounded subtract, multiply and add (no FMA contraction).
__device__ __forceinline__ float seq_step(float acc, float a, float b) {
  float diff = __fsub_rn(a, b);
  return __fadd_rn(acc, __fmul_rn(diff, diff));
}
// The sequential chain over a whole row (squared_l2, dataset.hpp:38-41) with
// 128-bit loads: rows are 16-byte aligned with a stride that is a multiple of
// 4 floats; the additions stay in index order, so the result is bit-equal.
__device__ __forceinline__ float seq_dist(const float* __restrict__ x, const float* __restrict__ q,
                                          uint32_t dim) {
  float acc = 0.0f;
  uint32_t i = 0;
  for (; i + 4 <= dim; i += 4) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(x + i));
    const float4 b = __ldg(reinterpret_cast<const float4*>(q + i));
    acc = seq_step(acc, a.x, b.x);
    acc = seq_step(acc, a.y, b.y);
    acc = seq_step(acc, a.z, b.z);
    acc = seq_step(acc, a.w, b.w);
  }
  for (; i < dim; ++i) acc = seq_step(acc, __ldg(x + i), __ldg(q + i));
  return acc;
}
// U independent sequential chains (U rows against one query) interleaved:
// U x the arithmetic ILP and U x the loads in flight of seq_dist; each chain
// keeps index order, so every result is bit-equal to seq_dist.
template <int U>
__device__ __forceinline__ void seq_dist_multi(const float* const (&x)[U],
                                               const float* __restrict__ q, uint32_t dim,
                                               float (&acc)[U]) {
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0f;
  uint32_t i = 0;
#pragma unroll 2
  for (; i + 4 <= dim; i += 4) {
    const float4 b = __ldg(reinterpret_cast<const float4*>(q + i));
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(x[u] + i));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u] = seq_step(acc[u], a[u].x, b.x);
      acc[u] = seq_step(acc[u], a[u].y, b.y);
      acc[u] = seq_step(acc[u], a[u].z, b.z);
      acc[u] = seq_step(acc[u], a[u].w, b.w);
    }
  }
  for (; i < dim; ++i) {
    const float b = __ldg(q + i);
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = seq_step(acc[u], __ldg(x[u] + i), b);
  }
}
#endif

// ---- host-side error types; capi.cu maps them to status codes ----
struct UsageErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LogicErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace cagra

#define CAGRA_CUDA_TRY(expr)                                                         \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      throw ::cagra::CudaErr(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
    }                                                                                \
  } while (0)

#define CAGRA_LAUNCH_CHECK() CAGRA_CUDA_TRY(cudaGetLastError())
