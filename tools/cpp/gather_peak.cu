// Random row-gather ceiling on this B200: the access pattern of the search
// kernel's distance phase (whole fp32 rows of `dim` floats at uniformly random
// ids, float4 loads by 8-lane teams) with no visited/merge work around it.
// Prints GB/s of row bytes delivered for several dataset sizes and
// rows-in-flight settings, so the search roofline can be stated against the
// ceiling of its own access pattern, not only the sequential copy peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peak gather_peak.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return (uint32_t)x;
}

// TEAM lanes per row, C float4 per lane (dim = 4*TEAM*C), U rows in flight per team
template <int TEAM, int C, int U>
__global__ void __launch_bounds__(256) gather_kernel(const float4* __restrict__ data, uint32_t n,
                                                     uint32_t rows_per_team, uint64_t seed,
                                                     float* out) {
  const int lt = threadIdx.x % TEAM;
  const uint64_t team = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / TEAM;
  const int ld4 = TEAM * C;
  float acc = 0.f;
  for (uint32_t r = 0; r < rows_per_team; r += U) {
    float4 v[U][C];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t id = mix(seed ^ (team * 0x9E3779B97F4A7C15ULL + r + u)) % n;
      const float4* row = data + (size_t)id * ld4;
#pragma unroll
      for (int c = 0; c < C; ++c) v[u][c] = __ldg(row + lt + TEAM * c);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) acc += v[u][c].x * v[u][c].y + v[u][c].z * v[u][c].w;
  }
  if (acc == 12345.678f) out[0] = acc;  // keep the loads alive
}

template <int U>
double run(const float4* d, uint32_t n, int grid, uint32_t rows, float* out) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int w = 0; w < 2; ++w) gather_kernel<8, 3, U><<<grid, 256>>>(d, n, rows, w + 1, out);
  CK(cudaEventRecord(a));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) gather_kernel<8, 3, U><<<grid, 256>>>(d, n, rows, 100 + r, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  const double bytes = (double)grid * 256 / 8 * rows * 384.0 * reps;
  return bytes / (ms * 1e-3) / 1e9;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint32_t sizes[] = {1000000u, 10000000u, 40000000u};
  float* out; CK(cudaMalloc(&out, 4));
  for (uint32_t n : sizes) {
    float4* d; size_t bytes = (size_t)n * 384;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemset(d, 0, bytes));
    for (int ctas = 4; ctas <= 8; ctas += 4) {
      int grid = sms * ctas;
      uint32_t rows = 6144;
      printf("n=%9u (%.2f GB) ctas/SM=%d  U=1 %7.0f  U=2 %7.0f  U=3 %7.0f  U=4 %7.0f  U=6 %7.0f GB/s\n",
             n, bytes / 1e9, ctas, run<1>(d, n, grid, rows, out), run<2>(d, n, grid, rows, out),
             run<3>(d, n, grid, rows, out), run<4>(d, n, grid, rows, out),
             run<6>(d, n, grid, rows, out));
    }
    CK(cudaFree(d));
  }
  return 0;
}
