// Host-side helpers shared by the C-ABI sources (capi.cu, multi.cu): status
// mapping, owning device buffers, streams/events, device selection, row
// uploads, and the device optimize pipeline.
#pragma once

#include <cuda_runtime.h>

#include <new>
#include <stdexcept>
#include <string>

#include "cagra/capi.h"
#include "common.cuh"
#include "kernels.hpp"

namespace cagra {

// thread-local message of the last failing C-ABI call (cagra_last_error)
std::string& last_error_slot();

template <class F>
int guarded(F&& f) {
  std::string& err = last_error_slot();
  try {
    f();
    return CAGRA_OK;
  } catch (const UsageErr& e) {
    err = e.what();
    return CAGRA_ERR_USAGE;
  } catch (const FormatErr& e) {
    err = e.what();
    return CAGRA_ERR_FORMAT;
  } catch (const LogicErr& e) {
    err = e.what();
    return CAGRA_ERR_LOGIC;
  } catch (const CudaErr& e) {
    err = e.what();
    return CAGRA_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    err = "host allocation failed";
    return CAGRA_ERR_CUDA;
  } catch (const std::exception& e) {
    err = e.what();
    return CAGRA_ERR_LOGIC;
  }
}

inline int resolve_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw CudaErr("no CUDA device available (the B200 engine has no CPU path)");
  int dev = device < 0 ? 0 : device;
  if (dev >= count) throw UsageErr("device index out of range");
  return dev;
}

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    CAGRA_CUDA_TRY(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Owning device allocation.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t b) { alloc(b); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  ~DBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b == 0) b = 16;
    CAGRA_CUDA_TRY(cudaMalloc(&p, b));
    bytes = b;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct Stream {
  cudaStream_t s = nullptr;
  Stream() { CAGRA_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s) cudaStreamDestroy(s);
  }
  void sync() { CAGRA_CUDA_TRY(cudaStreamSynchronize(s)); }
};

struct Event {
  cudaEvent_t e = nullptr;
  Event() { CAGRA_CUDA_TRY(cudaEventCreate(&e)); }
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
};

inline int sm_count_of(int dev) {
  int sms = 0;
  CAGRA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

// device row stride (floats): dim rounded up to 4 (16-byte rows for float4 gathers)
inline uint32_t row_stride(uint32_t dim) { return round_up_u32(dim, 4); }

// rows x dim host/device floats -> rows x ld device floats (zero padded)
inline void upload_rows(float* dst, const float* src, uint64_t rows, uint32_t dim, uint32_t ld,
                        cudaStream_t s, bool src_is_device = false) {
  if (rows == 0) return;
  cudaMemcpyKind kind = src_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (ld == dim) {
    CAGRA_CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(float) * rows * dim, kind, s));
  } else {
    CAGRA_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(float) * rows * ld, s));
    CAGRA_CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(float) * ld, src, sizeof(float) * dim,
                                     sizeof(float) * dim, rows, kind, s));
  }
}

inline void read_flag(int* d_flag, int* h, cudaStream_t s) {
  CAGRA_CUDA_TRY(cudaMemcpyAsync(h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CAGRA_CUDA_TRY(cudaStreamSynchronize(s));
}

// ---- optimize pipeline on device (graph_opt.cpp:211-246), capi.cu ----
struct OptOut {
  float ms[5] = {0, 0, 0, 0, 0};
};
void optimize_device(const uint32_t* d_knn, const float* d_dists, uint32_t n, uint32_t deg,
                     uint32_t d, bool reorder, bool add_reverse, uint32_t* d_out,
                     cudaStream_t s, OptOut* times);

}  // namespace cagra
