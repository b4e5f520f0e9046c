// common.cuh -- shared helpers for the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

#include "rdmm_cuda.h"

namespace rdmm_impl {

// Thread-local last error (rdmm_last_error); set by every failing entry point.
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define RDMM_CUDA_TRY(expr)                                                \
  do {                                                                     \
    cudaError_t e_ = (expr);                                               \
    if (e_ != cudaSuccess)                                                 \
      return ::rdmm_impl::fail(RDMM_ERR_CUDA, std::string(#expr ": ") +    \
                                                  cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t as_stream(rdmm_stream_t s) {
  return reinterpret_cast<cudaStream_t>(s);
}

inline int num_sms() {
  static thread_local int dev_cached = -1, sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dev_cached = dev;
  }
  return sms;
}

// Grow-only scratch per (device, stream, slot) used when the caller passes no
// workspace.  Reuse is stream-ordered (all users of a buffer run on its
// stream); growth frees/allocates on the stream (cudaFreeAsync /
// cudaMallocAsync), so no host synchronisation is needed.
void* scratch(size_t bytes, int slot, cudaStream_t stream);

// Launch accounting for bench.py's gpu_launches claim (our kernels only).
void count_launch(unsigned n = 1);

// Optional device timing of the hot kernels (CUDA events on the launching
// stream around each launch; rdmm_kernel_timing_* in the C-ABI).
struct KernelTimer {
  cudaEvent_t start = nullptr;
  cudaStream_t stream = nullptr;
  int kind = 0;
  KernelTimer(cudaStream_t s, int kind);
  ~KernelTimer();
};

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) {
  return (a + b - 1) / b;
}

}  // namespace rdmm_impl
