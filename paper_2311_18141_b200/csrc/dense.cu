// dense.cu -- c += x for row-major tiles (reference dense_add_into,
// /root/reference/proj/include/rdmm/tile.hpp:300-307).  Streaming, HBM-bound:
// 16-B vector loads/stores when aligned, grid sized to the SM count.
#include <algorithm>

#include "common.cuh"

namespace rdmm_impl {
namespace {

template <typename T, typename V>
__global__ void __launch_bounds__(256)
    dense_add_vec(uint32_t rows, uint32_t vcols, V* __restrict__ c,
                  uint64_t ldcv, const V* __restrict__ x, uint64_t ldxv) {
  constexpr int L = sizeof(V) / sizeof(T);
  const uint64_t total = uint64_t(rows) * vcols;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * 256) {
    const uint64_t r = i / vcols, q = i % vcols;
    V a = c[r * ldcv + q];
    const V b = __ldg(x + r * ldxv + q);
    T* pa = reinterpret_cast<T*>(&a);
    const T* pb = reinterpret_cast<const T*>(&b);
#pragma unroll
    for (int l = 0; l < L; ++l) pa[l] = pa[l] + pb[l];
    c[r * ldcv + q] = a;
  }
}

template <typename T, typename V>
int dense_add(uint32_t rows, uint32_t cols, T* c, uint64_t ldc, const T* x,
              uint64_t ldx, rdmm_stream_t stream) {
  if (ldc < cols || ldx < cols)
    return fail(RDMM_ERR_DIMENSION, "dense_add_into: leading dimension");
  if (rows == 0 || cols == 0) return RDMM_OK;
  constexpr int L = sizeof(V) / sizeof(T);
  const bool vec = cols % L == 0 && ldc % L == 0 && ldx % L == 0 &&
                   reinterpret_cast<uintptr_t>(c) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(x) % 16 == 0;
  const uint64_t units = uint64_t(rows) * (vec ? cols / L : cols);
  const int blocks =
      int(std::min<uint64_t>(uint64_t(num_sms()) * 8, ceil_div(units, 256)));
  cudaStream_t s = as_stream(stream);
  KernelTimer timer(s, 3);
  count_launch();
  if (vec)
    dense_add_vec<T, V><<<blocks, 256, 0, s>>>(
        rows, cols / L, reinterpret_cast<V*>(c), ldc / L,
        reinterpret_cast<const V*>(x), ldx / L);
  else
    dense_add_vec<T, T><<<blocks, 256, 0, s>>>(rows, cols, c, ldc, x, ldx);
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

}  // namespace
}  // namespace rdmm_impl

extern "C" int rdmm_dense_add_into_f32(uint32_t rows, uint32_t cols, float* c,
                                       uint64_t ldc, const float* x,
                                       uint64_t ldx, rdmm_stream_t stream) {
  return rdmm_impl::dense_add<float, float4>(rows, cols, c, ldc, x, ldx,
                                             stream);
}

extern "C" int rdmm_dense_add_into_f64(uint32_t rows, uint32_t cols, double* c,
                                       uint64_t ldc, const double* x,
                                       uint64_t ldx, rdmm_stream_t stream) {
  return rdmm_impl::dense_add<double, double2>(rows, cols, c, ldc, x, ldx,
                                               stream);
}
