// util.cu -- device helpers behind the distributed-matrix layer:
//   tile extraction from a device-resident global CSR (distmat.hpp:265-282),
//   per-tile value sums for the order-insensitive checksum
//   (algos.hpp:634-669), and the injected straggler delay (algos.hpp:212-220).
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace rdmm_impl {
namespace {

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a,
                                                    uint32_t lo, uint32_t hi,
                                                    uint64_t key) {
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (uint64_t(a[m]) < key)
      lo = m + 1;
    else
      hi = m;
  }
  return lo;
}

// count of row r's columns inside [c0, c1)
__global__ void k_extract_count(const uint32_t* rp, const uint32_t* ci,
                                uint64_t r0, uint32_t nrows, uint64_t c0,
                                uint64_t c1, uint32_t* cnt) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += gridDim.x * blockDim.x) {
    const uint32_t s = rp[r0 + r], e = rp[r0 + r + 1];
    const uint32_t a = lower_bound_u32(ci, s, e, c0);
    const uint32_t b = lower_bound_u32(ci, a, e, c1);
    cnt[r] = b - a;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[nrows] = 0;
}

template <typename T>
__global__ void k_extract_fill(const uint32_t* rp, const uint32_t* ci,
                               const T* val, uint64_t r0, uint32_t nrows,
                               uint64_t c0, uint64_t c1,
                               const uint32_t* out_rp, uint32_t* out_ci,
                               T* out_val) {
  // a warp per row: coalesced copy of the row's in-range slice
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = w; r < nrows; r += nw) {
    const uint32_t s = rp[r0 + r], e = rp[r0 + r + 1];
    const uint32_t a = lower_bound_u32(ci, s, e, c0);
    const uint32_t o = out_rp[r], n = out_rp[r + 1] - o;
    for (uint32_t q = lane; q < n; q += 32) {
      out_ci[o + q] = uint32_t(ci[a + q] - c0);
      out_val[o + q] = val[a + q];
    }
  }
  (void)c1;
}

template <typename T>
__global__ void k_tile_sum(uint32_t rows, uint32_t cols, uint64_t ld,
                           const T* p, double* out) {
  double s = 0;
  const uint64_t total = uint64_t(rows) * cols;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += double(p[(i / cols) * ld + i % cols]);
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  s = BR(tmp).Sum(s);
  if (threadIdx.x == 0) atomicAdd(out, s);
}

struct ConcatArgs {
  const uint32_t* rp[16];
  const uint32_t* ci[16];
  const void* val[16];
  uint32_t off[16];  // column offset added to tile k's indices
  uint32_t K;
};

// The tile pointer tables are staged in shared memory: indexing the
// kernel-parameter arrays with a runtime k would copy them to local memory.
__device__ __forceinline__ void stage_args(const ConcatArgs& a, ConcatArgs& sa) {
  if (threadIdx.x < 16) {
    sa.rp[threadIdx.x] = a.rp[threadIdx.x];
    sa.ci[threadIdx.x] = a.ci[threadIdx.x];
    sa.val[threadIdx.x] = a.val[threadIdx.x];
    sa.off[threadIdx.x] = a.off[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    sa.K = a.K;
  }
  __syncthreads();
}

// Column concatenation of K same-height CSR tiles for a block of rows
// [r0, r0 + rows): the output row pointer needs no scan, because every
// tile's row pointer is already a prefix: out_rp[r] = sum_k (rp_k[r0+r] -
// rp_k[r0]).  One thread per row copies the row's K segments (adjacent rows
// are adjacent in memory, so a warp's loads and stores stay within a few
// sectors; thousands of independent rows keep the memory system busy); rows
// with a segment longer than kLongRow are listed and copied by a warp each.
constexpr uint32_t kLongRow = 32;

template <typename T>
__global__ void k_concat_short(ConcatArgs a, uint32_t r0, uint32_t rows,
                               uint32_t* __restrict__ out_rp, uint32_t* __restrict__ out_ci,
                               T* __restrict__ out_val, uint32_t* __restrict__ long_rows,
                               uint32_t* __restrict__ nlong) {
  __shared__ ConcatArgs sa;
  __shared__ uint32_t base[16];
  stage_args(a, sa);
  if (threadIdx.x < sa.K) base[threadIdx.x] = __ldg(sa.rp[threadIdx.x] + r0);
  __syncthreads();
  const uint32_t K = sa.K;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= rows;
       r += gridDim.x * blockDim.x) {
    uint32_t o = 0, maxlen = 0;
    for (uint32_t k = 0; k < K; ++k) {
      const uint32_t s0 = __ldg(sa.rp[k] + r0 + r);
      o += s0 - base[k];
      if (r < rows) maxlen = max(maxlen, __ldg(sa.rp[k] + r0 + r + 1) - s0);
    }
    out_rp[r] = o;
    if (r == rows || maxlen == 0) continue;
    if (maxlen > kLongRow) {
      long_rows[atomicAdd(nlong, 1u)] = r;
      continue;
    }
    for (uint32_t k = 0; k < K; ++k) {
      const uint32_t s0 = __ldg(sa.rp[k] + r0 + r), e0 = __ldg(sa.rp[k] + r0 + r + 1);
      const uint32_t off = sa.off[k];
      const uint32_t* ci = sa.ci[k];
      const T* val = static_cast<const T*>(sa.val[k]);
      for (uint32_t t = s0; t < e0; t += 4, o += 4) {
        uint32_t cv[4];
        T vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t + u < e0) {
            cv[u] = __ldg(ci + t + u);
            vv[u] = __ldg(val + t + u);
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t + u < e0) {
            out_ci[o + u] = cv[u] + off;
            out_val[o + u] = vv[u];
          }
      }
      o -= (4 - (e0 - s0) % 4) % 4;
    }
  }
}

template <typename T>
__global__ void k_concat_long(ConcatArgs a, uint32_t r0, const uint32_t* __restrict__ out_rp,
                              uint32_t* __restrict__ out_ci, T* __restrict__ out_val,
                              const uint32_t* __restrict__ long_rows,
                              const uint32_t* __restrict__ nlong) {
  __shared__ ConcatArgs sa;
  stage_args(a, sa);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t n = *nlong;
  for (uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < n;
       x += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t r = long_rows[x];
    uint32_t o = out_rp[r];
    for (uint32_t k = 0; k < sa.K; ++k) {
      const uint32_t s0 = __ldg(sa.rp[k] + r0 + r), e0 = __ldg(sa.rp[k] + r0 + r + 1);
      const uint32_t off = sa.off[k];
      const uint32_t* ci = sa.ci[k];
      const T* val = static_cast<const T*>(sa.val[k]);
      for (uint32_t tb = s0; tb < e0; tb += 128) {
        uint32_t cv[4];
        T vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t t = tb + 32 * u + lane;
          if (t < e0) {
            cv[u] = __ldg(ci + t);
            vv[u] = __ldg(val + t);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t t = tb + 32 * u + lane;
          if (t < e0) {
            out_ci[o + (t - s0)] = cv[u] + off;
            out_val[o + (t - s0)] = vv[u];
          }
        }
      }
      o += e0 - s0;
    }
  }
}

__global__ void k_spin(unsigned long long ns) {
  const unsigned long long t0 = clock64();
  // clock64 runs at the SM clock (~1.9 GHz); spin ~ns nanoseconds
  while (clock64() - t0 < ns * 2) {
  }
}

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

extern "C" int rdmm_csr_extract_count(const uint32_t* rp, const uint32_t* ci,
                                      uint64_t r0, uint32_t nrows, uint64_t c0,
                                      uint32_t ncols, uint32_t* out_rp,
                                      uint64_t* nnz, rdmm_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  void* cnt = scratch(4ull * (nrows + 1), 1, s);
  if (!cnt) return fail(RDMM_ERR_CUDA, "extract: scratch allocation failed");
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>(ceil_div(nrows, 256), uint64_t(num_sms()) * 8)));
  count_launch();
  k_extract_count<<<blocks, 256, 0, s>>>(rp, ci, r0, nrows, c0, c0 + ncols,
                                         static_cast<uint32_t*>(cnt));
  size_t tb = 0;
  RDMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, static_cast<uint32_t*>(cnt),
                                              out_rp, int64_t(nrows) + 1, s));
  void* tmp = scratch(tb + 16, 2, s);
  if (!tmp) return fail(RDMM_ERR_CUDA, "extract: scratch allocation failed");
  RDMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, static_cast<uint32_t*>(cnt),
                                              out_rp, int64_t(nrows) + 1, s));
  uint32_t n = 0;
  RDMM_CUDA_TRY(cudaMemcpyAsync(&n, out_rp + nrows, 4, cudaMemcpyDeviceToHost, s));
  RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  *nnz = n;
  return RDMM_OK;
}

extern "C" int rdmm_csr_extract_fill(int dtype_bytes, const uint32_t* rp,
                                     const uint32_t* ci, const void* val,
                                     uint64_t r0, uint32_t nrows, uint64_t c0,
                                     uint32_t ncols, const uint32_t* out_rp,
                                     uint32_t* out_ci, void* out_val,
                                     rdmm_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  const unsigned blocks = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>(ceil_div(nrows, 8), uint64_t(num_sms()) * 16)));
  count_launch();
  if (dtype_bytes == 8)
    k_extract_fill<double><<<blocks, 256, 0, s>>>(
        rp, ci, static_cast<const double*>(val), r0, nrows, c0, c0 + ncols,
        out_rp, out_ci, static_cast<double*>(out_val));
  else
    k_extract_fill<float><<<blocks, 256, 0, s>>>(
        rp, ci, static_cast<const float*>(val), r0, nrows, c0, c0 + ncols,
        out_rp, out_ci, static_cast<float*>(out_val));
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

extern "C" int rdmm_tile_sum(int dtype_bytes, uint32_t rows, uint32_t cols,
                             uint64_t ld, const void* p, rdmm_stream_t stream,
                             double* out) {
  cudaStream_t s = as_stream(stream);
  double* d = static_cast<double*>(scratch(64, 3, s));
  if (!d) return fail(RDMM_ERR_CUDA, "tile_sum: scratch allocation failed");
  RDMM_CUDA_TRY(cudaMemsetAsync(d, 0, 8, s));
  const uint64_t total = uint64_t(rows) * cols;
  if (total) {
    const unsigned blocks = unsigned(std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(total, 256), uint64_t(num_sms()) * 4)));
    count_launch();
    if (dtype_bytes == 8)
      k_tile_sum<double><<<blocks, 256, 0, s>>>(rows, cols, ld,
                                                static_cast<const double*>(p), d);
    else
      k_tile_sum<float><<<blocks, 256, 0, s>>>(rows, cols, ld,
                                               static_cast<const float*>(p), d);
  }
  RDMM_CUDA_TRY(cudaMemcpyAsync(out, d, 8, cudaMemcpyDeviceToHost, s));
  RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  return RDMM_OK;
}

extern "C" int rdmm_spin_delay(uint64_t ns, rdmm_stream_t stream) {
  count_launch();
  if (!ns) return RDMM_OK;
  k_spin<<<1, 1, 0, as_stream(stream)>>>(ns);
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

extern "C" int rdmm_csr_concat_cols_rows(int dtype_bytes, uint32_t r0, uint32_t rows,
                                         uint32_t K, const uint32_t* const* rp,
                                         const uint32_t* const* ci, const void* const* val,
                                         uint64_t col_stride, const uint64_t* col_offsets,
                                         uint32_t* out_rp, uint32_t* out_ci, void* out_val,
                                         rdmm_stream_t stream) {
  if (K == 0 || K > 16) return fail(RDMM_ERR_INVALID, "concat: 1..16 tiles");
  ConcatArgs a{};
  for (uint32_t k = 0; k < K; ++k) {
    a.rp[k] = rp[k];
    a.ci[k] = ci[k];
    a.val[k] = val[k];
    const uint64_t off = col_offsets ? col_offsets[k] : uint64_t(k) * col_stride;
    if (off > 0xFFFFFFFFull)
      return fail(RDMM_ERR_INVALID, "concat: concatenated columns exceed index_t");
    a.off[k] = uint32_t(off);
  }
  a.K = K;
  cudaStream_t s = as_stream(stream);
  // long-row list: count + up to `rows` entries
  auto* nlong = static_cast<uint32_t*>(scratch((size_t(rows) + 2) * 4, 4, s));
  if (!nlong) return fail(RDMM_ERR_CUDA, "concat: scratch allocation failed");
  RDMM_CUDA_TRY(cudaMemsetAsync(nlong, 0, 4, s));
  const unsigned b1 = unsigned(std::max<uint64_t>(
      1, std::min<uint64_t>(ceil_div(uint64_t(rows) + 1, 256), uint64_t(num_sms()) * 16)));
  const unsigned b2 = unsigned(num_sms()) * 8;
  count_launch(2);
  if (dtype_bytes == 8) {
    k_concat_short<double><<<b1, 256, 0, s>>>(a, r0, rows, out_rp, out_ci,
                                              static_cast<double*>(out_val), nlong + 1, nlong);
    k_concat_long<double><<<b2, 256, 0, s>>>(a, r0, out_rp, out_ci, static_cast<double*>(out_val),
                                             nlong + 1, nlong);
  } else {
    k_concat_short<float><<<b1, 256, 0, s>>>(a, r0, rows, out_rp, out_ci,
                                             static_cast<float*>(out_val), nlong + 1, nlong);
    k_concat_long<float><<<b2, 256, 0, s>>>(a, r0, out_rp, out_ci, static_cast<float*>(out_val),
                                            nlong + 1, nlong);
  }
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

extern "C" int rdmm_csr_concat_cols(int dtype_bytes, uint32_t rows, uint32_t K,
                                    const uint32_t* const* rp,
                                    const uint32_t* const* ci,
                                    const void* const* val, const uint64_t* tile_nnz,
                                    uint64_t col_stride,
                                    uint32_t* out_rp, uint32_t* out_ci,
                                    void* out_val, rdmm_stream_t stream) {
  (void)tile_nnz;
  return rdmm_csr_concat_cols_rows(dtype_bytes, 0, rows, K, rp, ci, val, col_stride, nullptr,
                                   out_rp, out_ci, out_val, stream);
}
