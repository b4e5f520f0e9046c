// permute.cu -- symmetric random relabelling of a square device CSR,
// bit-identical to the reference permute_symmetric (gen.hpp:134-155).
//
// The permutation is the reference's Fisher-Yates over the counter RNG
// (a sequential swap chain, O(n) on the host: 4M rows in a few ms).  The
// relabelling is device work: output row lengths are scattered through the
// permutation and scanned, each source row is copied (one warp per row,
// coalesced) to its new row with its columns relabelled, and a CUB segmented
// sort restores column order inside every row.  A well-formed CSR has no
// duplicate (row, col), so the result equals the reference's from_coo.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace rdmm_impl {
namespace {

uint64_t splitmix64_h(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_new_lengths(uint32_t n, const uint32_t* __restrict__ rp,
                              const uint32_t* __restrict__ perm, uint32_t* __restrict__ out_rp) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    out_rp[perm[r] + 1] = rp[r + 1] - rp[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) out_rp[0] = 0;
}

template <typename T>
__global__ void k_relabel_rows(uint32_t n, const uint32_t* __restrict__ rp,
                               const uint32_t* __restrict__ ci, const T* __restrict__ vals,
                               const uint32_t* __restrict__ perm,
                               const uint32_t* __restrict__ out_rp, uint32_t* __restrict__ keys,
                               T* __restrict__ out_vals) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < n; r += warps) {
    const uint32_t s0 = rp[r], len = rp[r + 1] - s0, d0 = out_rp[perm[r]];
    for (uint32_t t = lane; t < len; t += 32) {
      keys[d0 + t] = perm[ci[s0 + t]];
      out_vals[d0 + t] = vals[s0 + t];
    }
  }
}

int launch_grid(uint64_t work) {
  return int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(num_sms()) * 8,
                                                      ceil_div(work, 256))));
}

template <typename T>
int permute(uint32_t n, uint64_t nnz, const uint32_t* rp, const uint32_t* ci, const void* vals,
            const uint32_t* perm_host, uint32_t* out_rp, uint32_t* out_ci, void* out_vals,
            cudaStream_t s) {
  uint32_t* perm = nullptr;
  uint32_t* keys = nullptr;
  T* tv = nullptr;
  void* tmp = nullptr;
  auto release = [&] {
    for (void* p : {static_cast<void*>(perm), static_cast<void*>(keys), static_cast<void*>(tv),
                    tmp})
      if (p) cudaFreeAsync(p, s);
  };
  cudaError_t e = cudaMallocAsync(&perm, size_t(n) * 4 + 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&keys, nnz * 4 + 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tv, nnz * sizeof(T) + sizeof(T), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(perm, perm_host, size_t(n) * 4, cudaMemcpyHostToDevice, s);
  size_t tb_scan = 0, tb_sort = 0;
  if (e == cudaSuccess)
    e = cub::DeviceScan::InclusiveSum(nullptr, tb_scan, out_rp + 1, out_rp + 1, int64_t(n), s);
  if (e == cudaSuccess && nnz)
    e = cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb_sort, keys, out_ci, tv,
                                                  static_cast<T*>(out_vals), int64_t(nnz),
                                                  int64_t(n), out_rp, out_rp + 1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, std::max<size_t>(16, std::max(tb_scan, tb_sort)), s);
  if (e != cudaSuccess) {
    release();
    return fail(RDMM_ERR_CUDA, std::string("permute_symmetric: ") + cudaGetErrorString(e));
  }
  count_launch(2);
  k_new_lengths<<<launch_grid(n), 256, 0, s>>>(n, rp, perm, out_rp);
  e = cub::DeviceScan::InclusiveSum(tmp, tb_scan, out_rp + 1, out_rp + 1, int64_t(n), s);
  if (e == cudaSuccess && nnz) {
    k_relabel_rows<T><<<launch_grid(uint64_t(n) * 32), 256, 0, s>>>(
        n, rp, ci, static_cast<const T*>(vals), perm, out_rp, keys, tv);
    e = cub::DeviceSegmentedSort::StableSortPairs(tmp, tb_sort, keys, out_ci, tv,
                                                  static_cast<T*>(out_vals), int64_t(nnz),
                                                  int64_t(n), out_rp, out_rp + 1, s);
  }
  release();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(RDMM_ERR_CUDA, std::string("permute_symmetric: ") + cudaGetErrorString(e));
  return RDMM_OK;
}

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

extern "C" int rdmm_permutation(uint32_t n, uint64_t seed, uint32_t* perm) {
  if (n && !perm) return fail(RDMM_ERR_INVALID, "permutation: null output");
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) {  // gen.hpp:143-147
    const uint32_t j = uint32_t(splitmix64_h(seed * 0x2545f4914f6cdd1dull + i) % i);
    std::swap(perm[i - 1], perm[j]);
  }
  return RDMM_OK;
}

extern "C" int rdmm_permute_symmetric(uint32_t rows, uint32_t cols, uint64_t nnz,
                                      const uint32_t* row_ptr, const uint32_t* col_idx,
                                      const void* values, int dtype_bytes, uint64_t seed,
                                      uint32_t* out_row_ptr, uint32_t* out_col_idx,
                                      void* out_values, rdmm_stream_t stream) {
  if (rows != cols) return fail(RDMM_ERR_DIMENSION, "permute_symmetric expects a square matrix");
  if (dtype_bytes != 4 && dtype_bytes != 8)
    return fail(RDMM_ERR_INVALID, "permute_symmetric: dtype_bytes must be 4 or 8");
  std::vector<uint32_t> perm(rows);
  rdmm_permutation(rows, seed, perm.data());
  const cudaStream_t s = as_stream(stream);
  return dtype_bytes == 8
             ? permute<double>(rows, nnz, row_ptr, col_idx, values, perm.data(), out_row_ptr,
                               out_col_idx, out_values, s)
             : permute<float>(rows, nnz, row_ptr, col_idx, values, perm.data(), out_row_ptr,
                              out_col_idx, out_values, s);
}
