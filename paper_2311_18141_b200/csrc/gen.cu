// gen.cu -- device-side input generators, bit-identical to the reference
// host generators (/root/reference/proj/include/rdmm/gen.hpp).
//
// The reference builds R-MAT s22 ef16 in ~40 s on one core (std::sort of
// 67M tuples); here every edge is an independent counter-RNG evaluation
// (gen.hpp:67-84), the COO->CSR step (tile.hpp:70-95) is a device radix sort
// + run-length encode, so the bench's synthetic inputs are built in HBM in
// milliseconds.  Parity is pinned against oracle/_ref in tests/.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace rdmm_impl {
namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t rng_at(uint64_t seed,
                                                    uint64_t ctr) {
  return splitmix64(seed * 0x2545f4914f6cdd1dull + ctr);
}
__device__ __forceinline__ double u01(uint64_t seed, uint64_t ctr) {
  return double(rng_at(seed, ctr) >> 11) * 0x1.0p-53;
}

int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

__global__ void k_rng_at(uint64_t seed, uint64_t first, uint64_t n,
                         uint64_t* out) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    out[i] = rng_at(seed, first + i);
}

template <typename T>
__global__ void k_random_dense(uint64_t n, uint64_t seed, uint64_t mod,
                               T* out) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    out[i] = T(int(rng_at(seed, i) % mod));
}

template <typename T>
__global__ void k_real_twin(uint64_t n, uint64_t seed, T* out) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    out[i] = T(2.0 * u01(seed, i) - 1.0);
}

// gen.hpp:67-84: edge e consumes counters e*scale .. e*scale+scale-1.
__global__ void k_rmat_edges(uint64_t edges, uint32_t scale, uint64_t seed,
                             double a, double ab, double abc, uint64_t* keys) {
  for (uint64_t e = blockIdx.x * 256ull + threadIdx.x; e < edges;
       e += uint64_t(gridDim.x) * 256) {
    uint64_t r = 0, c = 0, ctr = e * scale;
    for (uint32_t level = 0; level < scale; ++level) {
      const double u = u01(seed, ctr++);
      r <<= 1;
      c <<= 1;
      if (u < a) {
      } else if (u < ab) {
        c |= 1;
      } else if (u < abc) {
        r |= 1;
      } else {
        r |= 1;
        c |= 1;
      }
    }
    keys[e] = (r << scale) | c;
  }
}

// row_ptr[r] = first unique key with row >= r (keys are row*cols + col).
__global__ void k_row_ptr(const uint64_t* keys, uint64_t nnz, uint64_t rows,
                          uint64_t cols, uint32_t* row_ptr) {
  for (uint64_t r = blockIdx.x * 256ull + threadIdx.x; r <= rows;
       r += uint64_t(gridDim.x) * 256) {
    const uint64_t target = r * cols;
    uint64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (keys[m] < target)
        lo = m + 1;
      else
        hi = m;
    }
    row_ptr[r] = uint32_t(lo);
  }
}

template <typename T>
__global__ void k_cols_vals(const uint64_t* keys, const uint32_t* counts,
                            uint64_t nnz, uint64_t cols, uint32_t* col_idx,
                            T* vals) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * 256) {
    col_idx[i] = uint32_t(keys[i] % cols);
    vals[i] = counts ? T(counts[i]) : T(1);
  }
}

// uniform_tiles: draw cell = rng::at(seed, ctr0+i) % area, paired with i.
__global__ void k_draws(uint64_t n, uint64_t seed, uint64_t ctr0,
                        uint64_t area, uint64_t* cell, uint32_t* idx) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256) {
    cell[i] = rng_at(seed, ctr0 + i) % area;
    idx[i] = uint32_t(i);
  }
}

// After a stable sort by cell: the first element of each run is the first
// draw of that cell.
__global__ void k_first_occ(const uint64_t* cell, const uint32_t* idx,
                            uint64_t n, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    if (i == 0 || cell[i] != cell[i - 1]) flag[idx[i]] = 1;
}

__global__ void k_find_T(const uint32_t* cnt, uint64_t n, uint64_t want,
                         unsigned long long* T) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    if (cnt[i] == want && (i == 0 || cnt[i - 1] < want)) *T = i + 1;
}

__global__ void k_emit_cells(const uint64_t* cell_by_idx, const uint32_t* flag,
                             const uint32_t* cnt, uint64_t T, uint64_t tk,
                             uint64_t r0, uint64_t c0, uint64_t kcols,
                             uint64_t* out) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < T;
       i += uint64_t(gridDim.x) * 256)
    if (flag[i]) {
      const uint64_t cell = cell_by_idx[i];
      out[cnt[i] - 1] = (r0 + cell / tk) * kcols + c0 + cell % tk;
    }
}

__global__ void k_unsorted_cells(uint64_t n, uint64_t seed, uint64_t ctr0,
                                 uint64_t area, uint64_t* cell) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * 256)
    cell[i] = rng_at(seed, ctr0 + i) % area;
}

int grid_for(uint64_t n) {
  return int(std::max<uint64_t>(
      1, std::min<uint64_t>(uint64_t(num_sms()) * 16, ceil_div(n, 256))));
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() {
    return static_cast<T*>(p);
  }
  cudaError_t alloc(size_t n) {
    if (p) cudaFree(p);
    p = nullptr;
    return cudaMalloc(&p, n ? n : 8);
  }
};

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

struct rdmm_gen_state {
  uint64_t rows = 0, cols = 0, nnz = 0;
  DevBuf keys;    // unique sorted keys (row*cols + col)
  DevBuf counts;  // multiplicities, or empty
  bool multiplicity = false;
};

extern "C" int rdmm_gen_rng_at(uint64_t seed, uint64_t first, uint64_t count,
                               uint64_t* out, rdmm_stream_t stream) {
  count_launch();
  if (!count) return RDMM_OK;
  k_rng_at<<<grid_for(count), 256, 0, as_stream(stream)>>>(seed, first, count,
                                                           out);
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

extern "C" int rdmm_gen_random_dense(uint64_t count, uint64_t seed,
                                     int max_value, int dtype_bytes, void* out,
                                     rdmm_stream_t stream) {
  if (!count) return RDMM_OK;
  const uint64_t mod = uint64_t(max_value + 1);
  count_launch();
  if (dtype_bytes == 8)
    k_random_dense<double><<<grid_for(count), 256, 0, as_stream(stream)>>>(
        count, seed, mod, static_cast<double*>(out));
  else
    k_random_dense<float><<<grid_for(count), 256, 0, as_stream(stream)>>>(
        count, seed, mod, static_cast<float*>(out));
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

extern "C" int rdmm_gen_real_twin(uint64_t count, uint64_t seed,
                                  int dtype_bytes, void* out,
                                  rdmm_stream_t stream) {
  if (!count) return RDMM_OK;
  count_launch();
  if (dtype_bytes == 8)
    k_real_twin<double><<<grid_for(count), 256, 0, as_stream(stream)>>>(
        count, seed, static_cast<double*>(out));
  else
    k_real_twin<float><<<grid_for(count), 256, 0, as_stream(stream)>>>(
        count, seed, static_cast<float*>(out));
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

namespace {

// Sort keys, collapse duplicates (tile.hpp:70-95) into st->keys/counts.
int sort_unique(rdmm_gen_state* st, DevBuf& keys_in, uint64_t n, int end_bit) {
  DevBuf sorted, tmp, nruns, cnts;
  RDMM_CUDA_TRY(sorted.alloc(n * 8));
  size_t tb = 0;
  RDMM_CUDA_TRY(cub::DeviceRadixSort::SortKeys(
      nullptr, tb, keys_in.as<uint64_t>(), sorted.as<uint64_t>(), int64_t(n),
      0, end_bit));
  size_t tb2 = 0;
  RDMM_CUDA_TRY(cub::DeviceRunLengthEncode::Encode(
      nullptr, tb2, sorted.as<uint64_t>(), keys_in.as<uint64_t>(),
      static_cast<uint32_t*>(nullptr), static_cast<uint64_t*>(nullptr),
      int64_t(n)));
  RDMM_CUDA_TRY(tmp.alloc(std::max(tb, tb2)));
  RDMM_CUDA_TRY(cub::DeviceRadixSort::SortKeys(
      tmp.p, tb, keys_in.as<uint64_t>(), sorted.as<uint64_t>(), int64_t(n), 0,
      end_bit));
  RDMM_CUDA_TRY(cnts.alloc(n * 4));
  RDMM_CUDA_TRY(nruns.alloc(8));
  // unique keys land back in keys_in
  RDMM_CUDA_TRY(cub::DeviceRunLengthEncode::Encode(
      tmp.p, tb2, sorted.as<uint64_t>(), keys_in.as<uint64_t>(),
      cnts.as<uint32_t>(), nruns.as<uint64_t>(), int64_t(n)));
  uint64_t nnz = 0;
  RDMM_CUDA_TRY(cudaMemcpy(&nnz, nruns.p, 8, cudaMemcpyDeviceToHost));
  st->nnz = nnz;
  std::swap(st->keys.p, keys_in.p);
  std::swap(st->counts.p, cnts.p);
  return RDMM_OK;
}

}  // namespace

extern "C" int rdmm_gen_rmat_begin(double a, double b, double c, double d,
                                   uint32_t scale, uint32_t edgefactor,
                                   uint64_t seed, int multiplicity,
                                   rdmm_gen_state** out, uint64_t* nnz) {
  *out = nullptr;
  // gen.hpp:44-51 validation
  if (a < 0 || b < 0 || c < 0 || d < 0)
    return fail(RDMM_ERR_INVALID, "R-MAT probabilities must be nonnegative");
  if (std::abs(a + b + c + d - 1.0) > 1e-9)
    return fail(RDMM_ERR_INVALID, "R-MAT probabilities must sum to 1");
  if (scale > 26)
    return fail(RDMM_ERR_INVALID,
                "R-MAT scale > 26 exceeds the desk-scale guard");
  auto* st = new rdmm_gen_state();
  st->rows = st->cols = 1ull << scale;
  st->multiplicity = multiplicity != 0;
  const uint64_t edges = uint64_t(edgefactor) << scale;
  DevBuf keys;
  if (cudaMalloc(&keys.p, std::max<uint64_t>(edges, 1) * 8) != cudaSuccess) {
    delete st;
    return fail(RDMM_ERR_CUDA, "rmat: out of device memory");
  }
  if (edges) {
    count_launch();
    k_rmat_edges<<<grid_for(edges), 256>>>(edges, scale, seed, a, a + b,
                                           a + b + c, keys.as<uint64_t>());
    int rc = sort_unique(st, keys, edges, std::max(1, int(2 * scale)));
    if (rc) {
      delete st;
      return rc;
    }
  }
  *out = st;
  *nnz = st->nnz;
  return RDMM_OK;
}

extern "C" int rdmm_gen_uniform_tiles_begin(uint64_t m, uint64_t k, uint32_t p,
                                            double d, uint64_t seed,
                                            rdmm_gen_state** out,
                                            uint64_t* nnz) {
  *out = nullptr;
  // gen.hpp:100-111 validation
  const uint32_t s = uint32_t(std::lround(std::sqrt(double(p))));
  if (uint64_t(s) * s != p)
    return fail(RDMM_ERR_INVALID, "uniform_tiles: p must be a perfect square");
  if (m % s != 0 || k % s != 0)
    return fail(RDMM_ERR_INVALID,
                "uniform_tiles: grid must divide dimensions");
  const uint64_t tm = m / s, tk = k / s, area = tm * tk;
  const double per_tile_f = d * double(tm) * double(tk);
  const uint64_t per_tile = uint64_t(std::llround(per_tile_f));
  if (std::abs(per_tile_f - double(per_tile)) > 1e-9)
    return fail(RDMM_ERR_INVALID,
                "uniform_tiles: d * tile area must be integral");
  if (per_tile > area)
    return fail(RDMM_ERR_INVALID, "uniform_tiles: density exceeds 1");
  const uint64_t total = per_tile * p;
  auto* st = new rdmm_gen_state();
  st->rows = m;
  st->cols = k;
  DevBuf all;
  if (all.alloc(std::max<uint64_t>(total, 1) * 8) != cudaSuccess) {
    delete st;
    return fail(RDMM_ERR_CUDA, "uniform_tiles: out of device memory");
  }
  uint64_t ctr = 0, written = 0;
  for (uint32_t ti = 0; ti < s; ++ti)
    for (uint32_t tj = 0; tj < s; ++tj) {
      if (per_tile == 0) continue;
      // expected duplicates ~ n^2 / (2 area); draw a margin and grow if short
      double exp_dup = double(per_tile) * double(per_tile) / (2.0 * double(area));
      uint64_t D = per_tile + uint64_t(4 * exp_dup) + 1024;
      if (per_tile * 2 > area) D = per_tile * 8 + 1024;
      for (;;) {
        DevBuf cell, idx, cell_s, idx_s, tmp, flag, cnt, Tbuf, cell_u;
        int rc = 0;
        if (cell.alloc(D * 8) || idx.alloc(D * 4) || cell_s.alloc(D * 8) ||
            idx_s.alloc(D * 4) || flag.alloc(D * 4) || cnt.alloc(D * 4) ||
            Tbuf.alloc(8) || cell_u.alloc(D * 8)) {
          delete st;
          return fail(RDMM_ERR_CUDA, "uniform_tiles: out of device memory");
        }
        count_launch();
        k_draws<<<grid_for(D), 256>>>(D, seed, ctr, area, cell.as<uint64_t>(),
                                      idx.as<uint32_t>());
        count_launch();
        k_unsorted_cells<<<grid_for(D), 256>>>(D, seed, ctr, area,
                                               cell_u.as<uint64_t>());
        size_t tb = 0, tb2 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, cell.as<uint64_t>(),
                                        cell_s.as<uint64_t>(), idx.as<uint32_t>(),
                                        idx_s.as<uint32_t>(), int64_t(D), 0,
                                        bits_for(area - 1 ? area - 1 : 1));
        cub::DeviceScan::InclusiveSum(nullptr, tb2, flag.as<uint32_t>(),
                                      cnt.as<uint32_t>(), int64_t(D));
        if (tmp.alloc(std::max(tb, tb2))) {
          delete st;
          return fail(RDMM_ERR_CUDA, "uniform_tiles: out of device memory");
        }
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, cell.as<uint64_t>(),
                                        cell_s.as<uint64_t>(), idx.as<uint32_t>(),
                                        idx_s.as<uint32_t>(), int64_t(D), 0,
                                        bits_for(area - 1 ? area - 1 : 1));
        cudaMemset(flag.p, 0, D * 4);
        count_launch();
        k_first_occ<<<grid_for(D), 256>>>(cell_s.as<uint64_t>(),
                                          idx_s.as<uint32_t>(), D,
                                          flag.as<uint32_t>());
        cub::DeviceScan::InclusiveSum(tmp.p, tb2, flag.as<uint32_t>(),
                                      cnt.as<uint32_t>(), int64_t(D));
        unsigned long long T = 0;
        cudaMemset(Tbuf.p, 0, 8);
        count_launch();
        k_find_T<<<grid_for(D), 256>>>(cnt.as<uint32_t>(), D, per_tile,
                                       static_cast<unsigned long long*>(Tbuf.p));
        if (cudaMemcpy(&T, Tbuf.p, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
          rc = RDMM_ERR_CUDA;
        if (rc) {
          delete st;
          return fail(rc, "uniform_tiles: device failure");
        }
        if (T == 0) {  // not enough distinct draws yet
          D *= 2;
          continue;
        }
        count_launch();
        k_emit_cells<<<grid_for(T), 256>>>(
            cell_u.as<uint64_t>(), flag.as<uint32_t>(), cnt.as<uint32_t>(), T,
            tk, uint64_t(ti) * tm, uint64_t(tj) * tk, k,
            all.as<uint64_t>() + written);
        ctr += T;
        written += per_tile;
        break;
      }
    }
  if (total) {
    int rc = sort_unique(st, all, total, std::max(1, bits_for(m * k - 1)));
    if (rc) {
      delete st;
      return rc;
    }
  }
  RDMM_CUDA_TRY(cudaGetLastError());
  *out = st;
  *nnz = st->nnz;
  return RDMM_OK;
}

extern "C" int rdmm_gen_finish(rdmm_gen_state* st, int dtype_bytes,
                               uint32_t* row_ptr, uint32_t* col_idx,
                               void* values) {
  if (!st) return fail(RDMM_ERR_INVALID, "gen_finish: null state");
  const uint64_t rows = st->rows, nnz = st->nnz;
  count_launch();
  k_row_ptr<<<grid_for(rows + 1), 256>>>(st->keys.as<uint64_t>(), nnz, rows,
                                         st->cols, row_ptr);
  const uint32_t* counts = st->multiplicity ? st->counts.as<uint32_t>() : nullptr;
  if (nnz) {
    count_launch();
    if (dtype_bytes == 8)
      k_cols_vals<double><<<grid_for(nnz), 256>>>(
          st->keys.as<uint64_t>(), counts, nnz, st->cols, col_idx,
          static_cast<double*>(values));
    else
      k_cols_vals<float><<<grid_for(nnz), 256>>>(
          st->keys.as<uint64_t>(), counts, nnz, st->cols, col_idx,
          static_cast<float*>(values));
  }
  cudaError_t e = cudaDeviceSynchronize();
  delete st;
  if (e != cudaSuccess)
    return fail(RDMM_ERR_CUDA, std::string("gen_finish: ") + cudaGetErrorString(e));
  return RDMM_OK;
}

extern "C" void rdmm_gen_abort(rdmm_gen_state* st) { delete st; }
