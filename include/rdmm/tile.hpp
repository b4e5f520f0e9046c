// rdmm/tile.hpp -- tiles and per-tile kernels of the B200 build.
//
// Drop-in for /root/reference/proj/include/rdmm/tile.hpp: the host tile
// types (CsrTile, DenseTile, views, FlopMeter) keep the reference's layout
// and semantics (tile.hpp:17-168) for building inputs and gathering results;
// the hot path runs on DEVICE tiles (DevCsrTile / DevDenseTile and their
// views) through the C-ABI in rdmm_cuda.h (the sm_100a kernels).  The kernel
// entry points keep the reference names (spmm_local, spgemm_local,
// spgemm_flops, csr_add, dense_add_into) and raise the same exceptions.
#ifndef RDMM_B200_TILE_HPP
#define RDMM_B200_TILE_HPP

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "rdmm_cuda.h"

// Records a failure for rdmm_last_error() from layers above the C-ABI.
extern "C" int rdmm_impl_fail(int code, const char* msg);

namespace rdmm {

using index_t = std::uint32_t;  // tile.hpp:17

class dimension_error : public std::runtime_error {  // tile.hpp:19-23
 public:
  explicit dimension_error(const std::string& w) : std::runtime_error(w) {}
};
class fabric_error : public std::runtime_error {  // fabric.hpp:38-41
 public:
  explicit fabric_error(const std::string& w) : std::runtime_error(w) {}
};
class heap_exhausted_error : public fabric_error {  // fabric.hpp:43-53
 public:
  heap_exhausted_error(std::size_t requested, std::size_t remaining,
                       const std::string& w)
      : fabric_error(w), requested(requested), remaining(remaining) {}
  std::size_t requested;
  std::size_t remaining;
};
class queue_full_error : public fabric_error {  // fabric.hpp:55-60
 public:
  explicit queue_full_error(const std::string& w) : fabric_error(w) {}
};
class protocol_error : public fabric_error {  // algos.hpp:98-101
 public:
  explicit protocol_error(const std::string& w) : fabric_error(w) {}
};
class cuda_error : public std::runtime_error {
 public:
  explicit cuda_error(const std::string& w) : std::runtime_error(w) {}
};

// Map a C-ABI status to the reference exception taxonomy.
inline void check(int rc, const char* what = "", std::size_t requested = 0,
                  std::size_t remaining = 0) {
  if (rc == RDMM_OK) return;
  std::string msg = std::string(what) + (what[0] ? ": " : "") + rdmm_last_error();
  switch (rc) {
    case RDMM_ERR_DIMENSION: throw dimension_error(msg);
    case RDMM_ERR_HEAP_EXHAUSTED: throw heap_exhausted_error(requested, remaining, msg);
    case RDMM_ERR_QUEUE_FULL: throw queue_full_error(msg);
    case RDMM_ERR_PROTOCOL: throw protocol_error(msg);
    case RDMM_ERR_FABRIC: throw fabric_error(msg);
    case RDMM_ERR_INVALID: throw std::invalid_argument(msg);
    default: throw cuda_error(msg);
  }
}

template <typename T>
constexpr int dtype_bytes() {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "float or double tiles");
  return int(sizeof(T));
}

// tile.hpp:25-41
struct FlopMeter {
  std::uint64_t flops = 0;
  std::uint64_t output_nnz = 0;
  double cf() const {
    return output_nnz == 0 ? 0.0 : double(flops) / double(output_nnz);
  }
  FlopMeter& operator+=(const FlopMeter& o) {
    flops += o.flops;
    output_nnz += o.output_nnz;
    return *this;
  }
};

// ------------------------------------------------------------ host tiles

template <typename T>
struct DenseTile {  // tile.hpp:43-55
  index_t rows = 0, cols = 0;
  std::vector<T> values;  // row-major
  DenseTile() = default;
  DenseTile(index_t r, index_t c) : rows(r), cols(c), values(std::size_t(r) * c) {}
  T& at(index_t r, index_t c) { return values[std::size_t(r) * cols + c]; }
  const T& at(index_t r, index_t c) const { return values[std::size_t(r) * cols + c]; }
};

template <typename T>
struct CsrTile {  // tile.hpp:57-118
  index_t rows = 0, cols = 0;
  std::vector<index_t> row_ptr;
  std::vector<index_t> col_idx;
  std::vector<T> values;
  CsrTile() = default;
  CsrTile(index_t r, index_t c) : rows(r), cols(c), row_ptr(r + 1, 0) {}
  std::uint64_t nnz() const { return col_idx.size(); }

  static CsrTile from_coo(index_t rows, index_t cols,
                          std::vector<std::tuple<index_t, index_t, T>> coo) {
    std::sort(coo.begin(), coo.end(), [](const auto& a, const auto& b) {
      return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                              : std::get<1>(a) < std::get<1>(b);
    });
    CsrTile t(rows, cols);
    for (std::size_t s = 0; s < coo.size();) {
      const index_t r = std::get<0>(coo[s]), c = std::get<1>(coo[s]);
      T sum = std::get<2>(coo[s]);
      std::size_t e = s + 1;
      for (; e < coo.size() && std::get<0>(coo[e]) == r && std::get<1>(coo[e]) == c; ++e)
        sum += std::get<2>(coo[e]);
      t.col_idx.push_back(c);
      t.values.push_back(sum);
      t.row_ptr[r + 1]++;
      s = e;
    }
    for (index_t r = 0; r < rows; ++r) t.row_ptr[r + 1] += t.row_ptr[r];
    return t;
  }

  DenseTile<T> to_dense() const {
    DenseTile<T> d(rows, cols);
    for (index_t r = 0; r < rows; ++r)
      for (index_t s = row_ptr[r]; s < row_ptr[r + 1]; ++s) d.at(r, col_idx[s]) = values[s];
    return d;
  }

  bool well_formed() const {
    if (row_ptr.size() != std::size_t(rows) + 1) return false;
    if (row_ptr[0] != 0 || row_ptr[rows] != col_idx.size()) return false;
    if (col_idx.size() != values.size()) return false;
    for (index_t r = 0; r < rows; ++r) {
      if (row_ptr[r] > row_ptr[r + 1]) return false;
      for (index_t s = row_ptr[r]; s < row_ptr[r + 1]; ++s) {
        if (col_idx[s] >= cols) return false;
        if (s > row_ptr[r] && col_idx[s] <= col_idx[s - 1]) return false;
      }
    }
    return true;
  }
};

// ------------------------------------------------------------ device tiles

// Owning device allocation on one fabric rank's GPU (stream-ordered pool
// memory).  Aliases (owned=false) point into a fabric heap without owning.
class DevBuffer {
 public:
  DevBuffer() = default;
  DevBuffer(rdmm_fabric* f, std::uint32_t rank, std::uint64_t bytes, rdmm_stream_t s)
      : f_(f), rank_(rank), stream_(s), owned_(true) {
    check(rdmm_dev_alloc(f, rank, bytes, s, &p_), "dev_alloc");
  }
  static DevBuffer alias(void* p) {
    DevBuffer b;
    b.p_ = p;
    return b;
  }
  DevBuffer(DevBuffer&& o) noexcept { *this = std::move(o); }
  DevBuffer& operator=(DevBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      f_ = o.f_;
      rank_ = o.rank_;
      p_ = o.p_;
      stream_ = o.stream_;
      owned_ = o.owned_;
      o.p_ = nullptr;
      o.owned_ = false;
    }
    return *this;
  }
  DevBuffer(const DevBuffer&) = delete;
  DevBuffer& operator=(const DevBuffer&) = delete;
  ~DevBuffer() { reset(); }
  // The stream the buffer is released on (its last consumer).
  void release_on(rdmm_stream_t s) { stream_ = s; }
  void reset() {
    if (owned_ && p_) rdmm_dev_free(f_, rank_, p_, stream_);
    p_ = nullptr;
    owned_ = false;
  }
  void* get() const { return p_; }
  bool owned() const { return owned_; }

 private:
  rdmm_fabric* f_ = nullptr;
  std::uint32_t rank_ = 0;
  void* p_ = nullptr;
  rdmm_stream_t stream_ = nullptr;
  bool owned_ = false;
};

template <typename T>
struct DevCsrView {  // CsrView (tile.hpp:122-138) with device pointers
  index_t rows = 0, cols = 0;
  std::uint64_t nnz = 0;
  const index_t* row_ptr = nullptr;
  const index_t* col_idx = nullptr;
  const T* values = nullptr;
};

template <typename T>
struct DevDenseView {  // DenseView (tile.hpp:140-152), leading dimension ld
  index_t rows = 0, cols = 0;
  std::uint64_t ld = 0;
  T* values = nullptr;
};

template <typename T>
struct DevDenseConstView {
  index_t rows = 0, cols = 0;
  std::uint64_t ld = 0;
  const T* values = nullptr;
  DevDenseConstView() = default;
  DevDenseConstView(index_t r, index_t c, std::uint64_t l, const T* v)
      : rows(r), cols(c), ld(l), values(v) {}
  DevDenseConstView(const DevDenseView<T>& v)
      : rows(v.rows), cols(v.cols), ld(v.ld), values(v.values) {}
};

template <typename T>
struct DevCsrTile {
  index_t rows = 0, cols = 0;
  std::uint64_t nnz = 0;
  DevBuffer row_ptr, col_idx, values;
  DevCsrView<T> view() const {
    return {rows, cols, nnz, static_cast<const index_t*>(row_ptr.get()),
            static_cast<const index_t*>(col_idx.get()), static_cast<const T*>(values.get())};
  }
  void release_on(rdmm_stream_t s) {
    row_ptr.release_on(s);
    col_idx.release_on(s);
    values.release_on(s);
  }
};

template <typename T>
struct DevDenseTile {
  index_t rows = 0, cols = 0;
  DevBuffer buf;
  DevDenseView<T> view() const { return {rows, cols, cols, static_cast<T*>(buf.get())}; }
  DevDenseConstView<T> cview() const {
    return {rows, cols, cols, static_cast<const T*>(buf.get())};
  }
  void release_on(rdmm_stream_t s) { buf.release_on(s); }
};

// ------------------------------------------------------------ kernels

// c += a*b (tile.hpp:170-188) on `stream`.  c_zero: c is known all-zero
// (written, never read).  flops == 2*nnz(a)*b.cols.
template <typename T>
FlopMeter spmm_local(DevCsrView<T> a, DevDenseConstView<T> b, DevDenseView<T> c,
                     rdmm_stream_t stream, bool c_zero = false, bool atomic = false) {
  if (a.cols != b.rows || c.rows != a.rows || c.cols != b.cols)
    throw dimension_error("spmm_local: dimension mismatch");
  std::uint64_t fl = 0;
  check(rdmm_spmm_csr_ex(dtype_bytes<T>(), a.rows, a.cols, b.cols, a.nnz, a.row_ptr,
                         a.col_idx, a.values, b.values, b.ld, c.values, c.ld,
                         (c_zero ? RDMM_SPMM_C_ZERO : 0u) | (atomic ? RDMM_SPMM_ATOMIC : 0u),
                         nullptr, 0, stream, &fl),
        "spmm_local");
  FlopMeter m;
  m.flops = fl;
  m.output_nnz = std::uint64_t(c.rows) * c.cols;
  return m;
}

// Fused stationary-C product of one tile column: c += sum_k a_k * b_k in ONE
// pass over c (the K A tiles are concatenated side by side on the device).
// The tiles come in accumulation order with their natural k index `knat`;
// concatenated column indices are the natural ones (knat[k] * col_stride +
// c), so when the B tiles form one contiguous panel in natural order
// (DistDense's placement) B is read directly, else through the segment
// table.  `atomic`: accumulate into c with red.global.add (narrow rows).
template <typename T>
FlopMeter spmm_fused(rdmm_fabric* f, std::uint32_t rank, const std::vector<DevCsrView<T>>& a,
                     const std::vector<DevDenseConstView<T>>& b,
                     const std::vector<std::uint32_t>& knat, std::uint64_t col_stride,
                     DevDenseView<T> c, rdmm_stream_t stream, bool c_zero = false,
                     bool atomic = false) {
  const std::size_t K = a.size();
  if (K == 0 || b.size() != K || K > 16 || knat.size() != K)
    throw std::invalid_argument("spmm_fused: 1..16 tiles");
  if (K == 1) return spmm_local<T>(a[0], b[0], c, stream, c_zero, atomic);
  std::uint64_t nnz = 0;
  std::uint32_t kmax = 0;
  for (auto k : knat) kmax = std::max(kmax, k);
  std::vector<const index_t*> rp(K), ci(K);
  std::vector<const void*> vv(K);
  std::vector<const void*> bs(kmax + 1, nullptr);
  std::vector<std::uint64_t> coff(K);
  for (std::size_t k = 0; k < K; ++k) {
    if (a[k].rows != c.rows || a[k].cols != b[k].rows || b[k].cols != c.cols ||
        b[k].ld != b[0].ld || b[k].rows > col_stride || bs[knat[k]])
      throw dimension_error("spmm_fused: dimension mismatch");
    nnz += a[k].nnz;
    rp[k] = a[k].row_ptr;
    ci[k] = a[k].col_idx;
    vv[k] = a[k].values;
    bs[knat[k]] = b[k].values;
    coff[k] = std::uint64_t(knat[k]) * col_stride;
  }
  // one contiguous panel over natural k = 0..kmax (every segment present)?
  bool panel = true;
  for (std::size_t k = 0; k <= kmax; ++k)
    panel &= bs[k] != nullptr && static_cast<const T*>(bs[k]) ==
                                     static_cast<const T*>(bs[0]) + k * col_stride * b[0].ld;
  DevBuffer crp(f, rank, (std::uint64_t(c.rows) + 1) * sizeof(index_t), stream);
  DevBuffer cci(f, rank, std::max<std::uint64_t>(nnz, 1) * sizeof(index_t), stream);
  DevBuffer cvv(f, rank, std::max<std::uint64_t>(nnz, 1) * sizeof(T), stream);
  check(rdmm_csr_concat_cols_rows(dtype_bytes<T>(), 0, c.rows, std::uint32_t(K), rp.data(),
                                  ci.data(), vv.data(), col_stride, coff.data(),
                                  static_cast<index_t*>(crp.get()),
                                  static_cast<index_t*>(cci.get()), cvv.get(), stream),
        "spmm_fused concat");
  const unsigned flags = (c_zero ? RDMM_SPMM_C_ZERO : 0u) | (atomic ? RDMM_SPMM_ATOMIC : 0u);
  std::uint64_t fl = 0;
  if (panel) {
    check(rdmm_spmm_csr_ex(dtype_bytes<T>(), c.rows, std::uint32_t(col_stride * (kmax + 1)),
                           c.cols, nnz, static_cast<const index_t*>(crp.get()),
                           static_cast<const index_t*>(cci.get()), cvv.get(), bs[0], b[0].ld,
                           c.values, c.ld, flags, nullptr, 0, stream, &fl),
          "spmm_fused");
  } else {
    for (auto& p : bs)  // unused segments: any valid pointer (never indexed)
      if (!p) p = b[0].values;
    check(rdmm_spmm_csr_seg(dtype_bytes<T>(), c.rows, c.cols, nnz,
                            static_cast<const index_t*>(crp.get()),
                            static_cast<const index_t*>(cci.get()), cvv.get(), bs.data(),
                            kmax + 1, std::uint32_t(col_stride), b[0].ld, c.values, c.ld, flags,
                            nullptr, 0, stream, &fl),
          "spmm_fused");
  }
  FlopMeter m;
  m.flops = fl;
  m.output_nnz = std::uint64_t(c.rows) * c.cols;
  return m;  // the concat buffers are released stream-ordered after the kernel
}

// Row-block pipelined form of spmm_fused.  The rows of C are cut at
// `bounds` (bounds[0] = 0 ... bounds.back() = c.rows); for block b,
// before_concat(b, side) makes the side stream wait for whatever feeds the
// block (e.g. the copy-engine slices of remote A tiles), the K-tile
// concatenation of the block's rows (rdmm_csr_concat_cols_rows) runs on
// `side` while block b-1 multiplies on `stream`, and the block's SpMM reads
// its nonzero count on the device (no host round trip).  Two concat buffers
// alternate.  Same result as spmm_fused (concatenation in the tiles' order).
//
// The tiles come in accumulation order (the reference's offset order) with
// their natural k index `knat`: concatenated column indices are the natural
// ones (knat[k] * col_stride + c), so when the B tiles form one contiguous
// panel in natural order (DistDense places a rank's tiles of a column back
// to back) the SpMM reads B directly, else through the segment table.
template <typename T, typename BeforeConcat>
FlopMeter spmm_fused_rows(rdmm_fabric* f, std::uint32_t rank,
                          const std::vector<DevCsrView<T>>& a,
                          const std::vector<DevDenseConstView<T>>& b,
                          const std::vector<std::uint32_t>& knat, std::uint64_t col_stride,
                          DevDenseView<T> c, rdmm_stream_t stream, rdmm_stream_t side,
                          bool c_zero, const std::vector<std::uint32_t>& bounds,
                          BeforeConcat&& before_concat) {
  const std::size_t K = a.size();
  if (K == 0 || b.size() != K || K > 16) throw std::invalid_argument("spmm_fused_rows: 1..16 tiles");
  if (bounds.size() < 2 || bounds.front() != 0 || bounds.back() != c.rows)
    throw std::invalid_argument("spmm_fused_rows: bad row bounds");
  std::uint64_t nnz = 0;
  std::vector<const index_t*> rp(K), ci(K);
  std::vector<const void*> vv(K), bs(K, nullptr);
  std::vector<std::uint64_t> coff(K);
  if (knat.size() != K) throw std::invalid_argument("spmm_fused_rows: knat size");
  for (std::size_t k = 0; k < K; ++k) {
    if (a[k].rows != c.rows || a[k].cols != b[k].rows || b[k].cols != c.cols ||
        b[k].ld != b[0].ld || b[k].rows > col_stride || knat[k] >= K || bs[knat[k]])
      throw dimension_error("spmm_fused_rows: dimension mismatch");
    nnz += a[k].nnz;
    rp[k] = a[k].row_ptr;
    ci[k] = a[k].col_idx;
    vv[k] = a[k].values;
    bs[knat[k]] = b[k].values;
    coff[k] = std::uint64_t(knat[k]) * col_stride;
  }
  // one contiguous B panel in natural order?
  bool panel = true;
  for (std::size_t k = 1; k < K; ++k)
    panel &= static_cast<const T*>(bs[k]) ==
             static_cast<const T*>(bs[0]) + std::uint64_t(k) * col_stride * b[0].ld;
  FlopMeter m;
  m.flops = 2ull * nnz * c.cols;
  m.output_nnz = std::uint64_t(c.rows) * c.cols;
  const std::size_t blocks = bounds.size() - 1;
  std::uint32_t rbmax = 0;
  for (std::size_t q = 0; q < blocks; ++q) rbmax = std::max(rbmax, bounds[q + 1] - bounds[q]);
  DevBuffer rpb[2], cib[2], vvb[2];
  const std::size_t nbuf = blocks > 1 ? 2 : 1;
  for (std::size_t q = 0; q < nbuf; ++q) {
    rpb[q] = DevBuffer(f, rank, (std::uint64_t(rbmax) + 1) * sizeof(index_t), stream);
    cib[q] = DevBuffer(f, rank, std::max<std::uint64_t>(nnz, 1) * sizeof(index_t), stream);
    vvb[q] = DevBuffer(f, rank, std::max<std::uint64_t>(nnz, 1) * sizeof(T), stream);
  }
  // the side stream starts after the buffers exist (allocated on `stream`)
  void* ready = nullptr;
  check(rdmm_event_record(stream, &ready), "spmm_fused_rows");
  check(rdmm_event_wait(ready, side), "spmm_fused_rows");
  rdmm_event_destroy(ready);
  std::vector<void*> spmm_done(blocks, nullptr);
  for (std::size_t bk = 0; bk < blocks; ++bk) {
    const std::size_t q = bk % nbuf;
    const std::uint32_t r0 = bounds[bk], nr = bounds[bk + 1] - bounds[bk];
    before_concat(bk, side);
    if (nr == 0) continue;
    if (bk >= nbuf && spmm_done[bk - nbuf])
      check(rdmm_event_wait(spmm_done[bk - nbuf], side), "spmm_fused_rows");
    check(rdmm_csr_concat_cols_rows(dtype_bytes<T>(), r0, nr, std::uint32_t(K), rp.data(),
                                    ci.data(), vv.data(), col_stride, coff.data(),
                                    static_cast<index_t*>(rpb[q].get()),
                                    static_cast<index_t*>(cib[q].get()), vvb[q].get(), side),
          "spmm_fused_rows concat");
    void* cat = nullptr;
    check(rdmm_event_record(side, &cat), "spmm_fused_rows");
    check(rdmm_event_wait(cat, stream), "spmm_fused_rows");
    rdmm_event_destroy(cat);
    std::uint64_t fl = 0;
    const unsigned flags = (c_zero ? RDMM_SPMM_C_ZERO : 0u) | RDMM_SPMM_NNZ_ON_DEVICE;
    if (panel)
      check(rdmm_spmm_csr_ex(dtype_bytes<T>(), nr, std::uint32_t(col_stride * K), c.cols,
                             std::max<std::uint64_t>(nnz, 1),
                             static_cast<const index_t*>(rpb[q].get()),
                             static_cast<const index_t*>(cib[q].get()), vvb[q].get(), bs[0],
                             b[0].ld, c.values + std::uint64_t(r0) * c.ld, c.ld, flags, nullptr, 0,
                             stream, &fl),
            "spmm_fused_rows");
    else
      check(rdmm_spmm_csr_seg(dtype_bytes<T>(), nr, c.cols, std::max<std::uint64_t>(nnz, 1),
                              static_cast<const index_t*>(rpb[q].get()),
                              static_cast<const index_t*>(cib[q].get()), vvb[q].get(), bs.data(),
                              std::uint32_t(K), std::uint32_t(col_stride), b[0].ld,
                              c.values + std::uint64_t(r0) * c.ld, c.ld, flags, nullptr, 0, stream,
                              &fl),
            "spmm_fused_rows");
    check(rdmm_event_record(stream, &spmm_done[bk]), "spmm_fused_rows");
  }
  for (void* e : spmm_done)
    if (e) rdmm_event_destroy(e);
  return m;  // the buffers are released stream-ordered after the last SpMM
}

// c += x (tile.hpp:300-307); x may live in a peer GPU's heap (NVLink loads).
template <typename T>
void dense_add_into(DevDenseView<T> c, DevDenseConstView<T> x, rdmm_stream_t stream) {
  if (c.rows != x.rows || c.cols != x.cols)
    throw dimension_error("dense_add_into: dimension mismatch");
  if constexpr (sizeof(T) == 8)
    check(rdmm_dense_add_into_f64(c.rows, c.cols, c.values, c.ld, x.values, x.ld, stream),
          "dense_add_into");
  else
    check(rdmm_dense_add_into_f32(c.rows, c.cols, c.values, c.ld, x.values, x.ld, stream),
          "dense_add_into");
}

// One term of a fused sparse sum: a == nullptr-view (rows==0 && !row_ptr)
// means the identity (B as-is).
template <typename T>
struct SpgemmTerm {
  DevCsrView<T> a;
  DevCsrView<T> b;
  bool identity = false;
};

// sum_t A_t*B_t into a fresh device tile (tile.hpp:211-288 generalised);
// per-term FlopMeter flops returned in term_flops when non-null.
template <typename T>
DevCsrTile<T> spgemm_terms(rdmm_fabric* f, std::uint32_t rank, index_t rows, index_t cols,
                           const std::vector<SpgemmTerm<T>>& terms, rdmm_stream_t stream,
                           FlopMeter* meter = nullptr,
                           std::vector<std::uint64_t>* term_flops = nullptr,
                           bool deterministic = false) {
  std::vector<rdmm_spgemm_term> tt(terms.size());
  for (std::size_t i = 0; i < terms.size(); ++i) {
    const auto& t = terms[i];
    tt[i] = rdmm_spgemm_term{t.identity ? nullptr : t.a.row_ptr, t.a.col_idx, t.a.values,
                             t.b.row_ptr, t.b.col_idx, t.b.values};
  }
  DevCsrTile<T> out;
  out.rows = rows;
  out.cols = cols;
  out.row_ptr = DevBuffer(f, rank, (std::uint64_t(rows) + 1) * sizeof(index_t), stream);
  rdmm_spgemm_plan* plan = nullptr;
  std::uint64_t nnz = 0, fl = 0;
  check(rdmm_spgemm_symbolic(rows, cols, dtype_bytes<T>(), tt.data(), int(tt.size()),
                             static_cast<index_t*>(out.row_ptr.get()), &plan, &nnz, &fl,
                             stream),
        "spgemm symbolic");
  out.nnz = nnz;
  out.col_idx = DevBuffer(f, rank, nnz * sizeof(index_t), stream);
  out.values = DevBuffer(f, rank, nnz * sizeof(T), stream);
  int rc = rdmm_spgemm_numeric_ex(plan, static_cast<index_t*>(out.col_idx.get()),
                                  out.values.get(),
                                  deterministic ? RDMM_SPGEMM_DETERMINISTIC : 0u, stream);
  if (term_flops && rc == RDMM_OK) {
    term_flops->assign(terms.size(), 0);
    rdmm_spgemm_plan_term_flops(plan, term_flops->data());
  }
  rdmm_spgemm_plan_destroy(plan);
  check(rc, "spgemm numeric");
  if (meter) {
    meter->flops = fl;
    meter->output_nnz = nnz;
  }
  return out;
}

// (a*b, FlopMeter) -- tile.hpp:211-255
template <typename T>
std::pair<DevCsrTile<T>, FlopMeter> spgemm_local(rdmm_fabric* f, std::uint32_t rank,
                                                 DevCsrView<T> a, DevCsrView<T> b,
                                                 rdmm_stream_t stream,
                                                 bool deterministic = false) {
  if (a.cols != b.rows) throw dimension_error("spgemm_local: dimension mismatch");
  FlopMeter m;
  auto c = spgemm_terms<T>(f, rank, a.rows, b.cols, {{a, b, false}}, stream, &m, nullptr,
                           deterministic);
  return {std::move(c), m};
}

// Merged CSR sum (tile.hpp:257-288).
template <typename T>
DevCsrTile<T> csr_add(rdmm_fabric* f, std::uint32_t rank, DevCsrView<T> a, DevCsrView<T> b,
                      rdmm_stream_t stream) {
  if (a.rows != b.rows || a.cols != b.cols) throw dimension_error("csr_add: dimension mismatch");
  return spgemm_terms<T>(f, rank, a.rows, a.cols, {{{}, a, true}, {{}, b, true}}, stream);
}

}  // namespace rdmm

#endif  // RDMM_B200_TILE_HPP
