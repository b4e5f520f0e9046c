// rdmm/distmat.hpp -- distributed tiled matrices (reference
// /root/reference/proj/include/rdmm/distmat.hpp) with device-resident tiles.
//
// Same surface: ProcGrid, detail::TileGeom, TileFuture, DistDense,
// DistSparse (1 get per dense tile, 3 per sparse tile, owner-only tile_ref,
// replace_tile + collective renew_tiles, host to_global) and the contrib
// wire format.  Deltas: tiles live in the owners' device
// heaps; get_tile/async_get_tile return device tiles; a fetch of a rank's
// own tile aliases it instead of copying (recorded as self traffic); the
// replicated directory lives in the fabric's control segment so it is shared
// by all processes of a multi-process fabric.
#ifndef RDMM_B200_DISTMAT_HPP
#define RDMM_B200_DISTMAT_HPP

#include <cmath>
#include <cstring>
#include <functional>

#include "rdmm/fabric.hpp"
#include "rdmm/tile.hpp"

namespace rdmm {

struct ProcGrid {  // distmat.hpp:20-36
  rank_t pr = 1, pc = 1;
  rank_t nranks() const { return pr * pc; }
  rank_t owner(std::uint32_t i, std::uint32_t j) const { return (i % pr) * pc + (j % pc); }
  bool square() const { return pr == pc; }
  static ProcGrid square_of(rank_t p) {
    rank_t s = static_cast<rank_t>(std::lround(std::sqrt(double(p))));
    if (s * s != p) throw fabric_error("processor count is not a perfect square");
    return {s, s};
  }
};

namespace detail {

struct TileGeom {  // distmat.hpp:40-67
  std::uint64_t m = 0, n = 0;
  std::uint32_t tm = 0, tn = 0;
  std::uint32_t M = 0, N = 0;
  TileGeom() = default;
  TileGeom(std::uint64_t m, std::uint64_t n, std::uint32_t tm, std::uint32_t tn)
      : m(m), n(n), tm(tm), tn(tn) {
    if (tm == 0 || tn == 0) throw dimension_error("tile dims must be positive");
    M = static_cast<std::uint32_t>((m + tm - 1) / tm);
    N = static_cast<std::uint32_t>((n + tn - 1) / tn);
  }
  std::uint32_t tile_rows(std::uint32_t i) const {
    return static_cast<std::uint32_t>(std::min<std::uint64_t>(tm, m - std::uint64_t(i) * tm));
  }
  std::uint32_t tile_cols(std::uint32_t j) const {
    return static_cast<std::uint32_t>(std::min<std::uint64_t>(tn, n - std::uint64_t(j) * tn));
  }
  std::size_t idx(std::uint32_t i, std::uint32_t j) const { return std::size_t(i) * N + j; }
  void check(std::uint32_t i, std::uint32_t j) const {
    if (i >= M || j >= N) throw dimension_error("tile index out of range");
  }
};

// Per-Fabric matrix counter: processes construct matrices in the same order,
// so a matrix gets the same uid (and control-segment directory) everywhere.
inline std::uint64_t next_matrix_uid(Fabric& f) { return rdmm_fabric_next_uid(f.handle()); }

// Control-segment array shared by all ranks/processes (tag-addressed).
template <typename E>
E* shared_array(Fabric& f, std::uint64_t tag, std::size_t count, rdmm_gptr* where) {
  const std::uint64_t cells = (count * sizeof(E) + 7) / 8;
  check(rdmm_ctrl_cells(f.handle(), f.first_local(), tag, cells ? cells : 1, where),
        "directory");
  return static_cast<E*>(rdmm_ctrl_host(f.handle(), *where));
}

inline void release_shared(Fabric& f, std::uint64_t tag) {
  for (rank_t r = f.first_local(); r < f.first_local() + f.nlocal(); ++r)
    rdmm_ctrl_release(f.handle(), r, tag);
}

constexpr std::uint64_t kDirTag = 0x4449520000000000ull;  // "DIR"

}  // namespace detail

// Future for in-flight tile fetches (distmat.hpp:71-88).  get() makes the
// rank's compute stream wait for the copies (no host block) and returns the
// device tile.
template <typename TileT>
class TileFuture {
 public:
  TileFuture() = default;
  TileFuture(TileT tile, std::vector<Fabric::TransferHandle> handles, RankCtx* ctx)
      : tile_(std::move(tile)), handles_(std::move(handles)), ctx_(ctx) {}
  TileT get() {
    for (auto& h : handles_) ctx_->wait(h);
    tile_.release_on(ctx_->stream(0));
    return std::move(tile_);
  }
  bool valid() const { return ctx_ != nullptr; }

 private:
  TileT tile_;
  std::vector<Fabric::TransferHandle> handles_;
  RankCtx* ctx_ = nullptr;
};

// ------------------------------------------------------------------ dense

template <typename T>
class DistDense {  // distmat.hpp:92-205
 public:
  DistDense(Fabric& f, std::uint64_t m, std::uint64_t n, std::uint32_t tm, std::uint32_t tn,
            ProcGrid grid, int matrix_id = 0)
      : fabric_(&f), geom_(m, n, tm, tn), grid_(grid), matrix_id_(matrix_id) {
    if (grid.nranks() != f.nranks())
      throw fabric_error("processor grid does not match fabric rank count");
    tag_ = detail::kDirTag | detail::next_matrix_uid(f);
    dir_ = detail::shared_array<rdmm_gptr>(f, tag_, std::size_t(geom_.M) * geom_.N, &where_);
    zero_.assign(std::size_t(geom_.M) * geom_.N, 0);
  }
  ~DistDense() { detail::release_shared(*fabric_, tag_); }
  DistDense(const DistDense&) = delete;
  DistDense& operator=(const DistDense&) = delete;

  const detail::TileGeom& geom() const { return geom_; }
  const ProcGrid& grid() const { return grid_; }
  std::uint32_t tile_grid_rows() const { return geom_.M; }
  std::uint32_t tile_grid_cols() const { return geom_.N; }
  rank_t owner(std::uint32_t i, std::uint32_t j) const { return grid_.owner(i, j); }
  int matrix_id() const { return matrix_id_; }
  Fabric& fabric() const { return *fabric_; }

  // Collective.  fill(i, j) -> host DenseTile for owned tiles; nullptr zeros.
  void init(RankCtx& ctx, const std::function<DenseTile<T>(std::uint32_t, std::uint32_t)>&
                              fill = nullptr) {
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        const std::uint32_t r = geom_.tile_rows(i), c = geom_.tile_cols(j);
        GlobalPtr p = fresh_tile(ctx, i, j);
        if (fill) {
          DenseTile<T> t = fill(i, j);
          if (t.rows != r || t.cols != c) throw dimension_error("init fill produced wrong tile dims");
          ctx.put(std::as_bytes(std::span{t.values}), p);
          zero_[geom_.idx(i, j)] = 0;
        } else {
          check(rdmm_memset(fabric_->raw(p, ctx.rank()), 0, p.length, ctx.stream(0)), "init");
          zero_[geom_.idx(i, j)] = 1;
        }
        dir_[geom_.idx(i, j)] = p.c();
      }
    ctx.barrier();
  }

  // Collective; scatters a global row-major host array (distmat.hpp:134-145).
  void init_from_global(RankCtx& ctx, const std::vector<T>& global) {
    if (global.size() != geom_.m * geom_.n) throw dimension_error("global array size mismatch");
    init_from_host(ctx, global.data(), geom_.n);
  }
  void init_from_host(RankCtx& ctx, const T* global, std::uint64_t ld) {
    init_from_any(ctx, global, ld);
  }
  // B200: scatter from a device-resident global array (any GPU of the box).
  void init_from_device(RankCtx& ctx, const T* global, std::uint64_t ld) {
    init_from_any(ctx, global, ld);
  }

  // One get per dense tile (distmat.hpp:147-155); blocks until it landed.
  DevDenseTile<T> get_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j) const {
    auto f = async_get_tile(ctx, i, j);
    DevDenseTile<T> t = f.get();
    check(rdmm_stream_sync(ctx.stream(0)), "get_tile");
    return t;
  }

  TileFuture<DevDenseTile<T>> async_get_tile(RankCtx& ctx, std::uint32_t i,
                                             std::uint32_t j) const {
    geom_.check(i, j);
    GlobalPtr p = GlobalPtr::of(dir_[geom_.idx(i, j)]);
    DevDenseTile<T> t;
    t.rows = geom_.tile_rows(i);
    t.cols = geom_.tile_cols(j);
    std::vector<Fabric::TransferHandle> hs;
    if (p.rank == ctx.rank()) {
      t.buf = DevBuffer::alias(fabric_->raw(p, ctx.rank()));
      rdmm_record_self_get(ctx.h(), ctx.rank(), p.length);
    } else {
      t.buf = DevBuffer(ctx.h(), ctx.rank(), p.length, ctx.stream(1));
      hs.push_back(ctx.get_nb(p, t.buf.get(), 1));
    }
    ctx.record_tile_fetch(p.rank, matrix_id_, i, j);
    return TileFuture<DevDenseTile<T>>(std::move(t), std::move(hs), &ctx);
  }

  // Direct mutable device view of an owned tile; no traffic (distmat.hpp:169-180).
  DevDenseView<T> tile_ref(RankCtx& ctx, std::uint32_t i, std::uint32_t j) {
    geom_.check(i, j);
    if (owner(i, j) != ctx.rank()) throw fabric_error("tile_ref: caller does not own tile");
    GlobalPtr p = GlobalPtr::of(dir_[geom_.idx(i, j)]);
    const std::uint32_t c = geom_.tile_cols(j);
    return {geom_.tile_rows(i), c, c, static_cast<T*>(fabric_->raw(p, ctx.rank()))};
  }
  GlobalPtr tile_ptr(std::uint32_t i, std::uint32_t j) const {
    return GlobalPtr::of(dir_[geom_.idx(i, j)]);
  }
  // Collective: zero every owned tile in place (a fresh C for the next run).
  void zero(RankCtx& ctx) {
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        GlobalPtr p = tile_ptr(i, j);
        check(rdmm_memset(fabric_->raw(p, ctx.rank()), 0, p.length, ctx.stream(0)), "zero");
        zero_[geom_.idx(i, j)] = 1;
      }
    ctx.barrier();
  }
  // Copy the caller's owned tiles into a row-major global host array (the
  // device->host half of an end-to-end call; other ranks' tiles untouched).
  // With `stream` (a caller-owned stream on the rank's device) the copies are
  // only enqueued there, ordered after the rank's queued compute, and the
  // call returns at once (the download of one step overlaps the next).
  void owned_to_host(RankCtx& ctx, T* global, std::uint64_t ld, rdmm_stream_t stream = nullptr) {
    rdmm_stream_t s = stream ? stream : ctx.stream(0);
    if (stream) {
      void* done = nullptr;
      check(rdmm_event_record(ctx.stream(0), &done), "owned_to_host");
      check(rdmm_event_wait(done, stream), "owned_to_host");
      rdmm_event_destroy(done);
    }
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        const std::uint32_t r = geom_.tile_rows(i), c = geom_.tile_cols(j);
        T* dst = global + std::uint64_t(i) * geom_.tm * ld + std::uint64_t(j) * geom_.tn;
        check(rdmm_memcpy2d(dst, ld * sizeof(T), fabric_->raw(tile_ptr(i, j), ctx.rank()),
                            c * sizeof(T), c * sizeof(T), r, s),
              "owned_to_host");
      }
    if (!stream) check(rdmm_stream_sync(ctx.stream(0)), "owned_to_host");
  }
  // B200: zero-tracking so the first product into a fresh tile skips reading C.
  bool tile_is_zero(std::uint32_t i, std::uint32_t j) const { return zero_[geom_.idx(i, j)]; }
  void mark_nonzero(std::uint32_t i, std::uint32_t j) { zero_[geom_.idx(i, j)] = 0; }

  // Host-side gather for verification; bypasses traffic (distmat.hpp:183-197).
  std::vector<T> to_global() const {
    std::vector<T> g(geom_.m * geom_.n, T{});
    std::vector<T> buf;
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        GlobalPtr p = GlobalPtr::of(dir_[geom_.idx(i, j)]);
        const std::uint32_t r = geom_.tile_rows(i), c = geom_.tile_cols(j);
        buf.resize(std::size_t(r) * c);
        fabric_->peek(p, buf.data());
        for (std::uint32_t rr = 0; rr < r; ++rr)
          std::memcpy(&g[(std::uint64_t(i) * geom_.tm + rr) * geom_.n + std::uint64_t(j) * geom_.tn],
                      &buf[std::size_t(rr) * c], c * sizeof(T));
      }
    return g;
  }

 private:
  // Re-initialisation reuses the tile's allocation (same geometry).  B200:
  // the tiles a rank owns in one tile column are placed back to back in ONE
  // heap allocation (tile (i,j) right after its owned predecessor in column
  // j), so a column panel B(:, j) held by one rank is a single row-major
  // array and the fused SpMM can index it directly instead of by segments.
  GlobalPtr fresh_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j) {
    const rdmm_gptr old = dir_[geom_.idx(i, j)];
    if (old.length) return GlobalPtr::of(old);
    std::uint64_t total = 0;
    for (std::uint32_t q = 0; q < geom_.M; ++q)
      if (owner(q, j) == ctx.rank())
        total += std::uint64_t(geom_.tile_rows(q)) * geom_.tile_cols(j) * sizeof(T);
    auto pad = [](std::uint64_t b) { return (b + 255) & ~std::uint64_t{255}; };
    total = 0;
    for (std::uint32_t q = 0; q < geom_.M; ++q)
      if (owner(q, j) == ctx.rank())
        total += pad(std::uint64_t(geom_.tile_rows(q)) * geom_.tile_cols(j) * sizeof(T));
    GlobalPtr panel = ctx.alloc(total);
    std::uint64_t off = 0;
    for (std::uint32_t q = 0; q < geom_.M; ++q) {
      if (owner(q, j) != ctx.rank()) continue;
      const std::uint64_t bytes = std::uint64_t(geom_.tile_rows(q)) * geom_.tile_cols(j) * sizeof(T);
      dir_[geom_.idx(q, j)] = GlobalPtr{panel.rank, panel.offset + off, bytes}.c();
      off += pad(bytes);
    }
    return GlobalPtr::of(dir_[geom_.idx(i, j)]);
  }
  void init_from_any(RankCtx& ctx, const T* global, std::uint64_t ld) {
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        const std::uint32_t r = geom_.tile_rows(i), c = geom_.tile_cols(j);
        GlobalPtr p = fresh_tile(ctx, i, j);
        const T* src = global + std::uint64_t(i) * geom_.tm * ld + std::uint64_t(j) * geom_.tn;
        check(rdmm_memcpy2d(fabric_->raw(p, ctx.rank()), c * sizeof(T), src, ld * sizeof(T),
                            c * sizeof(T), r, ctx.stream(0)),
              "init_from_global");
        zero_[geom_.idx(i, j)] = 0;
        dir_[geom_.idx(i, j)] = p.c();
      }
    ctx.barrier();
  }

  Fabric* fabric_;
  detail::TileGeom geom_;
  ProcGrid grid_;
  int matrix_id_;
  std::uint64_t tag_ = 0;
  rdmm_gptr where_{};
  rdmm_gptr* dir_ = nullptr;
  std::vector<char> zero_;
};

// ------------------------------------------------------------------ sparse

template <typename T>
class DistSparse {  // distmat.hpp:210-398
 public:
  // B200: the tile's entry offsets at the boundaries of kRowBlocks equal row
  // blocks (row_ptr[b * row_block(rows)], b = 0..kRowBlocks), kept in the
  // replicated directory so a rank can fetch a remote tile block by block
  // without first reading its row_ptr (blocks_valid = 0: unknown).
  static constexpr std::uint32_t kRowBlocks = 16;
  static std::uint32_t row_block(std::uint32_t rows) { return (rows + kRowBlocks - 1) / kRowBlocks; }
  struct Entry {  // distmat.hpp:213-216 (+ block offsets)
    rdmm_gptr values, row_ptr, col_idx;
    std::uint64_t nnz = 0;
    std::uint32_t blocks_valid = 0;
    std::uint32_t blk_off[kRowBlocks + 1] = {};
  };
  const Entry& entry(std::uint32_t i, std::uint32_t j) const { return dir_[geom_.idx(i, j)]; }

  DistSparse(Fabric& f, std::uint64_t m, std::uint64_t n, std::uint32_t tm, std::uint32_t tn,
             ProcGrid grid, int matrix_id = 0)
      : fabric_(&f), geom_(m, n, tm, tn), grid_(grid), matrix_id_(matrix_id) {
    if (grid.nranks() != f.nranks())
      throw fabric_error("processor grid does not match fabric rank count");
    tag_ = detail::kDirTag | detail::next_matrix_uid(f);
    dir_ = detail::shared_array<Entry>(f, tag_, std::size_t(geom_.M) * geom_.N, &where_);
    pending_.resize(f.nranks());
  }
  ~DistSparse() { detail::release_shared(*fabric_, tag_); }
  DistSparse(const DistSparse&) = delete;
  DistSparse& operator=(const DistSparse&) = delete;

  const detail::TileGeom& geom() const { return geom_; }
  const ProcGrid& grid() const { return grid_; }
  std::uint32_t tile_grid_rows() const { return geom_.M; }
  std::uint32_t tile_grid_cols() const { return geom_.N; }
  rank_t owner(std::uint32_t i, std::uint32_t j) const { return grid_.owner(i, j); }
  int matrix_id() const { return matrix_id_; }
  std::uint64_t tile_nnz(std::uint32_t i, std::uint32_t j) const { return dir_[geom_.idx(i, j)].nnz; }
  Fabric& fabric() const { return *fabric_; }

  // Collective.  fill(i, j) -> host CsrTile for owned tiles; nullptr empty.
  void init(RankCtx& ctx, const std::function<CsrTile<T>(std::uint32_t, std::uint32_t)>&
                              fill = nullptr) {
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        CsrTile<T> t = fill ? fill(i, j) : CsrTile<T>(geom_.tile_rows(i), geom_.tile_cols(j));
        if (t.rows != geom_.tile_rows(i) || t.cols != geom_.tile_cols(j))
          throw dimension_error("init fill produced wrong tile dims");
        drop_tile(ctx, i, j);
        dir_[geom_.idx(i, j)] = store_host(ctx, t);
      }
    ctx.barrier();
  }

  void init_from_global(RankCtx& ctx, const CsrTile<T>& global) {  // distmat.hpp:257-263
    if (global.rows != geom_.m || global.cols != geom_.n)
      throw dimension_error("global matrix dims mismatch");
    init(ctx, [&](std::uint32_t i, std::uint32_t j) { return extract_tile(global, i, j); });
  }

  // B200: tiles cut on the device out of a device-resident global CSR.
  void init_from_device_global(RankCtx& ctx, DevCsrView<T> g) {
    if (g.rows != geom_.m || g.cols != geom_.n) throw dimension_error("global matrix dims mismatch");
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        const std::uint32_t r = geom_.tile_rows(i), c = geom_.tile_cols(j);
        drop_tile(ctx, i, j);
        Entry e;
        e.row_ptr = ctx.alloc((std::uint64_t(r) + 1) * sizeof(index_t)).c();
        auto* rp = static_cast<index_t*>(fabric_->raw(GlobalPtr::of(e.row_ptr), ctx.rank()));
        std::uint64_t nnz = 0;
        check(rdmm_csr_extract_count(g.row_ptr, g.col_idx, std::uint64_t(i) * geom_.tm, r,
                                     std::uint64_t(j) * geom_.tn, c, rp, &nnz, ctx.stream(0)),
              "extract");
        e.nnz = nnz;
        set_block_offsets_device(ctx, e, rp, r);
        e.col_idx = ctx.alloc(nnz * sizeof(index_t)).c();
        e.values = ctx.alloc(nnz * sizeof(T)).c();
        check(rdmm_csr_extract_fill(dtype_bytes<T>(), g.row_ptr, g.col_idx, g.values,
                                    std::uint64_t(i) * geom_.tm, r, std::uint64_t(j) * geom_.tn,
                                    c, rp,
                                    static_cast<index_t*>(fabric_->raw(GlobalPtr::of(e.col_idx), ctx.rank())),
                                    fabric_->raw(GlobalPtr::of(e.values), ctx.rank()),
                                    ctx.stream(0)),
              "extract");
        dir_[geom_.idx(i, j)] = e;
      }
    ctx.barrier();
  }

  CsrTile<T> extract_tile(const CsrTile<T>& global, std::uint32_t i, std::uint32_t j) const {
    CsrTile<T> t(geom_.tile_rows(i), geom_.tile_cols(j));  // distmat.hpp:265-282
    const std::uint64_t r0 = std::uint64_t(i) * geom_.tm, c0 = std::uint64_t(j) * geom_.tn;
    for (std::uint32_t r = 0; r < t.rows; ++r) {
      const index_t gr = static_cast<index_t>(r0 + r);
      for (index_t s = global.row_ptr[gr]; s < global.row_ptr[gr + 1]; ++s) {
        const std::uint64_t gc = global.col_idx[s];
        if (gc >= c0 && gc < c0 + t.cols) {
          t.col_idx.push_back(static_cast<index_t>(gc - c0));
          t.values.push_back(global.values[s]);
        }
      }
      t.row_ptr[r + 1] = static_cast<index_t>(t.col_idx.size());
    }
    return t;
  }

  // Three gets per sparse tile (distmat.hpp:284-296); blocks.
  DevCsrTile<T> get_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j) const {
    auto f = async_get_tile(ctx, i, j);
    DevCsrTile<T> t = f.get();
    check(rdmm_stream_sync(ctx.stream(0)), "get_tile");
    return t;
  }

  TileFuture<DevCsrTile<T>> async_get_tile(RankCtx& ctx, std::uint32_t i,
                                           std::uint32_t j) const {
    geom_.check(i, j);
    const Entry& e = dir_[geom_.idx(i, j)];
    DevCsrTile<T> t;
    t.rows = geom_.tile_rows(i);
    t.cols = geom_.tile_cols(j);
    t.nnz = e.nnz;
    std::vector<Fabric::TransferHandle> hs;
    if (e.values.rank == ctx.rank()) {
      t.row_ptr = DevBuffer::alias(fabric_->raw(GlobalPtr::of(e.row_ptr), ctx.rank()));
      t.col_idx = DevBuffer::alias(fabric_->raw(GlobalPtr::of(e.col_idx), ctx.rank()));
      t.values = DevBuffer::alias(fabric_->raw(GlobalPtr::of(e.values), ctx.rank()));
      for (auto g : {e.row_ptr, e.col_idx, e.values})
        rdmm_record_self_get(ctx.h(), ctx.rank(), g.length);
    } else {
      // Each buffer is allocated on the stream that fills it: the stream-
      // ordered pool may hand out a block freed on the compute stream and
      // orders only the allocating stream behind that free.
      t.row_ptr = DevBuffer(ctx.h(), ctx.rank(), e.row_ptr.length, ctx.stream(1));
      t.col_idx = DevBuffer(ctx.h(), ctx.rank(), e.col_idx.length, ctx.stream(2));
      t.values = DevBuffer(ctx.h(), ctx.rank(), e.values.length, ctx.stream(2));
      hs.push_back(ctx.get_nb(GlobalPtr::of(e.row_ptr), t.row_ptr.get(), 1));
      hs.push_back(ctx.get_nb(GlobalPtr::of(e.col_idx), t.col_idx.get(), 2));
      hs.push_back(ctx.get_nb(GlobalPtr::of(e.values), t.values.get(), 2));
    }
    ctx.record_tile_fetch(e.values.rank, matrix_id_, i, j);
    return TileFuture<DevCsrTile<T>>(std::move(t), std::move(hs), &ctx);
  }

  // Read-only device view of an owned tile (distmat.hpp:317-329).
  DevCsrView<T> tile_ref(RankCtx& ctx, std::uint32_t i, std::uint32_t j) const {
    geom_.check(i, j);
    if (owner(i, j) != ctx.rank()) throw fabric_error("tile_ref: caller does not own tile");
    return view_of(dir_[geom_.idx(i, j)], ctx.rank(), geom_.tile_rows(i), geom_.tile_cols(j));
  }
  // Device view of any tile from `viewer`'s GPU (peer-mapped, zero copy).
  DevCsrView<T> peer_view(rank_t viewer, std::uint32_t i, std::uint32_t j) const {
    return view_of(dir_[geom_.idx(i, j)], viewer, geom_.tile_rows(i), geom_.tile_cols(j));
  }

  // Owner stages a new tile (distmat.hpp:333-341).
  void replace_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j, const CsrTile<T>& t) {
    check_replace(ctx, i, j, t.rows, t.cols);
    pending_[ctx.rank()].push_back({geom_.idx(i, j), store_host(ctx, t)});
  }
  void replace_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j, const DevCsrTile<T>& t) {
    check_replace(ctx, i, j, t.rows, t.cols);
    pending_[ctx.rank()].push_back({geom_.idx(i, j), store_device(ctx, t.view())});
  }

  // Collective; publishes staged tiles and frees the old ones (distmat.hpp:345-356).
  void renew_tiles(RankCtx& ctx) {
    ctx.barrier();
    for (auto& [idx, entry] : pending_[ctx.rank()]) {
      Entry old = dir_[idx];
      dir_[idx] = entry;
      ctx.free(GlobalPtr::of(old.values));
      ctx.free(GlobalPtr::of(old.row_ptr));
      ctx.free(GlobalPtr::of(old.col_idx));
    }
    pending_[ctx.rank()].clear();
    ctx.barrier();
  }

  // Bytes of the caller's owned tiles (raw CSR arrays).
  std::uint64_t owned_bytes(rank_t r) const {
    std::uint64_t bytes = 0;
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j)
        if (owner(i, j) == r) {
          const Entry& e = dir_[geom_.idx(i, j)];
          bytes += e.row_ptr.length + e.col_idx.length + e.values.length;
        }
    return bytes;
  }
  // Copy the caller's owned tiles (raw CSR arrays, concatenated) into a host
  // buffer (the device->host half of an end-to-end call); returns bytes.
  std::uint64_t owned_to_host(RankCtx& ctx, char* out, std::uint64_t cap) {
    std::uint64_t bytes = 0;
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        if (owner(i, j) != ctx.rank()) continue;
        const Entry& e = dir_[geom_.idx(i, j)];
        for (auto g : {e.row_ptr, e.col_idx, e.values}) {
          if (bytes + g.length > cap) throw std::invalid_argument("owned_to_host: buffer too small");
          if (g.length)
            check(rdmm_memcpy(out + bytes, fabric_->raw(GlobalPtr::of(g), ctx.rank()), g.length,
                              ctx.stream(0)),
                  "owned_to_host");
          bytes += g.length;
        }
      }
    check(rdmm_stream_sync(ctx.stream(0)), "owned_to_host");
    return bytes;
  }

  // Host-side gather; bypasses traffic (distmat.hpp:359-377).
  CsrTile<T> to_global() const {
    CsrTile<T> g(static_cast<index_t>(geom_.m), static_cast<index_t>(geom_.n));
    std::vector<std::vector<index_t>> rp(geom_.M * std::size_t(geom_.N)),
        ci(geom_.M * std::size_t(geom_.N));
    std::vector<std::vector<T>> vv(geom_.M * std::size_t(geom_.N));
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t j = 0; j < geom_.N; ++j) {
        const std::size_t x = geom_.idx(i, j);
        const Entry& e = dir_[x];
        rp[x].resize(geom_.tile_rows(i) + 1);
        ci[x].resize(e.nnz);
        vv[x].resize(e.nnz);
        fabric_->peek(GlobalPtr::of(e.row_ptr), rp[x].data());
        if (e.nnz) {
          fabric_->peek(GlobalPtr::of(e.col_idx), ci[x].data());
          fabric_->peek(GlobalPtr::of(e.values), vv[x].data());
        }
      }
    // rows of tile-row i are the concatenation of tiles (i, 0..N-1): already
    // column-sorted across tiles because tile j covers [j*tn, (j+1)*tn)
    for (std::uint32_t i = 0; i < geom_.M; ++i)
      for (std::uint32_t r = 0; r < geom_.tile_rows(i); ++r) {
        const std::uint64_t gr = std::uint64_t(i) * geom_.tm + r;
        for (std::uint32_t j = 0; j < geom_.N; ++j) {
          const std::size_t x = geom_.idx(i, j);
          for (index_t s = rp[x][r]; s < rp[x][r + 1]; ++s) {
            g.col_idx.push_back(static_cast<index_t>(std::uint64_t(j) * geom_.tn + ci[x][s]));
            g.values.push_back(vv[x][s]);
          }
        }
        g.row_ptr[gr + 1] = static_cast<index_t>(g.col_idx.size());
      }
    return g;
  }

 private:
  DevCsrView<T> view_of(const Entry& e, rank_t viewer, std::uint32_t rows,
                        std::uint32_t cols) const {
    DevCsrView<T> v;
    v.rows = rows;
    v.cols = cols;
    v.nnz = e.nnz;
    v.row_ptr = static_cast<const index_t*>(fabric_->raw(GlobalPtr::of(e.row_ptr), viewer));
    v.col_idx = static_cast<const index_t*>(fabric_->raw(GlobalPtr::of(e.col_idx), viewer));
    v.values = static_cast<const T*>(fabric_->raw(GlobalPtr::of(e.values), viewer));
    return v;
  }
  // Re-initialisation releases the tile's previous allocations.
  void drop_tile(RankCtx& ctx, std::uint32_t i, std::uint32_t j) {
    Entry& e = dir_[geom_.idx(i, j)];
    if (!e.row_ptr.length) return;
    ctx.free(GlobalPtr::of(e.values));
    ctx.free(GlobalPtr::of(e.row_ptr));
    ctx.free(GlobalPtr::of(e.col_idx));
    e = Entry{};
  }
  void check_replace(RankCtx& ctx, std::uint32_t i, std::uint32_t j, index_t rows, index_t cols) {
    geom_.check(i, j);
    if (owner(i, j) != ctx.rank()) throw fabric_error("replace_tile: caller does not own tile");
    if (rows != geom_.tile_rows(i) || cols != geom_.tile_cols(j))
      throw dimension_error("replace_tile: wrong tile dims");
  }
  // distmat.hpp:380-390: 3 allocs + 3 puts
  void set_block_offsets_device(RankCtx& ctx, Entry& e, const index_t* dev_rp, std::uint32_t rows) {
    check(rdmm_stream_sync(ctx.stream(0)), "block offsets");
    const std::uint32_t rb = row_block(rows);
    for (std::uint32_t b = 0; b <= kRowBlocks; ++b) {
      const std::uint32_t r = std::min<std::uint64_t>(std::uint64_t(b) * rb, rows);
      check(rdmm_memcpy(&e.blk_off[b], dev_rp + r, sizeof(index_t), nullptr), "block offsets");
    }
    e.blocks_valid = 1;
  }
  Entry store_host(RankCtx& ctx, const CsrTile<T>& t) {
    Entry e;
    e.nnz = t.nnz();
    {
      const std::uint32_t rb = row_block(t.rows);
      for (std::uint32_t b = 0; b <= kRowBlocks; ++b)
        e.blk_off[b] = t.row_ptr[std::min<std::uint64_t>(std::uint64_t(b) * rb, t.rows)];
      e.blocks_valid = 1;
    }
    e.row_ptr = ctx.alloc(t.row_ptr.size() * sizeof(index_t)).c();
    e.col_idx = ctx.alloc(t.col_idx.size() * sizeof(index_t)).c();
    e.values = ctx.alloc(t.values.size() * sizeof(T)).c();
    ctx.put(std::as_bytes(std::span{t.row_ptr}), GlobalPtr::of(e.row_ptr));
    ctx.put(std::as_bytes(std::span{t.col_idx}), GlobalPtr::of(e.col_idx));
    ctx.put(std::as_bytes(std::span{t.values}), GlobalPtr::of(e.values));
    return e;
  }
  Entry store_device(RankCtx& ctx, DevCsrView<T> v) {
    Entry e;
    e.nnz = v.nnz;
    e.row_ptr = ctx.alloc((std::uint64_t(v.rows) + 1) * sizeof(index_t)).c();
    e.col_idx = ctx.alloc(v.nnz * sizeof(index_t)).c();
    e.values = ctx.alloc(v.nnz * sizeof(T)).c();
    Fabric::TransferHandle h[3];
    int rc = rdmm_put_nb(ctx.h(), ctx.rank(), v.row_ptr, e.row_ptr, ctx.stream(0), &h[0].h);
    if (!rc && v.nnz) rc = rdmm_put_nb(ctx.h(), ctx.rank(), v.col_idx, e.col_idx, ctx.stream(0), &h[1].h);
    if (!rc && v.nnz) rc = rdmm_put_nb(ctx.h(), ctx.rank(), v.values, e.values, ctx.stream(0), &h[2].h);
    check(rc, "replace_tile");
    for (auto& x : h) rdmm_event_destroy(x.h.event);
    return e;
  }

  Fabric* fabric_;
  detail::TileGeom geom_;
  ProcGrid grid_;
  int matrix_id_;
  std::uint64_t tag_ = 0;
  rdmm_gptr where_{};
  Entry* dir_ = nullptr;
  std::vector<std::vector<std::pair<std::size_t, Entry>>> pending_;
};

// Contribution wire format (distmat.hpp:406-452): a 32-byte header followed
// by the payload in the producer's heap; the queue entry carries the same
// header inline so the consumer never reads it back.  B200: the consumer
// reads the payload in place over NVLink and the consumed flag of triple
// (i,j,k) lives in a control-segment array, so reclaim is a host load.
namespace contrib {
struct Header {
  std::int64_t consumed = 0;
  std::uint32_t i = 0, j = 0;
  std::uint32_t rows = 0, cols = 0;
  std::uint64_t nnz = 0;  // ~0: dense payload
};
inline constexpr std::uint64_t kDenseTag = ~std::uint64_t{0};
inline std::size_t align8(std::size_t n) { return (n + 7) & ~std::size_t{7}; }
// Inline queue payload: header fields + the k of the triple.
struct Inline {
  std::uint32_t i, j, k, rows, cols, pad;
  std::uint64_t nnz;
};
static_assert(sizeof(Inline) <= 40, "inline queue payload");
}  // namespace contrib

}  // namespace rdmm

#endif  // RDMM_B200_DISTMAT_HPP
