// host_capi.cpp -- C-ABI over the C++ driver layer (include/rdmm/*.hpp),
// see include/rdmm_host.h.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <variant>

#include "rdmm/algos.hpp"
#include "rdmm/analytics.hpp"
#include "rdmm/mmio.hpp"
#include "rdmm_host.h"

using namespace rdmm;

struct rdmm_h_fabric {
  std::unique_ptr<Fabric> f;
};

struct rdmm_h_matrix {
  rdmm_h_fabric* fab = nullptr;
  int kind = 0, dtype = 4;
  std::variant<std::monostate, std::unique_ptr<DistSparse<float>>, std::unique_ptr<DistSparse<double>>,
               std::unique_ptr<DistDense<float>>, std::unique_ptr<DistDense<double>>>
      m;
};

namespace {

int to_code(const std::exception& e) {
  std::string msg = e.what();
  if (dynamic_cast<const mmio_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_IO, msg.c_str());
  if (dynamic_cast<const dimension_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_DIMENSION, msg.c_str());
  if (dynamic_cast<const heap_exhausted_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_HEAP_EXHAUSTED, msg.c_str());
  if (dynamic_cast<const queue_full_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_QUEUE_FULL, msg.c_str());
  if (dynamic_cast<const protocol_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_PROTOCOL, msg.c_str());
  if (dynamic_cast<const fabric_error*>(&e)) return rdmm_impl_fail(RDMM_ERR_FABRIC, msg.c_str());
  if (dynamic_cast<const std::invalid_argument*>(&e)) return rdmm_impl_fail(RDMM_ERR_INVALID, msg.c_str());
  return rdmm_impl_fail(RDMM_ERR_CUDA, msg.c_str());
}

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return RDMM_OK;
  } catch (const std::exception& e) {
    return to_code(e);
  } catch (...) {
    return rdmm_impl_fail(RDMM_ERR_CUDA, "unknown exception");
  }
}

template <typename T>
void sparse_init(Fabric& f, DistSparse<T>& A, const uint32_t* rp, const uint32_t* ci,
                 const void* vals, uint64_t nnz, int on_device) {
  if (!rp) {
    run_ranks(f, [&](RankCtx& ctx) { A.init(ctx); });
    return;
  }
  if (on_device) {
    DevCsrView<T> g{index_t(A.geom().m), index_t(A.geom().n), nnz, rp, ci,
                    static_cast<const T*>(vals)};
    run_ranks(f, [&](RankCtx& ctx) { A.init_from_device_global(ctx, g); });
    return;
  }
  CsrTile<T> g(index_t(A.geom().m), index_t(A.geom().n));
  g.row_ptr.assign(rp, rp + A.geom().m + 1);
  g.col_idx.assign(ci, ci + nnz);
  const T* v = static_cast<const T*>(vals);
  g.values.assign(v, v + nnz);
  run_ranks(f, [&](RankCtx& ctx) { A.init_from_global(ctx, g); });
}

template <typename T>
void dense_init(Fabric& f, DistDense<T>& B, const void* global, uint64_t ld) {
  if (!global) {
    run_ranks(f, [&](RankCtx& ctx) { B.init(ctx); });
    return;
  }
  run_ranks(f, [&](RankCtx& ctx) { B.init_from_host(ctx, static_cast<const T*>(global), ld); });
}

RunOptions opts_of(const rdmm_h_options* o) {
  RunOptions r;
  if (!o) return r;
  r.variant = static_cast<Variant>(o->variant);
  r.ws_base = static_cast<Variant>(o->ws_base);
  r.prefetch = o->prefetch != 0;
  r.offset = o->offset != 0;
  r.seed = o->seed;
  r.delay_ns_per_flop = o->delay_ns_per_flop;
  r.random_delay_ms_max = o->random_delay_ms_max;
  r.record_events = o->record_events != 0;
  r.record_triples = o->record_triples != 0;
  r.lookahead = o->lookahead > 0 ? o->lookahead : 2;
  r.ws_local_inplace = o->ws_local_inplace != 0;
  r.checksum = o->checksum != 0;
  r.fuse_k = o->fuse_k != 0;
  r.split_local = o->split_local != 0;
  r.time_stages = o->time_stages != 0;
  r.pipeline = o->pipeline != 0;
  if (o->row_blocks > 0) r.row_blocks = std::uint32_t(o->row_blocks);
  r.deterministic = o->deterministic != 0;
  return r;
}

void fill(const RunReport& r, rdmm_h_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->wall_seconds = r.wall_seconds;
  out->checksum = r.checksum;
  out->total_flops = r.total_flops();
  out->total_multiplies = r.total_multiplies();
  out->total_steals = r.total_steals();
  out->nranks = uint32_t(r.per_rank.size());
  uint64_t nt = 0;
  for (auto& t : r.triples) nt += t.size();
  for (std::size_t p = 0; p < r.per_rank.size() && p < RDMM_H_MAX_RANKS; ++p) {
    const auto& s = r.per_rank[p];
    out->multiplies[p] = s.multiplies;
    out->flops[p] = s.meter.flops;
    out->output_nnz[p] = s.meter.output_nnz;
    out->steals[p] = s.steals;
    out->steals_local[p] = s.steals_with_local_component;
    out->pushes[p] = s.queue_pushes;
    out->pops[p] = s.queue_pops;
    out->bytes_self[p] = s.bytes_self;
    out->bytes_on_node[p] = s.bytes_on_node;
    out->bytes_off_node[p] = s.bytes_off_node;
    out->total_seconds[p] = s.total_seconds;
  }
  std::size_t ns = 0;
  bool timed = false;
  for (auto& s : r.per_rank) {
    ns = std::max(ns, std::max(s.stage_flops.size(), s.stage_ms.size()));
    timed |= !s.stage_ms.empty();
  }
  out->nstages = uint32_t(ns);
  if (ns && !r.per_rank.empty()) {
    out->stage_flops =
        static_cast<uint64_t*>(std::calloc(r.per_rank.size() * ns, sizeof(uint64_t)));
    for (std::size_t p = 0; p < r.per_rank.size(); ++p)
      std::copy(r.per_rank[p].stage_flops.begin(), r.per_rank[p].stage_flops.end(),
                out->stage_flops + p * ns);
    if (timed) {
      out->stage_ms = static_cast<double*>(std::calloc(r.per_rank.size() * ns, sizeof(double)));
      for (std::size_t p = 0; p < r.per_rank.size(); ++p)
        std::copy(r.per_rank[p].stage_ms.begin(), r.per_rank[p].stage_ms.end(),
                  out->stage_ms + p * ns);
    }
  }
  out->ntriples = nt;
  if (nt) {
    out->triples = static_cast<uint32_t*>(std::malloc(nt * 16));
    uint64_t q = 0;
    for (std::size_t p = 0; p < r.triples.size(); ++p)
      for (auto& t : r.triples[p]) {
        out->triples[4 * q + 0] = uint32_t(p);
        out->triples[4 * q + 1] = t.i;
        out->triples[4 * q + 2] = t.j;
        out->triples[4 * q + 3] = t.k;
        ++q;
      }
  }
}

template <typename T>
void run_typed(rdmm_h_fabric* f, rdmm_h_matrix* A, rdmm_h_matrix* B, rdmm_h_matrix* C,
               const RunOptions& o, rdmm_h_report* rep) {
  auto& a = *std::get<std::unique_ptr<DistSparse<T>>>(A->m);
  RunReport r;
  if (B->kind == 1) {
    auto& b = *std::get<std::unique_ptr<DistDense<T>>>(B->m);
    auto& c = *std::get<std::unique_ptr<DistDense<T>>>(C->m);
    r = run_multiply(*f->f, a, b, c, o);
  } else {
    auto& b = *std::get<std::unique_ptr<DistSparse<T>>>(B->m);
    auto& c = *std::get<std::unique_ptr<DistSparse<T>>>(C->m);
    r = run_multiply(*f->f, a, b, c, o);
  }
  fill(r, rep);
}

}  // namespace

extern "C" int rdmm_h_fabric_create(uint32_t nranks, uint64_t heap_bytes, uint32_t node_group,
                                    uint64_t queue_capacity, uint32_t first_local,
                                    uint32_t nlocal, const int* devices, const char* session,
                                    rdmm_h_fabric** out) {
  *out = nullptr;
  return guarded([&] {
    FabricConfig c;
    c.nranks = nranks;
    c.heap_bytes = heap_bytes;
    c.node_group = node_group ? node_group : 6;
    c.queue_capacity = queue_capacity ? queue_capacity : 4096;
    c.first_local = first_local;
    c.nlocal = nlocal;
    if (devices) c.devices.assign(devices, devices + (nlocal ? nlocal : nranks));
    if (session) c.session = session;
    auto h = std::make_unique<rdmm_h_fabric>();
    h->f = std::make_unique<Fabric>(c);
    *out = h.release();
  });
}

extern "C" void rdmm_h_fabric_destroy(rdmm_h_fabric* f) { delete f; }
extern "C" void* rdmm_h_fabric_handle(rdmm_h_fabric* f) { return f->f->handle(); }

extern "C" int rdmm_h_matrix_create(rdmm_h_fabric* f, int kind, int dtype, uint64_t m, uint64_t n,
                                    uint32_t tm, uint32_t tn, uint32_t pr, uint32_t pc,
                                    int matrix_id, rdmm_h_matrix** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<rdmm_h_matrix>();
    h->fab = f;
    h->kind = kind;
    h->dtype = dtype;
    ProcGrid g{pr, pc};
    if (kind == 0 && dtype == 8)
      h->m = std::make_unique<DistSparse<double>>(*f->f, m, n, tm, tn, g, matrix_id);
    else if (kind == 0)
      h->m = std::make_unique<DistSparse<float>>(*f->f, m, n, tm, tn, g, matrix_id);
    else if (dtype == 8)
      h->m = std::make_unique<DistDense<double>>(*f->f, m, n, tm, tn, g, matrix_id);
    else
      h->m = std::make_unique<DistDense<float>>(*f->f, m, n, tm, tn, g, matrix_id);
    *out = h.release();
  });
}

extern "C" void rdmm_h_matrix_destroy(rdmm_h_matrix* mat) { delete mat; }

extern "C" int rdmm_h_sparse_init(rdmm_h_matrix* mat, const uint32_t* rp, const uint32_t* ci,
                                  const void* vals, uint64_t nnz, int on_device) {
  return guarded([&] {
    if (mat->kind != 0) throw std::invalid_argument("not a sparse matrix");
    if (mat->dtype == 8)
      sparse_init(*mat->fab->f, *std::get<std::unique_ptr<DistSparse<double>>>(mat->m), rp, ci,
                  vals, nnz, on_device);
    else
      sparse_init(*mat->fab->f, *std::get<std::unique_ptr<DistSparse<float>>>(mat->m), rp, ci,
                  vals, nnz, on_device);
  });
}

extern "C" int rdmm_h_dense_init(rdmm_h_matrix* mat, const void* global, uint64_t ld) {
  return guarded([&] {
    if (mat->kind != 1) throw std::invalid_argument("not a dense matrix");
    if (mat->dtype == 8)
      dense_init(*mat->fab->f, *std::get<std::unique_ptr<DistDense<double>>>(mat->m), global, ld);
    else
      dense_init(*mat->fab->f, *std::get<std::unique_ptr<DistDense<float>>>(mat->m), global, ld);
  });
}

extern "C" int rdmm_h_dense_to_host(rdmm_h_matrix* mat, void* out) {
  return guarded([&] {
    if (mat->dtype == 8) {
      auto g = std::get<std::unique_ptr<DistDense<double>>>(mat->m)->to_global();
      std::memcpy(out, g.data(), g.size() * 8);
    } else {
      auto g = std::get<std::unique_ptr<DistDense<float>>>(mat->m)->to_global();
      std::memcpy(out, g.data(), g.size() * 4);
    }
  });
}

extern "C" int rdmm_h_sparse_nnz(rdmm_h_matrix* mat, uint64_t* nnz) {
  return guarded([&] {
    uint64_t n = 0;
    auto count = [&](auto& A) {
      for (uint32_t i = 0; i < A.tile_grid_rows(); ++i)
        for (uint32_t j = 0; j < A.tile_grid_cols(); ++j) n += A.tile_nnz(i, j);
    };
    if (mat->dtype == 8)
      count(*std::get<std::unique_ptr<DistSparse<double>>>(mat->m));
    else
      count(*std::get<std::unique_ptr<DistSparse<float>>>(mat->m));
    *nnz = n;
  });
}

extern "C" int rdmm_h_sparse_to_host(rdmm_h_matrix* mat, uint32_t* rp, uint32_t* ci,
                                     void* vals) {
  return guarded([&] {
    auto out = [&](auto g) {
      std::memcpy(rp, g.row_ptr.data(), g.row_ptr.size() * 4);
      std::memcpy(ci, g.col_idx.data(), g.col_idx.size() * 4);
      std::memcpy(vals, g.values.data(), g.values.size() * sizeof(g.values[0]));
    };
    if (mat->dtype == 8)
      out(std::get<std::unique_ptr<DistSparse<double>>>(mat->m)->to_global());
    else
      out(std::get<std::unique_ptr<DistSparse<float>>>(mat->m)->to_global());
  });
}

extern "C" int rdmm_h_run_multiply(rdmm_h_fabric* f, rdmm_h_matrix* A, rdmm_h_matrix* B,
                                   rdmm_h_matrix* C, const rdmm_h_options* o,
                                   rdmm_h_report* rep) {
  return guarded([&] {
    if (A->kind != 0) throw std::invalid_argument("A must be sparse");
    if (B->kind != C->kind) throw std::invalid_argument("B and C must be both dense or sparse");
    if (A->dtype != B->dtype || A->dtype != C->dtype) throw std::invalid_argument("dtype mismatch");
    const RunOptions ro = opts_of(o);
    if (A->dtype == 8)
      run_typed<double>(f, A, B, C, ro, rep);
    else
      run_typed<float>(f, A, B, C, ro, rep);
  });
}

extern "C" void rdmm_h_free(void* p) { std::free(p); }

extern "C" int rdmm_h_dense_zero(rdmm_h_matrix* mat) {
  return guarded([&] {
    if (mat->kind != 1) throw std::invalid_argument("not a dense matrix");
    if (mat->dtype == 8) {
      auto& m = *std::get<std::unique_ptr<DistDense<double>>>(mat->m);
      run_ranks(*mat->fab->f, [&](RankCtx& ctx) { m.zero(ctx); });
    } else {
      auto& m = *std::get<std::unique_ptr<DistDense<float>>>(mat->m);
      run_ranks(*mat->fab->f, [&](RankCtx& ctx) { m.zero(ctx); });
    }
  });
}

extern "C" int rdmm_h_dense_owned_to_host(rdmm_h_matrix* mat, void* global, uint64_t ld) {
  return guarded([&] {
    if (mat->kind != 1) throw std::invalid_argument("not a dense matrix");
    if (mat->dtype == 8) {
      auto& m = *std::get<std::unique_ptr<DistDense<double>>>(mat->m);
      run_ranks(*mat->fab->f,
                [&](RankCtx& ctx) { m.owned_to_host(ctx, static_cast<double*>(global), ld); });
    } else {
      auto& m = *std::get<std::unique_ptr<DistDense<float>>>(mat->m);
      run_ranks(*mat->fab->f,
                [&](RankCtx& ctx) { m.owned_to_host(ctx, static_cast<float*>(global), ld); });
    }
  });
}

extern "C" int rdmm_h_dense_owned_to_host_async(rdmm_h_matrix* mat, void* global, uint64_t ld,
                                                void* stream) {
  return guarded([&] {
    if (mat->kind != 1) throw std::invalid_argument("not a dense matrix");
    if (!stream) throw std::invalid_argument("owned_to_host_async: a stream is required");
    auto* s = static_cast<rdmm_stream_t>(stream);
    if (mat->dtype == 8) {
      auto& m = *std::get<std::unique_ptr<DistDense<double>>>(mat->m);
      run_ranks(*mat->fab->f,
                [&](RankCtx& ctx) { m.owned_to_host(ctx, static_cast<double*>(global), ld, s); });
    } else {
      auto& m = *std::get<std::unique_ptr<DistDense<float>>>(mat->m);
      run_ranks(*mat->fab->f,
                [&](RankCtx& ctx) { m.owned_to_host(ctx, static_cast<float*>(global), ld, s); });
    }
  });
}

extern "C" int rdmm_h_sparse_owned_to_host(rdmm_h_matrix* mat, void* buf, uint64_t cap,
                                           uint64_t* bytes) {
  return guarded([&] {
    if (mat->kind != 0) throw std::invalid_argument("not a sparse matrix");
    std::atomic<uint64_t> total{0};
    auto go = [&](auto& m) {
      // local ranks write disjoint consecutive slices of buf
      std::vector<uint64_t> off(mat->fab->f->nlocal() + 1, 0);
      for (rank_t i = 0; i < mat->fab->f->nlocal(); ++i)
        off[i + 1] = off[i] + m.owned_bytes(mat->fab->f->first_local() + i);
      if (!buf) {
        total = off.back();
        return;
      }
      if (off.back() > cap) throw std::invalid_argument("owned_to_host: buffer too small");
      run_ranks(*mat->fab->f, [&](RankCtx& ctx) {
        const rank_t i = ctx.rank() - mat->fab->f->first_local();
        total += m.owned_to_host(ctx, static_cast<char*>(buf) + off[i], off[i + 1] - off[i]);
      });
    };
    if (mat->dtype == 8)
      go(*std::get<std::unique_ptr<DistSparse<double>>>(mat->m));
    else
      go(*std::get<std::unique_ptr<DistSparse<float>>>(mat->m));
    *bytes = total;
  });
}

extern "C" void* rdmm_h_fabric_stream(rdmm_h_fabric* f, uint32_t rank) {
  return rdmm_fabric_stream(f->f->handle(), rank, 0);
}

namespace {
template <typename T>
void mm_read(const char* path, uint32_t* rows, uint32_t* cols, uint64_t* nnz, uint32_t** rp,
             uint32_t** ci, void** vals) {
  CsrTile<T> t = read_matrix_market<T>(path);
  *rows = t.rows;
  *cols = t.cols;
  *nnz = t.col_idx.size();
  auto dup = [](const auto& v) {
    using E = typename std::decay_t<decltype(v)>::value_type;
    E* p = static_cast<E*>(std::malloc(std::max<std::size_t>(1, v.size()) * sizeof(E)));
    if (!p) throw std::bad_alloc();
    std::copy(v.begin(), v.end(), p);
    return p;
  };
  *rp = dup(t.row_ptr);
  *ci = dup(t.col_idx);
  *vals = dup(t.values);
}

template <typename T>
void mm_write(const char* path, uint32_t rows, uint32_t cols, const uint32_t* rp,
              const uint32_t* ci, const void* vals) {
  CsrTile<T> t(rows, cols);
  t.row_ptr.assign(rp, rp + rows + 1);
  t.col_idx.assign(ci, ci + rp[rows]);
  const T* v = static_cast<const T*>(vals);
  t.values.assign(v, v + rp[rows]);
  write_matrix_market(t, path);
}
}  // namespace

extern "C" int rdmm_h_read_matrix_market(const char* path, int dtype_bytes, uint32_t* rows,
                                         uint32_t* cols, uint64_t* nnz, uint32_t** row_ptr,
                                         uint32_t** col_idx, void** values) {
  return guarded([&] {
    if (dtype_bytes == 8)
      mm_read<double>(path, rows, cols, nnz, row_ptr, col_idx, values);
    else if (dtype_bytes == 4)
      mm_read<float>(path, rows, cols, nnz, row_ptr, col_idx, values);
    else
      throw std::invalid_argument("dtype_bytes must be 4 or 8");
  });
}

extern "C" int rdmm_h_write_matrix_market(const char* path, int dtype_bytes, uint32_t rows,
                                          uint32_t cols, const uint32_t* row_ptr,
                                          const uint32_t* col_idx, const void* values) {
  return guarded([&] {
    if (dtype_bytes == 8)
      mm_write<double>(path, rows, cols, row_ptr, col_idx, values);
    else if (dtype_bytes == 4)
      mm_write<float>(path, rows, cols, row_ptr, col_idx, values);
    else
      throw std::invalid_argument("dtype_bytes must be 4 or 8");
  });
}
