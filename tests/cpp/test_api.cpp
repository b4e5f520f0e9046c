// C++ drop-in API tests: the reference's own test shapes
// (/root/reference/proj/tests/test_fabric.cpp, test_distmat.cpp,
// test_algos.cpp) written against include/rdmm/*.hpp and run on the GPU.
// Built by tests/test_cpp_gpu.py; prints one line per check and exits
// non-zero on the first failure.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <string>

#include "rdmm/algos.hpp"
#include "rdmm/analytics.hpp"

using namespace rdmm;

static int g_checks = 0;
#define REQUIRE(...)                                                          \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(__VA_ARGS__)) {                                                     \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)
#define RT_CHECK(...)                                                          \
  do {                                                                         \
    if (!(__VA_ARGS__)) throw std::runtime_error("rank check failed: " #__VA_ARGS__); \
  } while (0)
template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static FabricConfig cfg(rank_t p, std::size_t heap) {
  FabricConfig c;
  c.nranks = p;
  c.heap_bytes = heap;
  return c;
}

// gen.hpp:20-30 counter RNG (test inputs only)
static std::uint64_t sm64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
static std::uint64_t at(std::uint64_t s, std::uint64_t c) { return sm64(s * 0x2545f4914f6cdd1dull + c); }
static double u01(std::uint64_t s, std::uint64_t c) { return double(at(s, c) >> 11) * 0x1.0p-53; }
template <typename T>
CsrTile<T> random_csr(index_t rows, index_t cols, double d, std::uint64_t seed) {
  std::vector<std::tuple<index_t, index_t, T>> coo;
  std::uint64_t ctr = 0;
  for (index_t r = 0; r < rows; ++r)
    for (index_t c = 0; c < cols; ++c) {
      if (u01(seed, ctr++) < d) coo.emplace_back(r, c, T(1 + int(at(seed, ctr) % 3)));
      ++ctr;
    }
  return CsrTile<T>::from_coo(rows, cols, std::move(coo));
}
template <typename T>
DenseTile<T> random_dense(index_t rows, index_t cols, std::uint64_t seed) {
  DenseTile<T> t(rows, cols);
  std::uint64_t ctr = 0;
  for (auto& v : t.values) v = T(int(at(seed, ctr++) % 4));
  return t;
}
static std::vector<double> densify(const CsrTile<double>& t) {
  std::vector<double> d(std::size_t(t.rows) * t.cols, 0.0);
  for (index_t r = 0; r < t.rows; ++r)
    for (index_t s = t.row_ptr[r]; s < t.row_ptr[r + 1]; ++s) d[std::size_t(r) * t.cols + t.col_idx[s]] += t.values[s];
  return d;
}

// ------------------------------------------------------------------ fabric

static void test_fabric() {
  Fabric f(cfg(4, 1 << 20));
  // alloc / free / exhaustion (test_fabric.cpp:32-70)
  GlobalPtr p = f.alloc(1, 100);
  REQUIRE(p.rank == 1 && p.length == 100 && p.offset % 8 == 0);
  REQUIRE(f.heap_remaining(1) == (1u << 20) - 104);
  f.free(p);
  REQUIRE(f.heap_remaining(1) == (1u << 20));
  REQUIRE(throws<heap_exhausted_error>([&] { f.alloc(0, 2 << 20); }));
  REQUIRE(throws<fabric_error>([&] { f.free(p); }));
  // put/get accounting + one-sidedness (test_fabric.cpp:72-102, 297-313)
  f.traffic().clear();
  run_ranks(f, [&](RankCtx& ctx) {
    if (ctx.rank() == 0) {
      GlobalPtr q = ctx.alloc(64);
      std::vector<std::byte> buf(64, std::byte{7});
      ctx.put(buf, q);
      std::vector<std::byte> back(64);
      ctx.get(q, back);
      RT_CHECK(back == buf);
      ctx.free(q);
    }
    ctx.barrier();
  });
  auto t = f.traffic().pair_total(0, 0);
  REQUIRE(t.bytes_put == 64 && t.bytes_got == 64 && t.puts == 1 && t.gets == 1);
  // fetch_add linearisability across ranks (test_fabric.cpp:188-210)
  Fabric f8(cfg(8, 1 << 20));
  std::atomic<int> seen_mask_bad{0};
  std::vector<int> seen(8 * 100, 0);
  std::mutex mu;
  run_ranks(f8, [&](RankCtx& ctx) {
    rdmm_gptr cell;
    check(rdmm_ctrl_cells(ctx.h(), ctx.rank(), 0xC0FFEE, 1, &cell), "cells");
    ctx.barrier();
    for (int n = 0; n < 100; ++n) {
      std::int64_t v = ctx.fetch_add(GlobalPtr::of(cell), 1);
      std::scoped_lock lk(mu);
      if (v < 0 || v >= 800 || seen[v]) seen_mask_bad = 1;
      else seen[v] = 1;
    }
    ctx.barrier();
    rdmm_ctrl_release(ctx.h(), ctx.rank(), 0xC0FFEE);
  });
  REQUIRE(seen_mask_bad == 0);
  for (int v : seen) REQUIRE(v == 1);
  // queues: exactly-once delivery (test_fabric.cpp:250-278)
  std::vector<int> got(4 * 50, 0);
  run_ranks(f, [&](RankCtx& ctx) {
    std::vector<std::uint64_t> q(4);
    check(rdmm_queue_open(ctx.h(), ctx.rank(), 0xABC, 1024, q.data()), "q");
    ctx.barrier();
    for (int n = 0; n < 50; ++n)
      ctx.queue_push(q[0], GlobalPtr{ctx.rank(), std::uint64_t(n), 0});
    ctx.barrier();
    if (ctx.rank() == 0) {
      while (auto e = ctx.queue_pop(q[0])) got[e->rank * 50 + e->offset]++;
    } else {
      RT_CHECK(throws<fabric_error>([&] { ctx.queue_pop(q[0]); }));
    }
    ctx.barrier();
    rdmm_ctrl_release(ctx.h(), ctx.rank(), 0xABC);
  });
  for (int v : got) REQUIRE(v == 1);
  // rank failure propagates instead of deadlocking peers in a barrier
  Fabric fx(cfg(2, 1 << 20));
  REQUIRE(throws<std::runtime_error>([&] {
    run_ranks(fx, [&](RankCtx& ctx) {
      if (ctx.rank() == 1) throw std::runtime_error("boom");
      ctx.barrier();
    });
  }));
  std::printf("fabric: ok\n");
}

// ------------------------------------------------------------------ distmat

static void test_distmat() {
  // ProcGrid mapping and edge tiles (test_distmat.cpp:37-64)
  ProcGrid g{2, 3};
  REQUIRE(g.owner(0, 0) == 0 && g.owner(1, 2) == 5 && g.owner(2, 4) == 1);
  detail::TileGeom geom(10, 7, 4, 3);
  REQUIRE(geom.M == 3 && geom.N == 3 && geom.tile_rows(2) == 2 && geom.tile_cols(2) == 1);
  Fabric f(cfg(4, 4 << 20));
  ProcGrid g2{2, 2};
  auto ga = random_csr<double>(10, 7, 0.4, 3);
  auto gb = random_dense<double>(10, 7, 4);
  DistSparse<double> A(f, 10, 7, 4, 3, g2, 0);
  DistDense<double> B(f, 10, 7, 4, 3, g2, 1);
  run_ranks(f, [&](RankCtx& ctx) {
    A.init_from_global(ctx, ga);
    B.init_from_global(ctx, gb.values);
  });
  REQUIRE(B.to_global() == gb.values);
  auto back = A.to_global();
  REQUIRE(back.row_ptr == ga.row_ptr && back.col_idx == ga.col_idx && back.values == ga.values);
  // 1 get per dense tile, 3 per sparse tile (test_distmat.cpp:66-174)
  f.traffic().clear();
  run_ranks(f, [&](RankCtx& ctx) {
    if (ctx.rank() != 3) return;
    auto d = B.get_tile(ctx, 0, 0);  // owner 0
    auto s = A.get_tile(ctx, 0, 0);
    RT_CHECK(d.rows == 4 && d.cols == 3 && s.nnz == A.tile_nnz(0, 0));
  });
  auto tr = f.traffic().pair_total(0, 3);
  REQUIRE(tr.gets == 4);
  // replace + renew (test_distmat.cpp:176-212)
  run_ranks(f, [&](RankCtx& ctx) {
    if (ctx.rank() == 0) {
      CsrTile<double> t(4, 3);
      t.col_idx = {1};
      t.values = {9.0};
      t.row_ptr = {0, 1, 1, 1, 1};
      A.replace_tile(ctx, 0, 0, t);
    }
    A.renew_tiles(ctx);
  });
  REQUIRE(A.tile_nnz(0, 0) == 1);
  REQUIRE(throws<fabric_error>([&] {
    run_ranks(f, [&](RankCtx& ctx) {
      if (ctx.rank() == 1) A.tile_ref(ctx, 0, 0);
    });
  }));
  std::printf("distmat: ok\n");
}

// ------------------------------------------------------------------ algos

static void test_algos() {
  constexpr std::uint64_t kM = 12, kK = 9, kN = 10;
  constexpr std::uint32_t kTm = 4, kTk = 3, kTn = 4;
  const Variant all[] = {Variant::summa_bsp, Variant::stationary_c, Variant::stationary_a,
                         Variant::stationary_b, Variant::ws_random, Variant::ws_locality};
  auto ga = random_csr<double>(kM, kK, 0.35, 5);
  auto gb = random_dense<double>(kK, kN, 6);
  auto gc0 = random_dense<double>(kM, kN, 7);
  auto ad = densify(ga);
  std::vector<double> want = gc0.values;
  for (std::uint64_t i = 0; i < kM; ++i)
    for (std::uint64_t l = 0; l < kK; ++l)
      for (std::uint64_t j = 0; j < kN; ++j) want[i * kN + j] += ad[i * kK + l] * gb.values[l * kN + j];
  auto sb = random_csr<double>(kK, kN, 0.35, 16);
  auto sc0 = random_csr<double>(kM, kN, 0.15, 17);
  auto bd = densify(sb), c0d = densify(sc0);
  std::vector<double> swant = c0d;
  for (std::uint64_t i = 0; i < kM; ++i)
    for (std::uint64_t l = 0; l < kK; ++l)
      for (std::uint64_t j = 0; j < kN; ++j) swant[i * kN + j] += ad[i * kK + l] * bd[l * kN + j];
  for (Variant v : all) {
    // SpMM (test_algos.cpp:98-109)
    {
      Fabric f(cfg(4, 4 << 20));
      ProcGrid g{2, 2};
      DistSparse<double> A(f, kM, kK, kTm, kTk, g, 0);
      DistDense<double> B(f, kK, kN, kTk, kTn, g, 1);
      DistDense<double> C(f, kM, kN, kTm, kTn, g, 2);
      run_ranks(f, [&](RankCtx& ctx) {
        A.init_from_global(ctx, ga);
        B.init_from_global(ctx, gb.values);
        C.init_from_global(ctx, gc0.values);
      });
      RunOptions o;
      o.variant = v;
      o.record_triples = true;
      RunReport rep = run_multiply(f, A, B, C, o);
      REQUIRE(C.to_global() == want);
      std::set<Triple> tr;
      for (auto& pr : rep.triples) tr.insert(pr.begin(), pr.end());
      REQUIRE(tr.size() == 27 && rep.total_multiplies() == 27);
      REQUIRE(rep.checksum == matrix_checksum(C));
      // analytics.hpp:66-90 over the run's own per-k-step flop table
      ImbalanceReport imb = run_imbalance(rep);
      std::uint64_t staged = 0;
      for (auto& r : imb.stage_flops)
        for (auto x : r) staged += x;
      REQUIRE(staged == rep.total_flops() && imb.stage_flops.size() == 4);
      REQUIRE(imb.per_stage_flop_imbalance + 1e-12 >= imb.end_to_end_flop_imbalance);
      REQUIRE(imb.end_to_end_flop_imbalance >= 1.0);
    }
    // SpGEMM
    {
      Fabric f(cfg(4, 4 << 20));
      ProcGrid g{2, 2};
      DistSparse<double> A(f, kM, kK, kTm, kTk, g, 0);
      DistSparse<double> B(f, kK, kN, kTk, kTn, g, 1);
      DistSparse<double> C(f, kM, kN, kTm, kTn, g, 2);
      run_ranks(f, [&](RankCtx& ctx) {
        A.init_from_global(ctx, ga);
        B.init_from_global(ctx, sb);
        C.init_from_global(ctx, sc0);
      });
      RunOptions o;
      o.variant = v;
      run_multiply(f, A, B, C, o);
      auto out = C.to_global();
      REQUIRE(out.well_formed());
      REQUIRE(densify(out) == swant);
    }
    std::printf("algos %s: ok\n", variant_name(v));
  }
  // malformed configurations (test_algos.cpp:228-276)
  Fabric f(cfg(4, 1 << 20));
  ProcGrid g{2, 2};
  DistSparse<double> A(f, 8, 8, 4, 4, g);
  DistDense<double> B(f, 6, 8, 3, 4, g);
  DistDense<double> C(f, 8, 8, 4, 4, g);
  run_ranks(f, [&](RankCtx& ctx) {
    A.init(ctx);
    B.init(ctx);
    C.init(ctx);
  });
  RunOptions o;
  o.variant = Variant::summa_bsp;
  REQUIRE(throws<dimension_error>([&] { run_multiply(f, A, B, C, o); }));
}

int main() {
  test_fabric();
  test_distmat();
  test_algos();
  std::printf("all %d checks passed\n", g_checks);
  return 0;
}
