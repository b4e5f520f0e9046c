// spmm.cu -- C += A*B for CSR A and row-major tall-skinny B on sm_100a.
//
// Reference: spmm_local, /root/reference/proj/include/rdmm/tile.hpp:170-188
// (scalar triple loop, one B-row gather per nonzero, k ascending).
//
// B200 design (memory-bound, CUDA cores):
//  * nnz-balanced chunks.  The nonzeros are cut into `nchunks` equal ranges
//    of Q; a worker (a group of G lanes) owns whole chunks, so hub rows of
//    R-MAT (32K nnz at scale 22) are spread over many workers and 41% empty
//    rows cost nothing.  A row wholly inside a chunk is accumulated in the
//    reference order starting from C (fma chain) and stored once -> bitwise
//    equal to the reference for any values.  A row cut by chunk boundaries
//    leaves per-chunk partials (the first one seeded with C); a fix-up pass
//    adds them in ascending chunk order -> deterministic.
//  * One 512-B row of B per nonzero is gathered as 32 lanes x 16 B
//    (float4 / double2) through the read-only path, U=8 gathers in flight per
//    worker before the fused multiply-adds.
//  * col_idx/val are read 32 at a time (one coalesced load per lane) and
//    broadcast with shuffles.
#include <algorithm>
#include <atomic>

#include <cstdlib>
#include <string>

#include "common.cuh"

namespace rdmm_impl {
namespace {

template <typename T, int VEC>
struct VecOf;
template <>
struct VecOf<float, 4> {
  using type = float4;
};
template <>
struct VecOf<double, 2> {
  using type = double2;
};
// 32-byte vectors: one 256-bit load per lane (LDG.E.ENL2.256 on sm_100a).
struct __align__(32) float8 {
  float4 lo, hi;
};
struct __align__(32) double4x {
  double2 lo, hi;
};
template <>
struct VecOf<float, 8> {
  using type = float8;
};
template <>
struct VecOf<double, 4> {
  using type = double4x;
};
template <>
struct VecOf<float, 1> {
  using type = float;
};
template <>
struct VecOf<double, 1> {
  using type = double;
};

__device__ __forceinline__ float4 vfma(float a, float4 b, float4 c) {
  return make_float4(fmaf(a, b.x, c.x), fmaf(a, b.y, c.y), fmaf(a, b.z, c.z),
                     fmaf(a, b.w, c.w));
}
__device__ __forceinline__ double2 vfma(double a, double2 b, double2 c) {
  return make_double2(fma(a, b.x, c.x), fma(a, b.y, c.y));
}
__device__ __forceinline__ float8 vfma(float a, float8 b, float8 c) {
  return float8{vfma(a, b.lo, c.lo), vfma(a, b.hi, c.hi)};
}
__device__ __forceinline__ double4x vfma(double a, double4x b, double4x c) {
  return double4x{vfma(a, b.lo, c.lo), vfma(a, b.hi, c.hi)};
}
__device__ __forceinline__ float vfma(float a, float b, float c) {
  return fmaf(a, b, c);
}
__device__ __forceinline__ double vfma(double a, double b, double c) {
  return fma(a, b, c);
}
__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ double2 vadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ float8 vadd(float8 a, float8 b) {
  return float8{vadd(a.lo, b.lo), vadd(a.hi, b.hi)};
}
__device__ __forceinline__ double4x vadd(double4x a, double4x b) {
  return double4x{vadd(a.lo, b.lo), vadd(a.hi, b.hi)};
}
__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
__device__ __forceinline__ double vadd(double a, double b) { return a + b; }
__device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) {
  return a < b ? a : b;
}
__device__ __forceinline__ uint64_t umax(uint64_t a, uint64_t b) {
  return a > b ? a : b;
}
// Read-only gather of one vector (256-bit loads for the 32-byte types).
template <typename V>
__device__ __forceinline__ V ldg_v(const V* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float8 ldg_v(const float8* p) {
  float8 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.lo.x), "=f"(r.lo.y), "=f"(r.lo.z), "=f"(r.lo.w), "=f"(r.hi.x),
                 "=f"(r.hi.y), "=f"(r.hi.z), "=f"(r.hi.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ double4x ldg_v(const double4x* p) {
  double4x r;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.lo.x), "=d"(r.lo.y), "=d"(r.hi.x), "=d"(r.hi.y)
               : "l"(p));
  return r;
}
template <typename V>
__device__ __forceinline__ V vzero() {
  V v;
  memset(&v, 0, sizeof(V));
  return v;
}

template <typename T>
struct SpmmArgs {
  const uint32_t* __restrict__ rp;
  const uint32_t* __restrict__ ci;
  const T* __restrict__ val;
  const T* __restrict__ B;
  T* __restrict__ C;
  T* __restrict__ head_val;  // [nchunks][wstride]
  T* __restrict__ tail_val;  // [nchunks][wstride]
  int32_t* __restrict__ tail_row;  // [nchunks]
  const uint32_t* __restrict__ chunk_row;  // [nchunks] row holding nonzero c*Q
  // RDMM_SPMM_NNZ_ON_DEVICE: nnz = *dyn_end (= rp[rows]) read by the kernels,
  // nchunks an upper bound and Q derived on the device (no host round trip)
  const uint32_t* __restrict__ dyn_end;
  // RDMM_SPMM_ATOMIC (narrow slot kernels): every row flush, including the
  // pieces of rows cut by chunk boundaries, is a red.global.add into C; no
  // C read, no head/tail fix-up, products of several launches may overlap
  int atomic;
  // spmm_stream_full may run: rows of exactly 32 16-byte vectors, one
  // contiguous B, B/C vector indices and chunk positions within 32 bits
  int full_ok;
  uint64_t ldb, ldc;
  uint64_t nnz, Q;
  uint32_t rows, nvec, nchunks, wstride;
  // Segmented B (fused K-tile products): B row g lives in segment
  // g / seg_rows at row g % seg_rows; nseg == 0 means one contiguous B.
  const T* bseg[16];
  uint64_t boff;  // element offset applied to every segment (column panel)
  uint32_t nseg, seg_rows, seg_shift;
};


// Segment base pointers staged in shared memory once per CTA (indexing the
// kernel-parameter array with a runtime segment number forces a local copy).
template <typename T>
struct SegTable {
  const T* base[16];
};

template <typename T, bool SEG>
__device__ __forceinline__ void load_segs(const SpmmArgs<T>& p, SegTable<T>& st) {
  if constexpr (SEG) {
    if (threadIdx.x < 16) st.base[threadIdx.x] = p.bseg[threadIdx.x] + p.boff;
    __syncthreads();
  }
}

template <typename T, typename V, bool SEG>
__device__ __forceinline__ const V* brow_ptr(const SpmmArgs<T>& p, const SegTable<T>& st,
                                             const V* Bv, uint32_t k, uint64_t ldbv,
                                             uint32_t voff) {
  if constexpr (!SEG) return Bv + uint64_t(k) * ldbv + voff;
  const uint32_t sg = p.seg_shift < 32 ? (k >> p.seg_shift) : (k / p.seg_rows);
  const uint32_t r = k - sg * p.seg_rows;
  return reinterpret_cast<const V*>(st.base[sg]) + uint64_t(r) * ldbv + voff;
}

// arr[idx] for a runtime idx without dynamic register indexing (which would
// put the array in local memory): unrolled predicated selects.
template <int SL, typename X>
__device__ __forceinline__ X sel(const X (&arr)[SL], uint32_t idx) {
  X v = arr[0];
#pragma unroll
  for (int j = 1; j < SL; ++j)
    if (idx == uint32_t(j)) v = arr[j];
  return v;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << G) - 1u) << (lane / G * G);
  }
}

constexpr int kThreads = 256;
constexpr int kMaxDevices = 64;
constexpr int kWin = 32;  // nonzeros staged per window
constexpr int kU = 8;     // B-row gathers in flight per worker

// Index of the first of the 32 window rows [rb, rb+32) whose end exceeds pos
// (the row holding nonzero `pos`); 32 if every window row ends <= pos.
template <int G, int SL>
__device__ __forceinline__ uint32_t rows_done(const uint32_t (&rew)[SL],
                                              uint64_t pos, unsigned gm) {
  uint32_t n = 0;
#pragma unroll
  for (int j = 0; j < SL; ++j)
    n += __popc(__ballot_sync(gm, uint64_t(rew[j]) <= pos) & gm);
  return n;
}

template <int G, int SL>
__device__ __forceinline__ uint32_t win_get(const uint32_t (&rew)[SL],
                                            uint32_t idx, unsigned gm) {
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < SL; ++j) {
    const uint32_t x = __shfl_sync(gm, rew[j], idx % G, G);
    if (idx / G == uint32_t(j)) v = x;
  }
  return v;
}

template <int G, int SL>
__device__ __forceinline__ void win_load(uint32_t (&rew)[SL],
                                         const uint32_t* __restrict__ rp,
                                         uint32_t rb, uint32_t rows,
                                         uint32_t lane) {
#pragma unroll
  for (int j = 0; j < SL; ++j) {
    const uint32_t rr = rb + lane + G * j;  // row whose end we hold
    rew[j] = rr < rows ? __ldg(rp + rr + 1) : 0xFFFFFFFFu;
  }
}

// Stream one nnz chunk [lo, hi): the chunk's nonzeros are consumed 32 at a
// time regardless of row boundaries (col/val of the next window load while
// the current window's gathers are in flight), rows are
// tracked through a 32-entry window of row ends held in registers, and a row
// is flushed to C (or to a carry slot if the chunk cuts it) when the stream
// crosses its end.  CZERO: C is known to be zero on entry (first product
// into a fresh tile), so C is written but never read.
template <typename T, int VEC, int G, int NV, bool CZERO, int MINB, bool SEG>
__global__ void __launch_bounds__(kThreads, MINB)
    spmm_stream(const SpmmArgs<T> p) {
  using V = typename VecOf<T, VEC>::type;
  __shared__ SegTable<T> segs;
  load_segs<T, SEG>(p, segs);
  constexpr int SL = kWin / G;  // staged entries per lane
  const unsigned gm = group_mask<G>();
  const uint32_t lane = threadIdx.x % G;
  const uint32_t worker = (blockIdx.x * kThreads + threadIdx.x) / G;
  const uint32_t nworkers = gridDim.x * (kThreads / G);
  const V* __restrict__ Bv = reinterpret_cast<const V*>(p.B);
  V* __restrict__ Cv = reinterpret_cast<V*>(p.C);
  const uint64_t ldbv = p.ldb / VEC, ldcv = p.ldc / VEC;
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) colok[v] = lane + G * v < p.nvec;

  for (uint32_t c = worker; c < p.nchunks; c += nworkers) {
    const uint64_t lo = uint64_t(c) * p.Q;
    const uint64_t hi = umin(lo + p.Q, p.nnz);
    // row containing nonzero `lo` (spmm_chunk_rows)
    const uint32_t l = __ldg(p.chunk_row + c);
    uint32_t rb = l, row = l;
    uint32_t rew[SL];
    win_load<G, SL>(rew, p.rp, rb, p.rows, lane);
    bool starts = __ldg(p.rp + row) >= lo;
    uint32_t rend = win_get<G, SL>(rew, 0, gm);
    V acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      acc[v] = (!CZERO && starts && colok[v])
                   ? __ldcs(Cv + uint64_t(row) * ldcv + lane + G * v)
                   : vzero<V>();
    // first window of col/val
    uint32_t kk[SL];
    T aa[SL];
#pragma unroll
    for (int j = 0; j < SL; ++j) {
      const uint64_t idx = lo + lane + G * j;
      const bool ok = idx < hi;
      kk[j] = ok ? __ldcs(p.ci + idx) : 0u;
      aa[j] = ok ? __ldcs(p.val + idx) : T(0);
    }
    for (uint64_t w = lo; w < hi; w += kWin) {
      const uint32_t cnt = uint32_t(umin(kWin, hi - w));
      // next window's col/val (software pipelined one window ahead)
      uint32_t kn[SL];
      T an[SL];
#pragma unroll
      for (int j = 0; j < SL; ++j) {
        const uint64_t idx = w + kWin + lane + G * j;
        const bool ok = idx < hi;
        kn[j] = ok ? __ldcs(p.ci + idx) : 0u;
        an[j] = ok ? __ldcs(p.val + idx) : T(0);
      }
      // not unrolled: the row-flush code below would otherwise be inlined
      // kWin times (instruction-cache misses showed up as no_instruction
      // stalls in ncu)
#pragma unroll 1
      for (int t = 0; t < kWin; t += kU) {
        if (t < int(cnt)) {
          V bv[kU][NV];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int q = t + u;
            const uint32_t k = __shfl_sync(gm, sel<SL>(kk, q / G), q % G, G);
            if (q < int(cnt)) {
              const V* brow = brow_ptr<T, V, SEG>(p, segs, Bv, k, ldbv, lane);
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if (colok[v]) bv[u][v] = __ldg(brow + G * v);
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int q = t + u;
            const T a = __shfl_sync(gm, sel<SL>(aa, q / G), q % G, G);
            if (q < int(cnt)) {
              const uint64_t pos = w + q;
              if (pos >= rend) {
                // the stream crossed the end of `row`: it lies inside the
                // chunk, so flush to C (or to the head slot if the chunk
                // started inside it)
                if (starts) {
#pragma unroll
                  for (int v = 0; v < NV; ++v)
                    if (colok[v])
                      __stcs(Cv + uint64_t(row) * ldcv + lane + G * v, acc[v]);
                } else {
                  V* dst = reinterpret_cast<V*>(p.head_val) +
                           uint64_t(c) * (p.wstride / VEC);
#pragma unroll
                  for (int v = 0; v < NV; ++v)
                    if (colok[v]) dst[lane + G * v] = acc[v];
                }
                // next row holding `pos` (skips empty rows)
                for (;;) {
                  const uint32_t d = rows_done<G, SL>(rew, pos, gm);
                  if (d < uint32_t(kWin)) {
                    row = rb + d;
                    rend = win_get<G, SL>(rew, d, gm);
                    break;
                  }
                  rb += kWin;
                  win_load<G, SL>(rew, p.rp, rb, p.rows, lane);
                }
                starts = true;
#pragma unroll
                for (int v = 0; v < NV; ++v)
                  acc[v] = (!CZERO && colok[v])
                               ? __ldcs(Cv + uint64_t(row) * ldcv + lane + G * v)
                               : vzero<V>();
              }
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if (colok[v]) acc[v] = vfma(a, bv[u][v], acc[v]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < SL; ++j) {
        kk[j] = kn[j];
        aa[j] = an[j];
      }
    }
    // the chunk's last row
    int32_t trow = -1;
    if (rend <= hi && starts) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (colok[v]) __stcs(Cv + uint64_t(row) * ldcv + lane + G * v, acc[v]);
    } else {
      V* dst = reinterpret_cast<V*>(starts ? p.tail_val : p.head_val) +
               uint64_t(c) * (p.wstride / VEC);
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (colok[v]) dst[lane + G * v] = acc[v];
      if (starts) trow = int32_t(row);
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
}


// spmm_stream_full: the stream crossed the end of `row` at position pos --
// store it (or park it in the head slot when the chunk started inside it)
// and move to the row holding pos (skipping empty rows).
template <typename T, bool CZERO, typename V>
__device__ __forceinline__ void stream_next_row(const SpmmArgs<T>& p, V* __restrict__ Cl,
                                                uint32_t ldcv, uint32_t head_idx, uint32_t pos,
                                                uint32_t lane, uint32_t& rb, uint32_t& row,
                                                uint32_t& rew, uint32_t& rend, bool& starts,
                                                V& acc) {
  if (starts) __stcs(Cl + row * ldcv, acc);
  else reinterpret_cast<V*>(p.head_val)[head_idx] = acc;
  for (;;) {
    const uint32_t d = __popc(__ballot_sync(0xffffffffu, rew <= pos));
    if (d < 32u) {
      row = rb + d;
      rend = __shfl_sync(0xffffffffu, rew, d);
      break;
    }
    rb += 32;
    rew = rb + lane < p.rows ? __ldg(p.rp + rb + lane + 1) : 0xFFFFFFFFu;
  }
  starts = true;
  acc = CZERO ? vzero<V>() : __ldcs(Cl + row * ldcv);
}


// spmm_stream for the headline shape (rows of exactly 32 16-byte vectors:
// N = 128 fp32 / 64 fp64, one contiguous B): the same nnz-chunk stream with
// the per-nonzero instruction count cut from ~30 to ~10 -- every lane holds
// its window entry's B row offset (k * ldb, 32-bit) so a gather is one
// shuffle + one IMAD.WIDE + one LDG, positions are 32-bit, a full window
// (32 nonzeros) runs without bounds checks and no lane is masked.
template <typename T, bool CZERO>
__global__ void __launch_bounds__(kThreads, 4) spmm_stream_full(const SpmmArgs<T> p) {
  constexpr int VEC = 16 / sizeof(T);
  using V = typename VecOf<T, VEC>::type;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int U = 8;  // gathers in flight per lane
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = gridDim.x * (kThreads / 32);
  const V* __restrict__ Bl = reinterpret_cast<const V*>(p.B) + lane;
  V* __restrict__ Cl = reinterpret_cast<V*>(p.C) + lane;
  const uint32_t ldbv = uint32_t(p.ldb / VEC), ldcv = uint32_t(p.ldc / VEC);
  const uint32_t nnz = uint32_t(p.nnz), Q = uint32_t(p.Q);
  const uint32_t wsv = p.wstride / VEC;

  for (uint32_t c = warp; c < p.nchunks; c += nwarps) {
    const uint32_t lo = c * Q;
    const uint32_t hi = min(lo + Q, nnz);
    uint32_t rb = __ldg(p.chunk_row + c), row = rb;
    uint32_t rew = rb + lane < p.rows ? __ldg(p.rp + rb + lane + 1) : 0xFFFFFFFFu;
    bool starts = __ldg(p.rp + row) >= lo;
    uint32_t rend = __shfl_sync(FULL, rew, 0);
    V acc = (!CZERO && starts) ? __ldcs(Cl + row * ldcv) : vzero<V>();
    uint32_t off;
    T a;
    {
      const uint32_t idx = lo + lane;
      const bool ok = idx < hi;
      off = (ok ? __ldcs(p.ci + idx) : 0u) * ldbv;
      a = ok ? __ldcs(p.val + idx) : T(0);
    }
    for (uint32_t w = lo; w < hi; w += 32) {
      uint32_t kn;
      T an;
      {
        const uint32_t idx = w + 32 + lane;
        const bool ok = idx < hi;
        kn = ok ? __ldcs(p.ci + idx) : 0u;
        an = ok ? __ldcs(p.val + idx) : T(0);
      }
      // a partial last window gathers row 0 for its missing entries (off =
      // 0) and skips them: one code path, no per-gather bounds checks
#pragma unroll 1
      for (int t = 0; t < 32; t += U) {
        V bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) bv[u] = __ldg(Bl + __shfl_sync(FULL, off, t + u));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T au = __shfl_sync(FULL, a, t + u);
          const uint32_t pos = w + t + u;
          if (pos < hi) {
            if (pos >= rend)
              stream_next_row<T, CZERO>(p, Cl, ldcv, c * wsv + lane, pos, lane, rb, row, rew,
                                        rend, starts, acc);
            acc = vfma(au, bv[u], acc);
          }
        }
      }
      off = kn * ldbv;
      a = an;
    }
    // the chunk's last row
    int32_t trow = -1;
    if (rend <= hi && starts) {
      __stcs(Cl + row * ldcv, acc);
    } else {
      reinterpret_cast<V*>(starts ? p.tail_val : p.head_val)[c * wsv + lane] = acc;
      if (starts) trow = int32_t(row);
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
}




// Chunking of a launch: nnz, chunk length Q and chunk count, from the host
// plan or, with a device-resident nnz, derived on the device from the
// planned chunk count (an upper bound).
struct Chunking {
  uint32_t nnz, Q, nch;
};
__device__ __forceinline__ Chunking chunking(uint64_t nnz, uint64_t Q, uint32_t nchunks,
                                             const uint32_t* dyn_end) {
  if (!dyn_end) return {uint32_t(nnz), uint32_t(Q), nchunks};
  // at least 256 nonzeros per chunk: a small block gets fewer, longer chunks
  const uint32_t n = __ldg(dyn_end);
  const uint32_t q = max(256u, (n + nchunks - 1) / nchunks);
  return {n, q, n ? (n + q - 1) / q : 0u};
}
template <typename T>
__device__ __forceinline__ Chunking chunking(const SpmmArgs<T>& p) {
  return chunking(p.nnz, p.Q, p.nchunks, p.dyn_end);
}

// Chunk start rows: chunk c begins at nonzero c*Q, inside the row r with
// rp[r] <= c*Q < rp[r+1].  One coalesced pass over the row pointer replaces
// a 22-step dependent binary search per chunk in the SpMM kernels.
__global__ void spmm_chunk_rows(const uint32_t* __restrict__ rp, uint32_t rows, uint64_t Q0,
                                uint32_t nchunks, uint32_t* __restrict__ chunk_row,
                                const uint32_t* __restrict__ dyn_end) {
  const Chunking ck = chunking(0, Q0, nchunks, dyn_end);
  const uint64_t Q = dyn_end ? ck.Q : Q0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += gridDim.x * blockDim.x) {
    const uint64_t s = __ldg(rp + r), e = __ldg(rp + r + 1);
    for (uint64_t c = (s + Q - 1) / Q; c * Q < e && c < nchunks; ++c)
      chunk_row[c] = r;
  }
}

// cp.async (LDGSTS) helpers: 4/8-byte global -> shared copies that do not
// occupy registers while in flight; src_size 0 zero-fills.
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool ok, int bytes) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = ok ? bytes : 0;
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool ok) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Narrow rows (N < 128 fp32: a B row is L vectors of VEC elements, L < 32):
// the warp is ONE worker streaming its nnz chunks, split into S = 32/L slots
// of L lanes; a step feeds S consecutive nonzeros to the S slots (one B-row
// gather per slot, U steps = U gathers per lane in flight), so every row
// boundary is warp-uniform: no divergent per-group row flushes, and a step
// inside a row is U-independent FMAs with one compare.  The chunk's col/val
// stream is staged in a per-warp shared-memory ring NST windows ahead with
// cp.async (continuing across the warp's chunks), so the A stream's latency
// never stalls the gathers; the next chunk's start row is prefetched too.
// A row is accumulated as S slot partials and combined by a reduce-scatter
// over the slots when the stream crosses the row's end (each level halves
// the vector a lane keeps: log2(S) shuffles of VEC/2, VEC/4, ... elements);
// lane (slot, v) then owns elements [v*VEC + coff, +LEN) of the row and
// stores them.  Rows cut by chunk boundaries leave head/tail partials for
// spmm_fixup as in spmm_stream.  Summation order: fixed slot partials and
// tree, then C -- deterministic, exact for integer data, within the fp
// tolerance otherwise.
template <typename T, int VEC, int S, bool CZERO, int MINB, bool SEG>
__global__ void __launch_bounds__(kThreads, MINB)
    spmm_slots(const SpmmArgs<T> p) {
  using V = typename VecOf<T, VEC>::type;
  constexpr int L = 32 / S;                // lanes (vectors) per slot
  // steps per batch = gathers in flight per lane: 128 bytes of B per lane,
  // and at most 64 nonzeros per staged window
  constexpr int UB = sizeof(V) >= 32 ? 4 : 8;
  constexpr int U = UB * S > 64 ? 64 / S : UB;
  constexpr int STEP = S * U;              // nonzeros per batch
  constexpr int W = STEP > 32 ? STEP : 32; // nonzeros per staged window (<= 64)
  constexpr int SLW = W / 32;              // staged col/val per lane
  constexpr int NST = 4;                   // ring stages (windows in flight)
  constexpr int WARPS = kThreads / 32;
  constexpr int LOGS = S == 1 ? 0 : S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;
  constexpr int LOGV = VEC == 1 ? 0 : VEC == 2 ? 1 : VEC == 4 ? 2 : 3;
  constexpr int SCAT = LOGS < LOGV ? LOGS : LOGV;  // scatter levels
  constexpr int LEN = VEC >> SCAT;                 // elements a lane owns at the end
  __shared__ SegTable<T> segs;
  __shared__ uint32_t s_ci[WARPS][NST][W];
  __shared__ T s_val[WARPS][NST][W];
  load_segs<T, SEG>(p, segs);
  const uint32_t lane = threadIdx.x & 31u, slot = lane / L, v = lane % L;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = gridDim.x * WARPS;
  const V* __restrict__ Bv = reinterpret_cast<const V*>(p.B);
  T* __restrict__ Cs = p.C;
  const uint64_t ldbv = p.ldb / VEC;
  const bool colok = v < p.nvec;
  // element offset of this lane's share after the reduce-scatter, and
  // whether it stores (slots beyond the scatter levels hold copies)
  uint32_t coff = 0;
#pragma unroll
  for (int lv = 0; lv < SCAT; ++lv)
    if (slot & (1u << lv)) coff += VEC >> (lv + 1);
  const bool owner = colok && (slot >> SCAT) == 0;
  const uint32_t col0 = v * VEC + coff;  // first owned column within the row
  constexpr unsigned full = 0xffffffffu;
  // positions fit in 32 bits: row_ptr is uint32 (tile.hpp:17)
  const Chunking ck = chunking(p);
  const uint32_t nnz = ck.nnz, Q = ck.Q, nch = ck.nch;
  auto chunk_hi = [&](uint32_t c) { return uint32_t(umin(uint64_t(c) * Q + Q, nnz)); };

  // issue side of the ring: windows of the warp's chunks in consume order
  uint32_t ic = warp, iw = warp * Q, ist = 0;
  auto issue = [&]() {
    if (ic < nch) {
      const uint32_t h = chunk_hi(ic);
#pragma unroll
      for (int j = 0; j < SLW; ++j) {
        const uint32_t idx = iw + lane + 32 * j;
        const bool ok = idx < h;
        cp_async(&s_ci[wib][ist][lane + 32 * j], p.ci + (ok ? idx : 0), ok, 4);
        cp_async(&s_val[wib][ist][lane + 32 * j], p.val + (ok ? idx : 0), ok, int(sizeof(T)));
      }
      iw += W;
      if (iw >= h) {
        ic += nwarps;
        iw = ic * Q;
      }
    }
    cp_async_commit();
    ist = ist + 1 == NST ? 0 : ist + 1;
  };
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) issue();

  // reduce-scatter the S slot partials into out[0..LEN)
  auto reduce = [&](const V& acc, T (&out)[LEN]) {
    T r[VEC];
    const T* pa = reinterpret_cast<const T*>(&acc);
#pragma unroll
    for (int x = 0; x < VEC; ++x) r[x] = pa[x];
#pragma unroll
    for (int lv = 0; lv < LOGS; ++lv) {
      const int off = L << lv;
      if (lv < SCAT) {
        constexpr int dummy = 0;
        (void)dummy;
        const int half = VEC >> (lv + 1);
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int x = 0; x < VEC / 2; ++x) {
          if (x < half) {
            const T send = upper ? r[x] : r[x + half];
            const T keep = upper ? r[x + half] : r[x];
            r[x] = keep + __shfl_xor_sync(full, send, off);
          }
        }
      } else {
        r[0] += __shfl_xor_sync(full, r[0], off);
      }
    }
#pragma unroll
    for (int x = 0; x < LEN; ++x) out[x] = r[x];
  };
  // C's initial elements of this lane's share, loaded when the row starts
  // and added after the tree (the load's latency hides behind the gathers)
  auto cload = [&](uint32_t row, bool starts, T (&cin)[LEN]) {
#pragma unroll
    for (int x = 0; x < LEN; ++x)
      cin[x] = (!CZERO && !p.atomic && starts && owner)
                   ? __ldcs(Cs + uint64_t(row) * p.ldc + col0 + x)
                   : T(0);
  };
  auto put = [&](T* dst, const T (&o)[LEN]) {
#pragma unroll
    for (int x = 0; x < LEN; ++x) dst[x] = o[x];
  };
  auto put_cs = [&](T* dst, const T (&o)[LEN]) {
#pragma unroll
    for (int x = 0; x < LEN; ++x) __stcs(dst + x, o[x]);
  };

  uint32_t cst = 0;  // consume-side ring stage
  uint32_t nrow = warp < nch ? __ldg(p.chunk_row + warp) : 0;
  for (uint32_t c = warp; c < nch; c += nwarps) {
    const uint32_t lo = c * Q, hi = chunk_hi(c);
    uint32_t row = nrow, rb = row;
    uint32_t rew[1];
    win_load<32, 1>(rew, p.rp, rb, p.rows, lane);
    bool starts = __ldg(p.rp + row) >= lo;
    if (c + nwarps < nch) nrow = __ldg(p.chunk_row + c + nwarps);
    uint32_t rend = win_get<32, 1>(rew, 0, full);
    uint32_t rstart = lo;
    V acc = vzero<V>();
    T cin[LEN];
    cload(row, starts, cin);
    // flush the current row (it ends at rend) and move to the next one
    auto flush = [&]() {
      T o[LEN];
      reduce(acc, o);
      if (owner) {
        if (p.atomic) {
#pragma unroll
          for (int x = 0; x < LEN; ++x) atomicAdd(Cs + uint64_t(row) * p.ldc + col0 + x, o[x]);
        } else if (starts) {
          if (!CZERO)
#pragma unroll
            for (int x = 0; x < LEN; ++x) o[x] = cin[x] + o[x];
          put_cs(Cs + uint64_t(row) * p.ldc + col0, o);
        } else {
          put(p.head_val + uint64_t(c) * p.wstride + col0, o);
        }
      }
      rstart = rend;
      for (;;) {  // next row holding position rstart (skips empty rows)
        const uint32_t d = rows_done<32, 1>(rew, rstart, full);
        if (d < 32u) {
          row = rb + d;
          rend = win_get<32, 1>(rew, d, full);
          break;
        }
        rb += 32;
        win_load<32, 1>(rew, p.rp, rb, p.rows, lane);
      }
      starts = true;
      acc = vzero<V>();
      cload(row, true, cin);
    };
    for (uint32_t w = lo; w < hi; w += W) {
      issue();
      cp_async_wait<NST - 1>();
      __syncwarp();
      const uint32_t* kw = s_ci[wib][cst];
      const T* aw = s_val[wib][cst];
#pragma unroll 1
      for (int t = 0; t < W; t += STEP) {
        const uint32_t b0 = w + uint32_t(t);
        if (b0 >= hi) break;
        V bv[U];
        T av[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t q = uint32_t(t + u * S) + slot;
          const uint32_t k = kw[q];  // zero-filled past the chunk: a harmless row-0 load
          av[u] = aw[q];
          if (colok) bv[u] = ldg_v(brow_ptr<T, V, SEG>(p, segs, Bv, k, ldbv, v));
        }
        if (b0 + STEP <= hi) {
          // whole batch inside the chunk
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t base = b0 + uint32_t(u * S);
            if (rend >= base + S) {  // the step lies inside the current row
              acc = vfma(av[u], bv[u], acc);
            } else {
              const uint32_t pos = base + slot;
              do {
                if (pos >= rstart && pos < rend) acc = vfma(av[u], bv[u], acc);
                flush();
              } while (rend < base + S);
              if (pos >= rstart) acc = vfma(av[u], bv[u], acc);
            }
          }
        } else {
          // the chunk's last, partial batch
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t base = b0 + uint32_t(u * S);
            if (base >= hi) break;
            const uint32_t pos = base + slot;
            const bool valid = pos < hi;
            const uint32_t lim = min(base + S, hi);
            while (rend < lim) {
              if (valid && pos >= rstart && pos < rend) acc = vfma(av[u], bv[u], acc);
              flush();
            }
            if (valid && pos >= rstart) acc = vfma(av[u], bv[u], acc);
          }
        }
      }
      __syncwarp();
      cst = cst + 1 == NST ? 0 : cst + 1;
    }
    // the chunk's last row
    T o[LEN];
    reduce(acc, o);
    if (!CZERO && starts)
#pragma unroll
      for (int x = 0; x < LEN; ++x) o[x] = cin[x] + o[x];
    int32_t trow = -1;
    if (p.atomic) {
      if (owner)
#pragma unroll
        for (int x = 0; x < LEN; ++x) atomicAdd(Cs + uint64_t(row) * p.ldc + col0 + x, o[x]);
    } else if (rend <= hi && starts) {
      if (owner) put_cs(Cs + uint64_t(row) * p.ldc + col0, o);
    } else {
      if (owner) put((starts ? p.tail_val : p.head_val) + uint64_t(c) * p.wstride + col0, o);
      if (starts) trow = int32_t(row);
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
  cp_async_wait<0>();
}

// Load N consecutive 4- or 8-byte elements from shared memory (16-byte
// aligned when N * sizeof(E) >= 16) with the widest loads.
template <int N, typename E>
__device__ __forceinline__ void lds_vec(E (&out)[N], const E* src) {
  constexpr int BYTES = N * int(sizeof(E));
  if constexpr (BYTES >= 16 && BYTES % 16 == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
    for (int i = 0; i < BYTES / 16; ++i) reinterpret_cast<uint4*>(out)[i] = s4[i];
  } else if constexpr (BYTES == 8) {
    *reinterpret_cast<uint2*>(out) = *reinterpret_cast<const uint2*>(src);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = src[i];
  }
}

// Narrow rows with the B-row gathers themselves staged by cp.async (16-byte
// LDGSTS per lane) into a per-warp shared-memory ring GST batches deep: the
// gathers in flight no longer live in registers, so each warp keeps GST
// batches of 32 B rows in flight instead of one (the register-staged
// spmm_slots stalled on its first FMA of every batch: ncu long_scoreboard,
// profiles/).  Same slot / row / reduce-scatter logic as spmm_slots; a batch
// is 32 nonzeros = U steps of S.  Pipeline per warp, one commit group per
// batch i: {col/val window i+D, gathers of batch i+GST-1}; the gathers of a
// batch read its col indices from the window ring, D = 2*GST-1 batches
// ahead, so wait_group(GST-1) covers both.
template <typename T>
struct AsyncCfg {
  static constexpr int VEC = 16 / sizeof(T);
  static constexpr int GST = 3;            // gather stages in flight
  static constexpr int D = 2 * GST - 1;    // col/val windows ahead of consumption
  static constexpr int NA = D + 1;         // col/val ring slots
  static constexpr int WARPS = kThreads / 32;
  static size_t smem(int L) {
    return size_t(WARPS) * (size_t(NA) * 32 * (4 + sizeof(T)) + size_t(GST) * 32 * L * 16);
  }
};

template <typename T, int S, bool CZERO, bool SEG, bool ATOMIC>
__global__ void __launch_bounds__(kThreads, 2)
    spmm_slots_async(const SpmmArgs<T> p) {
  using C_ = AsyncCfg<T>;
  constexpr int VEC = C_::VEC;
  using V = typename VecOf<T, VEC>::type;
  constexpr int L = 32 / S;   // lanes (16-byte vectors) per slot
  constexpr int U = 32 / S;   // steps per batch of 32 nonzeros
  constexpr int GST = C_::GST, D = C_::D, NA = C_::NA, WARPS = C_::WARPS;
  constexpr int LOGS = S == 1 ? 0 : S == 2 ? 1 : S == 4 ? 2 : S == 8 ? 3 : S == 16 ? 4 : 5;
  constexpr int LOGV = VEC == 2 ? 1 : 2;
  constexpr int SCAT = LOGS < LOGV ? LOGS : LOGV;
  constexpr int LEN = VEC >> SCAT;
  __shared__ SegTable<T> segs;
  extern __shared__ __align__(16) unsigned char dsm[];
  load_segs<T, SEG>(p, segs);
  const uint32_t lane = threadIdx.x & 31u, slot = lane / L, v = lane % L;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = gridDim.x * WARPS;
  // per-warp rings: B rows [GST][32][L] (16-byte vectors), col [NA][32], val [NA][32]
  V* const s_b = reinterpret_cast<V*>(dsm) + size_t(wib) * GST * 32 * L;
  uint32_t* const s_ci = reinterpret_cast<uint32_t*>(dsm + size_t(WARPS) * GST * 32 * L * 16) +
                         size_t(wib) * NA * 32;
  T* const s_val = reinterpret_cast<T*>(dsm + size_t(WARPS) * GST * 32 * L * 16 +
                                        size_t(WARPS) * NA * 32 * 4) +
                   size_t(wib) * NA * 32;
  const bool colok = v < p.nvec;
  // this lane's 16 bytes of B row 0: a gather adds k * ldb bytes (one
  // IMAD.WIDE.U32; B rows are < 4 GB)
  const uint32_t vb = (colok ? v : 0) * 16u;
  const char* const Blane = reinterpret_cast<const char*>(p.B) + vb;
  const uint32_t ldbb = uint32_t(p.ldb * sizeof(T));
  T* __restrict__ Cs = p.C;
  uint32_t coff = 0;
#pragma unroll
  for (int lv = 0; lv < SCAT; ++lv)
    if (slot & (1u << lv)) coff += VEC >> (lv + 1);
  const bool owner = colok && (slot >> SCAT) == 0;
  const uint32_t col0 = v * VEC + coff;
  constexpr unsigned full = 0xffffffffu;
  // positions fit in 32 bits: row_ptr is uint32 (tile.hpp:17)
  const Chunking ck = chunking(p);
  const uint32_t nnz = ck.nnz, Q = ck.Q, nch = ck.nch;
  auto chunk_hi = [&](uint32_t lo) { return nnz - lo > Q ? lo + Q : nnz; };

  // issue sides: (chunk, window start, chunk end) of the next col/val window
  // and of the next gather batch, walking the warp's chunks in order
  uint32_t iac = warp, iaw = warp * Q, iah = warp < nch ? chunk_hi(warp * Q) : 0;
  uint32_t igc = warp, igw = iaw, igh = iah;
  uint32_t na = 0, ng = 0, ga = 0;
  // a window is stored slot-major ([S][U]: position u*S + s at s*U + u) so a
  // lane reads the U col/val entries of its slot as whole vectors
  const uint32_t adst = (lane % S) * U + lane / S;
  auto issue_a = [&]() {
    if (iac < nch) {
      const uint32_t idx = iaw + lane;
      const bool ok = idx < iah;
      cp_async(&s_ci[na * 32 + adst], p.ci + (ok ? idx : 0), ok, 4);
      cp_async(&s_val[na * 32 + adst], p.val + (ok ? idx : 0), ok, int(sizeof(T)));
      iaw += 32;
      if (iaw >= iah) {
        iac += nwarps;
        iaw = iac * Q;
        iah = iac < nch ? chunk_hi(iaw) : 0;
      }
    }
    na = na + 1 == NA ? 0 : na + 1;
  };
  auto gsrc = [&](uint32_t k) -> const void* {
    if constexpr (SEG) {
      const uint32_t sg = p.seg_shift < 32 ? (k >> p.seg_shift) : (k / p.seg_rows);
      const uint32_t r = k - sg * p.seg_rows;
      return reinterpret_cast<const char*>(segs.base[sg]) + vb + uint64_t(r) * ldbb;
    } else {
      return Blane + uint64_t(k) * ldbb;
    }
  };
  auto issue_g = [&]() {
    if (igc < nch) {
      uint32_t kk[U];
      lds_vec<U>(kk, s_ci + ga * 32 + slot * U);
      V* dst = s_b + size_t(ng) * 32 * L + lane;
      if (igw + 32 <= igh) {
#pragma unroll
        for (int u = 0; u < U; ++u) cp_async16(dst + u * 32, gsrc(kk[u]), colok);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
          cp_async16(dst + u * 32, gsrc(kk[u]), colok && igw + uint32_t(u * S) + slot < igh);
      }
      igw += 32;
      if (igw >= igh) {
        igc += nwarps;
        igw = igc * Q;
        igh = igc < nch ? chunk_hi(igw) : 0;
      }
    }
    ng = ng + 1 == GST ? 0 : ng + 1;
    ga = ga + 1 == NA ? 0 : ga + 1;
  };
  // prologue: D col/val windows (one group each), then GST-1 gather batches
#pragma unroll 1
  for (int q = 0; q < D; ++q) {
    issue_a();
    cp_async_commit();
  }
  cp_async_wait<D - GST>();
  __syncwarp();
#pragma unroll 1
  for (int q = 0; q < GST - 1; ++q) {
    issue_g();
    cp_async_commit();
  }

  auto reduce = [&](const V& acc, T (&out)[LEN]) {
    T r[VEC];
    const T* pa = reinterpret_cast<const T*>(&acc);
#pragma unroll
    for (int x = 0; x < VEC; ++x) r[x] = pa[x];
#pragma unroll
    for (int lv = 0; lv < LOGS; ++lv) {
      const int off = L << lv;
      if (lv < SCAT) {
        const int half = VEC >> (lv + 1);
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int x = 0; x < VEC / 2; ++x) {
          if (x < half) {
            const T send = upper ? r[x] : r[x + half];
            const T keep = upper ? r[x + half] : r[x];
            r[x] = keep + __shfl_xor_sync(full, send, off);
          }
        }
      } else {
        r[0] += __shfl_xor_sync(full, r[0], off);
      }
    }
#pragma unroll
    for (int x = 0; x < LEN; ++x) out[x] = r[x];
  };

  uint32_t ca = 0, cg = 0;  // consume-side ring slots
  uint32_t nrow = warp < nch ? __ldg(p.chunk_row + warp) : 0;
  for (uint32_t c = warp; c < nch; c += nwarps) {
    const uint32_t lo = c * Q, hi = chunk_hi(lo);
    uint32_t row = nrow, rb = row;
    uint32_t rew = rb + lane < p.rows ? __ldg(p.rp + rb + lane + 1) : 0xFFFFFFFFu;
    bool starts = __ldg(p.rp + row) >= lo;
    if (c + nwarps < nch) nrow = __ldg(p.chunk_row + c + nwarps);
    uint32_t rend = __shfl_sync(full, rew, 0);
    uint32_t rstart = lo;
    V acc = vzero<V>();
    T cin[LEN];
    T* crow = Cs + uint64_t(row) * p.ldc + col0;
#pragma unroll
    for (int x = 0; x < LEN; ++x)
      cin[x] = (!CZERO && !ATOMIC && starts && owner) ? __ldcs(crow + x) : T(0);
    // flush the current row (it ends at rend) and move to the next one
    auto flush = [&]() {
      T o[LEN];
      reduce(acc, o);
      if (owner) {
        if (ATOMIC) {
#pragma unroll
          for (int x = 0; x < LEN; ++x) atomicAdd(crow + x, o[x]);
        } else if (starts) {
#pragma unroll
          for (int x = 0; x < LEN; ++x) __stcs(crow + x, CZERO ? o[x] : cin[x] + o[x]);
        } else {
#pragma unroll
          for (int x = 0; x < LEN; ++x) p.head_val[uint64_t(c) * p.wstride + col0 + x] = o[x];
        }
      }
      rstart = rend;
      for (;;) {  // next row holding position rstart (skips empty rows)
        const uint32_t d = __popc(__ballot_sync(full, rew <= rstart));
        if (d < 32u) {
          row = rb + d;
          rend = __shfl_sync(full, rew, d);
          break;
        }
        rb += 32;
        rew = rb + lane < p.rows ? __ldg(p.rp + rb + lane + 1) : 0xFFFFFFFFu;
      }
      starts = true;
      acc = vzero<V>();
      crow = Cs + uint64_t(row) * p.ldc + col0;
#pragma unroll
      for (int x = 0; x < LEN; ++x) cin[x] = (!CZERO && !ATOMIC && owner) ? __ldcs(crow + x) : T(0);
    };
    for (uint32_t w = lo; w < hi; w += 32) {
      issue_a();
      issue_g();
      cp_async_commit();
      cp_async_wait<GST - 1>();
      __syncwarp();
      T aw[U];
      lds_vec<U>(aw, s_val + ca * 32 + slot * U);
      const V* bw = s_b + size_t(cg) * 32 * L + lane;
      if (rend >= w + 32 && w + 32 <= hi) {
        // the whole batch lies inside the current row
#pragma unroll
        for (int u = 0; u < U; ++u) acc = vfma(aw[u], bw[u * 32], acc);
      } else if (w + 32 <= hi) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t base = w + uint32_t(u * S);
          const T a = aw[u];
          const V b = bw[u * 32];
          if (rend >= base + S) {
            acc = vfma(a, b, acc);
          } else {
            const uint32_t pos = base + slot;
            do {
              if (pos >= rstart && pos < rend) acc = vfma(a, b, acc);
              flush();
            } while (rend < base + S);
            if (pos >= rstart) acc = vfma(a, b, acc);
          }
        }
      } else {
        // the chunk's last, partial batch
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t base = w + uint32_t(u * S);
          if (base >= hi) break;
          const T a = aw[u];
          const V b = bw[u * 32];
          const uint32_t pos = base + slot;
          const bool valid = pos < hi;
          const uint32_t lim = min(base + S, hi);
          while (rend < lim) {
            if (valid && pos >= rstart && pos < rend) acc = vfma(a, b, acc);
            flush();
          }
          if (valid && pos >= rstart) acc = vfma(a, b, acc);
        }
      }
      __syncwarp();
      ca = ca + 1 == NA ? 0 : ca + 1;
      cg = cg + 1 == GST ? 0 : cg + 1;
    }
    T o[LEN];
    reduce(acc, o);
    if (!CZERO && starts)
#pragma unroll
      for (int x = 0; x < LEN; ++x) o[x] = cin[x] + o[x];
    int32_t trow = -1;
    if (ATOMIC) {
      if (owner)
#pragma unroll
        for (int x = 0; x < LEN; ++x) atomicAdd(crow + x, o[x]);
    } else if (rend <= hi && starts) {
      if (owner)
#pragma unroll
        for (int x = 0; x < LEN; ++x) __stcs(crow + x, o[x]);
    } else {
      if (owner)
#pragma unroll
        for (int x = 0; x < LEN; ++x)
          (starts ? p.tail_val : p.head_val)[uint64_t(c) * p.wstride + col0 + x] = o[x];
      if (starts) trow = int32_t(row);
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
  cp_async_wait<0>();
}

// Row-oriented variant: the worker walks the chunk row by row; each row
// (or the chunk's slice of it) is accumulated from its own col/val window.
template <typename T, int VEC, int G, int NV, bool CZERO, int MINB, bool SEG>
__global__ void __launch_bounds__(kThreads, MINB)
    spmm_rows(const SpmmArgs<T> p) {
  using V = typename VecOf<T, VEC>::type;
  __shared__ SegTable<T> segs;
  load_segs<T, SEG>(p, segs);
  constexpr int SL = kWin / G;
  const unsigned gm = group_mask<G>();
  const uint32_t lane = threadIdx.x % G;
  const uint32_t worker = (blockIdx.x * kThreads + threadIdx.x) / G;
  const uint32_t nworkers = gridDim.x * (kThreads / G);
  const V* __restrict__ Bv = reinterpret_cast<const V*>(p.B);
  V* __restrict__ Cv = reinterpret_cast<V*>(p.C);
  const uint64_t ldbv = p.ldb / VEC, ldcv = p.ldc / VEC;
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) colok[v] = lane + G * v < p.nvec;
  for (uint32_t c = worker; c < p.nchunks; c += nworkers) {
    const uint64_t lo = uint64_t(c) * p.Q;
    const uint64_t hi = umin(lo + p.Q, p.nnz);
    const uint32_t l = __ldg(p.chunk_row + c);
    uint32_t r = l;
    uint32_t rs = __ldg(p.rp + r);
    uint32_t re = __ldg(p.rp + r + 1);
    int32_t trow = -1;
    while (rs < hi) {
      const uint32_t re_next = (r + 2 <= p.rows) ? __ldg(p.rp + r + 2) : re;
      const uint64_t s = umax(rs, lo), e = umin(re, hi);
      if (s < e) {
        const bool starts = rs >= lo, ends = re <= hi;
        V acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v)
          acc[v] = (!CZERO && starts && colok[v])
                       ? Cv[uint64_t(r) * ldcv + lane + G * v]
                       : vzero<V>();
        for (uint64_t base = s; base < e; base += kWin) {
          const uint32_t cnt = uint32_t(umin(kWin, e - base));
          uint32_t kk[SL];
          T aa[SL];
#pragma unroll
          for (int j = 0; j < SL; ++j) {
            const uint64_t idx = base + lane + G * j;
            const bool ok = idx < e;
            kk[j] = ok ? __ldg(p.ci + idx) : 0u;
            aa[j] = ok ? __ldg(p.val + idx) : T(0);
          }
#pragma unroll
          for (int t = 0; t < kWin; t += kU) {
            if (t < int(cnt)) {
              V bv[kU][NV];
#pragma unroll
              for (int u = 0; u < kU; ++u) {
                const int q = t + u;
                const uint32_t k = __shfl_sync(gm, kk[q / G], q % G, G);
                if (q < int(cnt)) {
                  const V* brow = brow_ptr<T, V, SEG>(p, segs, Bv, k, ldbv, lane);
#pragma unroll
                  for (int v = 0; v < NV; ++v)
                    if (colok[v]) bv[u][v] = __ldg(brow + G * v);
                }
              }
#pragma unroll
              for (int u = 0; u < kU; ++u) {
                const int q = t + u;
                const T a = __shfl_sync(gm, aa[q / G], q % G, G);
                if (q < int(cnt)) {
#pragma unroll
                  for (int v = 0; v < NV; ++v)
                    if (colok[v]) acc[v] = vfma(a, bv[u][v], acc[v]);
                }
              }
            }
          }
        }
        if (starts && ends) {
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (colok[v]) Cv[uint64_t(r) * ldcv + lane + G * v] = acc[v];
        } else {
          V* dst = reinterpret_cast<V*>(starts ? p.tail_val : p.head_val) +
                   uint64_t(c) * (p.wstride / VEC);
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (colok[v]) dst[lane + G * v] = acc[v];
          if (starts) trow = int32_t(r);
        }
      }
      ++r;
      rs = re;
      re = re_next;
      if (r >= p.rows) break;
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
}

// Narrow rows (N < 128 fp32: L = N/4 < 32 vectors per B row): the whole warp
// works on ONE row at a time; lane (s, v) takes every S-th nonzero of the
// row (S = 32/L slots) and vector v of its B row, so S gathers of L*16 bytes
// are in flight per load instruction and the warp never splits into
// divergent per-row groups; the S partial sums of a row are combined with
// shuffles before the store.  (Summation order differs from the reference
// for real values: slot partials, then their sum; exact for integer data.)
template <typename T, int VEC, int L, bool CZERO, bool SEG>
__global__ void __launch_bounds__(kThreads)
    spmm_vec(const SpmmArgs<T> p) {
  using V = typename VecOf<T, VEC>::type;
  __shared__ SegTable<T> segs;
  load_segs<T, SEG>(p, segs);
  constexpr int S = 32 / L;
  constexpr int U = 4;
  const uint32_t lane = threadIdx.x & 31u, sl = lane / L, v = lane % L;
  const uint32_t warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint32_t nwarps = gridDim.x * (kThreads / 32);
  const V* __restrict__ Bv = reinterpret_cast<const V*>(p.B);
  V* __restrict__ Cv = reinterpret_cast<V*>(p.C);
  const uint64_t ldbv = p.ldb / VEC, ldcv = p.ldc / VEC;
  const bool colok = v < p.nvec;
  for (uint32_t c = warp; c < p.nchunks; c += nwarps) {
    const uint64_t lo = uint64_t(c) * p.Q;
    const uint64_t hi = umin(lo + p.Q, p.nnz);
    const uint32_t l = __ldg(p.chunk_row + c);
    uint32_t r = l;
    uint32_t rs = __ldg(p.rp + r), re = __ldg(p.rp + r + 1);
    int32_t trow = -1;
    while (rs < hi) {
      const uint32_t re_next = (r + 2 <= p.rows) ? __ldg(p.rp + r + 2) : re;
      const uint64_t s0 = umax(rs, lo), e0 = umin(re, hi);
      if (s0 < e0) {
        const bool starts = rs >= lo, ends = re <= hi;
        V acc = vzero<V>();
        for (uint64_t base = s0; base < e0; base += 32) {
          const uint32_t cnt = uint32_t(umin(32, e0 - base));
          const bool ok0 = lane < cnt;
          const uint32_t kk = ok0 ? __ldg(p.ci + base + lane) : 0u;
          const T aa = ok0 ? __ldg(p.val + base + lane) : T(0);
#pragma unroll
          for (int t = 0; t < 32; t += S * U) {
            if (t < int(cnt)) {
              V bv[U];
              T av[U];
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int q = t + u * S + int(sl);
                const uint32_t k = __shfl_sync(0xffffffffu, kk, q & 31);
                av[u] = __shfl_sync(0xffffffffu, aa, q & 31);
                if (q < int(cnt) && colok) bv[u] = __ldg(brow_ptr<T, V, SEG>(p, segs, Bv, k, ldbv, v));
              }
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int q = t + u * S + int(sl);
                if (q < int(cnt) && colok) acc = vfma(av[u], bv[u], acc);
              }
            }
          }
        }
        // combine the S slot partials (lanes v, v+L, v+2L, ...)
        T* pa = reinterpret_cast<T*>(&acc);
#pragma unroll
        for (int off = L; off < 32; off <<= 1)
#pragma unroll
          for (int x = 0; x < VEC; ++x) pa[x] += __shfl_xor_sync(0xffffffffu, pa[x], off);
        if (sl == 0 && colok) {
          if (starts && ends) {
            if (!CZERO) acc = vadd(Cv[uint64_t(r) * ldcv + v], acc);
            __stcs(Cv + uint64_t(r) * ldcv + v, acc);
          } else {
            if (!CZERO && starts) acc = vadd(Cv[uint64_t(r) * ldcv + v], acc);
            V* dst = reinterpret_cast<V*>(starts ? p.tail_val : p.head_val) +
                     uint64_t(c) * (p.wstride / VEC);
            dst[v] = acc;
          }
        }
        if (starts && !ends) trow = int32_t(r);
      }
      ++r;
      rs = re;
      re = re_next;
      if (r >= p.rows) break;
    }
    if (lane == 0) p.tail_row[c] = trow;
  }
}

// Rows cut by chunk boundaries: C[r] = tail(c) + head(c+1) + head(c+2) + ...
template <typename T, int VEC, int G, int NV>
__global__ void __launch_bounds__(kThreads) spmm_fixup(const SpmmArgs<T> p) {
  using V = typename VecOf<T, VEC>::type;
  const uint32_t lane = threadIdx.x % G;
  const uint32_t worker = (blockIdx.x * kThreads + threadIdx.x) / G;
  const uint32_t nworkers = gridDim.x * (kThreads / G);
  const uint32_t ws = p.wstride / VEC;
  V* __restrict__ Cv = reinterpret_cast<V*>(p.C);
  const V* hv = reinterpret_cast<const V*>(p.head_val);
  const V* tv = reinterpret_cast<const V*>(p.tail_val);
  const Chunking ck = chunking(p);
  for (uint32_t c = worker; c < ck.nch; c += nworkers) {
    const int32_t r = p.tail_row[c];
    if (r < 0) continue;
    const uint64_t re = p.rp[r + 1];
    V acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + G * v < p.nvec) acc[v] = tv[uint64_t(c) * ws + lane + G * v];
    for (uint32_t c2 = c + 1; c2 < ck.nch; ++c2) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + G * v < p.nvec)
          acc[v] = vadd(acc[v], hv[uint64_t(c2) * ws + lane + G * v]);
      if (re <= umin(uint64_t(c2 + 1) * ck.Q, ck.nnz)) break;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + G * v < p.nvec)
        Cv[uint64_t(r) * (p.ldc / VEC) + lane + G * v] = acc[v];
  }
}

// RDMM_SPMM_KERNEL=rows|stream|vec forces a kernel family (a measurement
// switch; default auto).
inline int kernel_variant() {
  static const int v = [] {
    const char* e = std::getenv("RDMM_SPMM_KERNEL");
    if (!e) return 0;  // auto
    const std::string s(e);
    return s == "rows" ? 1 : s == "stream" ? 2 : s == "vec" ? 3 : 0;
  }();
  return v;
}

// RDMM_SPMM_ASYNC=0 disables the cp.async-gather narrow kernel (rows of at
// most 128 bytes).  A measurement switch.
inline bool async_mode() {
  static const bool v = [] {
    const char* e = std::getenv("RDMM_SPMM_ASYNC");
    return !(e && std::string(e) == "0");
  }();
  return v;
}

// RDMM_SPMM_FULL=0 disables spmm_stream_full (a measurement switch).
inline bool full_mode() {
  static const bool v = [] {
    const char* e = std::getenv("RDMM_SPMM_FULL");
    return !(e && std::string(e) == "0");
  }();
  return v;
}

// Kernel choice, measured on B200 (profiles/):
//  * narrow rows (nvec < 32 vectors: N < 128 fp32) -> spmm_slots, the warp
//    streaming one nnz chunk with S = 32/L slots (N = 32 on cfg3's A:
//    spmm_vec 2.82 ms, per-group spmm_stream 2.08 ms);
//  * one 16-B vector per lane (N = 128 fp32) -> spmm_stream at 64 registers,
//    4 CTAs/SM;
//  * wider rows (NV >= 2 vectors per lane) -> spmm_rows, at the HBM gather
//    roofline on ER (cfg5).
template <typename T, int VEC, int G, int NV, bool SEG>
void launch_seg(const SpmmArgs<T>& a, bool czero, int blocks, cudaStream_t s) {
  const int kv = kernel_variant();
  if constexpr (G < 32) {
    constexpr int S = 32 / G;
    constexpr bool v16 = sizeof(typename VecOf<T, VEC>::type) <= 16;
    if constexpr (!v16) {  // 32-byte vectors: spmm_slots only
      if (czero) spmm_slots<T, VEC, S, true, 3, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_slots<T, VEC, S, false, 3, SEG><<<blocks, kThreads, 0, s>>>(a);
    } else if (kv == 0 && G <= 8 && VEC * sizeof(T) == 16 && async_mode()) {
      const size_t sm = AsyncCfg<T>::smem(G);
      // atomic accumulation never reads C: one instantiation serves it
      const int variant = a.atomic ? 2 : czero ? 1 : 0;
      auto fn = variant == 2   ? spmm_slots_async<T, S, false, SEG, true>
                : variant == 1 ? spmm_slots_async<T, S, true, SEG, false>
                               : spmm_slots_async<T, S, false, SEG, false>;
      // the dynamic shared-memory opt-in is per device
      static std::atomic<int> resident[3][kMaxDevices] = {};  // CTAs per SM (persistent grid)
      int dev = 0;
      cudaGetDevice(&dev);
      std::atomic<int>& res = resident[variant][dev < kMaxDevices ? dev : 0];
      if (!res.load()) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, sm);
        res.store(nb > 0 ? nb : 1);
      }
      fn<<<std::min(blocks, res.load() * num_sms()), kThreads, sm, s>>>(a);
    } else if (kv == 1) {
      if (czero) spmm_rows<T, VEC, G, NV, true, 1, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_rows<T, VEC, G, NV, false, 1, SEG><<<blocks, kThreads, 0, s>>>(a);
    } else if (kv == 3) {
      if (czero) spmm_vec<T, VEC, G, true, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_vec<T, VEC, G, false, SEG><<<blocks, kThreads, 0, s>>>(a);
    } else {
      if (czero) spmm_slots<T, VEC, S, true, 3, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_slots<T, VEC, S, false, 3, SEG><<<blocks, kThreads, 0, s>>>(a);
    }
  } else {
    constexpr int MB = NV == 1 ? 4 : 1;
    const bool use_rows = kv == 1 || (kv != 2 && NV != 1);
    if (use_rows) {
      if (czero) spmm_rows<T, VEC, G, NV, true, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_rows<T, VEC, G, NV, false, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
    } else if (a.full_ok && !SEG && NV == 1 && G == 32 && VEC * sizeof(T) == 16) {
      if (czero) spmm_stream_full<T, true><<<blocks, kThreads, 0, s>>>(a);
      else spmm_stream_full<T, false><<<blocks, kThreads, 0, s>>>(a);
    } else {
      if (czero) spmm_stream<T, VEC, G, NV, true, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_stream<T, VEC, G, NV, false, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
    }
  }
}

template <typename T, int VEC, int G, int NV>
void launch(const SpmmArgs<T>& a, bool czero, int blocks, int fix_blocks,
            cudaStream_t s) {
  if (a.nseg)
    launch_seg<T, VEC, G, NV, true>(a, czero, blocks, s);
  else
    launch_seg<T, VEC, G, NV, false>(a, czero, blocks, s);
  if (!a.atomic) spmm_fixup<T, VEC, G, NV><<<fix_blocks, kThreads, 0, s>>>(a);
}

template <typename T, int VEC>
void dispatch(const SpmmArgs<T>& a, bool cz, int G, int NV, int blocks,
              int fix_blocks, cudaStream_t s) {
  switch (G) {
    case 1: launch<T, VEC, 1, 1>(a, cz, blocks, fix_blocks, s); break;
    case 2: launch<T, VEC, 2, 1>(a, cz, blocks, fix_blocks, s); break;
    case 4: launch<T, VEC, 4, 1>(a, cz, blocks, fix_blocks, s); break;
    case 8: launch<T, VEC, 8, 1>(a, cz, blocks, fix_blocks, s); break;
    case 16: launch<T, VEC, 16, 1>(a, cz, blocks, fix_blocks, s); break;
    default:
      if (NV == 1)
        launch<T, VEC, 32, 1>(a, cz, blocks, fix_blocks, s);
      else if (NV == 2)
        launch<T, VEC, 32, 2>(a, cz, blocks, fix_blocks, s);
      else
        launch<T, VEC, 32, 4>(a, cz, blocks, fix_blocks, s);
  }
}

// 32-byte vectors: narrow rows only (G < 32, spmm_slots)
template <typename T, int VEC>
void dispatch_narrow(const SpmmArgs<T>& a, bool cz, int G, int blocks, int fix_blocks,
                     cudaStream_t s) {
  switch (G) {
    case 1: launch<T, VEC, 1, 1>(a, cz, blocks, fix_blocks, s); break;
    case 2: launch<T, VEC, 2, 1>(a, cz, blocks, fix_blocks, s); break;
    case 4: launch<T, VEC, 4, 1>(a, cz, blocks, fix_blocks, s); break;
    case 8: launch<T, VEC, 8, 1>(a, cz, blocks, fix_blocks, s); break;
    default: launch<T, VEC, 16, 1>(a, cz, blocks, fix_blocks, s); break;
  }
}

constexpr int kMaxNV = 4;

// Panel width in vectors handled by one launch pair.
inline uint32_t panel_vecs() { return 32u * kMaxNV; }

inline uint32_t chunk_count(uint64_t nnz, uint32_t workers, bool narrow) {
  // chunks per resident worker for tail smoothing, >= 64 nnz each: 8 for
  // full-width rows and rows under 8 vectors, 16 for the narrow slot kernels
  // of 8-31 vectors (cfg3's A at N = 32: 1.120 -> 1.054 ms, N = 64 1.87 ->
  // 1.80; N = 16 measured 0.809 at 8 vs 0.836 at 16).  RDMM_SPMM_CPW
  // overrides (a measurement switch).
  static const int env = [] {
    const char* e = std::getenv("RDMM_SPMM_CPW");
    return e ? std::atoi(e) : 0;
  }();
  const uint64_t cpw = env > 0 ? uint64_t(env) : narrow ? 16u : 8u;
  uint64_t by_size = ceil_div(nnz, 64);
  uint64_t by_workers = uint64_t(workers) * cpw;
  uint64_t n = std::max<uint64_t>(1, std::min(by_size, by_workers));
  return uint32_t(std::min<uint64_t>(n, 1u << 30));
}

inline int groups_for(uint32_t nvec, int* NV) {
  if (nvec >= 32) {
    *NV = int(std::min<uint32_t>(kMaxNV, uint32_t(ceil_div(nvec, 32))));
    if (*NV == 3) *NV = 4;
    return 32;
  }
  *NV = 1;
  int g = 1;
  while (uint32_t(g) < nvec) g <<= 1;
  return g;
}

struct SpmmPlan {
  int VEC = 1, blocks = 0, fix_blocks = 0, chunk_blocks = 0;
  uint32_t pv = 0, nchunks = 0, wstride = 0;
  uint64_t Q = 0;
  size_t bytes = 0;
};

// RDMM_SPMM_V32=0 disables the 32-byte-vector narrow path; =all extends it to
// rows of 512 bytes (N = 128 fp32).  A measurement switch.
inline int v32_mode() {
  static const int v = [] {
    const char* e = std::getenv("RDMM_SPMM_V32");
    if (!e) return 1;
    const std::string s(e);
    return s == "0" ? 0 : s == "all" ? 2 : 1;
  }();
  return v;
}

// vmode: 0 scalar, 1 16-byte vectors, 2 32-byte vectors (narrow rows only)
template <typename T>
SpmmPlan make_plan(uint32_t rows, uint64_t nnz, uint32_t n, int vmode) {
  constexpr int VV = sizeof(T) == 4 ? 4 : 2;
  SpmmPlan P;
  P.VEC = vmode == 2 ? 2 * VV : vmode == 1 ? VV : 1;
  const uint32_t nvec_total = n / P.VEC;
  const int sms = num_sms();
  P.pv = std::min<uint32_t>(nvec_total, panel_vecs());
  int NV = 1;
  const int G = groups_for(P.pv, &NV);
  // a worker is a warp (spmm_slots / spmm_stream / spmm_rows at G = 32), or
  // a G-lane group for the forced narrow row kernels
  const int wl = (G < 32 && kernel_variant() == 0) ? 32 : G;
  const int blocks_max = sms * 8;  // 8 x 256 threads per SM (register bound)
  const uint32_t per_block = kThreads / wl;
  const uint32_t workers = uint32_t(blocks_max) * per_block;
  const uint32_t nchunks = chunk_count(std::max<uint64_t>(nnz, 1), workers, G >= 8 && G < 32);
  P.Q = ceil_div(std::max<uint64_t>(nnz, 1), nchunks);
  P.nchunks = uint32_t(ceil_div(std::max<uint64_t>(nnz, 1), P.Q));
  P.wstride = uint32_t(ceil_div(uint64_t(P.pv) * P.VEC, 4) * 4);
  P.bytes = 2 * size_t(P.nchunks) * P.wstride * sizeof(T) + 2 * size_t(P.nchunks) * 4 + 256;
  P.blocks = int(std::min<uint64_t>(blocks_max, ceil_div(P.nchunks, per_block)));
  P.fix_blocks = int(std::min<uint64_t>(sms * 4, ceil_div(P.nchunks, kThreads / G)));
  P.chunk_blocks = int(std::max<uint64_t>(
      1, std::min<uint64_t>(uint64_t(sms) * 8, ceil_div(uint64_t(rows), kThreads))));
  return P;
}

template <typename T>
size_t workspace_bytes_impl(uint32_t rows, uint64_t nnz, uint32_t n) {
  size_t b = 0;
  for (int vm = 0; vm < 3; ++vm) b = std::max(b, make_plan<T>(rows, nnz, n, vm).bytes);
  return b;
}

template <typename T>
int spmm_impl(uint32_t rows, uint32_t cols, uint32_t n, uint64_t nnz,
              const uint32_t* rp, const uint32_t* ci, const T* val, const T* B,
              uint64_t ldb, T* C, uint64_t ldc, unsigned flags, void* ws,
              size_t ws_bytes, rdmm_stream_t stream, uint64_t* flops,
              const T* const* bseg = nullptr, uint32_t nseg = 0, uint32_t seg_rows = 0) {
  bool dyn = (flags & RDMM_SPMM_NNZ_ON_DEVICE) != 0;
  if (flops) *flops = dyn ? 0 : 2ull * nnz * n;
  const bool czero = (flags & RDMM_SPMM_C_ZERO) != 0;
  if (ldb < n || ldc < n)
    return fail(RDMM_ERR_DIMENSION, "spmm: leading dimension smaller than n");
  if (rows == 0 || n == 0 || nnz == 0) return RDMM_OK;
  if (!rp || !ci || !val || (!B && !nseg) || !C)
    return fail(RDMM_ERR_INVALID, "spmm: null device pointer");
  cudaStream_t s = as_stream(stream);
  constexpr int VV = sizeof(T) == 4 ? 4 : 2;
  if (nseg > 16) return fail(RDMM_ERR_INVALID, "spmm: at most 16 B segments");
  auto aligned = [&](uintptr_t a) {
    bool ok = (reinterpret_cast<uintptr_t>(C) % a) == 0;
    if (nseg)
      for (uint32_t q = 0; q < nseg; ++q) ok &= (reinterpret_cast<uintptr_t>(bseg[q]) % a) == 0;
    else
      ok &= (reinterpret_cast<uintptr_t>(B) % a) == 0;
    return ok;
  };
  const bool vec_ok = n % VV == 0 && ldb % VV == 0 && ldc % VV == 0 && aligned(16);
  // 32-byte vectors for narrow rows (<= 256 bytes; <= 512 with RDMM_SPMM_V32=all)
  const uint64_t max_row = v32_mode() == 2 ? 512 : 256;
  const bool async_rows = async_mode() && kernel_variant() == 0 && uint64_t(n) * sizeof(T) <= 128;
  const bool v32_ok = !async_rows && v32_mode() != 0 && kernel_variant() == 0 && n % (2 * VV) == 0 &&
                      ldb % (2 * VV) == 0 && ldc % (2 * VV) == 0 && aligned(32) &&
                      uint64_t(n) * sizeof(T) <= max_row;
  const int vmode = v32_ok ? 2 : vec_ok ? 1 : 0;
  const uint32_t vec_chosen = vmode == 2 ? 2 * VV : vmode == 1 ? VV : 1;
  // the narrow slot kernels chunk on the device; the others need nnz here
  const bool narrow_slots = kernel_variant() == 0 && n / vec_chosen < 32;
  if (dyn && !narrow_slots) {
    // only the narrow cp.async kernel chunks on the device: read nnz here
    uint32_t nd = 0;
    RDMM_CUDA_TRY(cudaMemcpyAsync(&nd, rp + rows, 4, cudaMemcpyDeviceToHost, s));
    RDMM_CUDA_TRY(cudaStreamSynchronize(s));
    nnz = nd;
    dyn = false;
    if (nnz == 0) return RDMM_OK;
  }
  const SpmmPlan P = make_plan<T>(rows, nnz, n, vmode);
  void* w = ws;
  if (!w || ws_bytes < P.bytes) {
    if (ws) return fail(RDMM_ERR_INVALID, "spmm: workspace too small");
    w = scratch(P.bytes, 0, s);
    if (!w) return fail(RDMM_ERR_CUDA, "spmm: scratch allocation failed");
  }
  SpmmArgs<T> a{};
  a.rp = rp;
  a.ci = ci;
  a.val = val;
  a.ldb = ldb;
  a.ldc = ldc;
  a.nnz = nnz;
  a.Q = P.Q;
  a.rows = rows;
  a.nchunks = P.nchunks;
  a.wstride = P.wstride;
  a.nseg = nseg;
  a.seg_rows = seg_rows;
  a.seg_shift = 32;
  if (nseg) {
    if (seg_rows == 0) return fail(RDMM_ERR_INVALID, "spmm: seg_rows must be positive");
    for (uint32_t q = 0; q < nseg; ++q) a.bseg[q] = bseg[q];
    if ((seg_rows & (seg_rows - 1)) == 0) a.seg_shift = uint32_t(__builtin_ctz(seg_rows));
  }
  char* base = static_cast<char*>(w);
  const size_t vbytes = size_t(P.nchunks) * P.wstride * sizeof(T);
  a.head_val = reinterpret_cast<T*>(base);
  a.tail_val = reinterpret_cast<T*>(base + vbytes);
  a.tail_row = reinterpret_cast<int32_t*>(base + 2 * vbytes);
  uint32_t* chunk_row = reinterpret_cast<uint32_t*>(base + 2 * vbytes + size_t(P.nchunks) * 4);
  a.chunk_row = chunk_row;
  a.dyn_end = dyn ? rp + rows : nullptr;
  // atomic accumulation: the narrow slot kernels only (others ignore it)
  a.atomic = (flags & RDMM_SPMM_ATOMIC) != 0 && narrow_slots;
  const uint32_t nvec_total = n / P.VEC;
  a.full_ok = full_mode() && !nseg && P.VEC == VV && nvec_total == 32 &&
              (kernel_variant() == 0 || kernel_variant() == 2) &&
              uint64_t(cols) * (ldb / VV) < (1ull << 32) &&
              uint64_t(rows) * (ldc / VV) < (1ull << 32) && nnz + P.Q < (1ull << 32);
  KernelTimer timer(s, 1);
  count_launch(1);
  spmm_chunk_rows<<<P.chunk_blocks, kThreads, 0, s>>>(rp, rows, P.Q, P.nchunks, chunk_row,
                                                      a.dyn_end);
  for (uint32_t v0 = 0; v0 < nvec_total; v0 += P.pv) {
    count_launch(2);
    const uint32_t nv = std::min<uint32_t>(P.pv, nvec_total - v0);
    int nvp = 1;
    const int g = groups_for(nv, &nvp);
    a.B = nseg ? nullptr : B + uint64_t(v0) * P.VEC;
    a.boff = uint64_t(v0) * P.VEC;
    a.C = C + uint64_t(v0) * P.VEC;
    a.nvec = nv;
    if (P.VEC == 1)
      dispatch<T, 1>(a, czero, g, nvp, P.blocks, P.fix_blocks, s);
    else if (P.VEC == VV)
      dispatch<T, VV>(a, czero, g, nvp, P.blocks, P.fix_blocks, s);
    else
      dispatch_narrow<T, 2 * VV>(a, czero, g, P.blocks, P.fix_blocks, s);
  }
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

extern "C" size_t rdmm_spmm_workspace_bytes(uint32_t rows, uint64_t nnz,
                                            uint32_t n, int dtype_bytes) {
  return dtype_bytes == 8 ? workspace_bytes_impl<double>(rows, nnz, n)
                          : workspace_bytes_impl<float>(rows, nnz, n);
}

extern "C" int rdmm_spmm_csr_f32(uint32_t rows, uint32_t cols, uint32_t n,
                                 uint64_t nnz, const uint32_t* row_ptr,
                                 const uint32_t* col_idx, const float* val,
                                 const float* B, uint64_t ldb, float* C,
                                 uint64_t ldc, void* workspace,
                                 size_t workspace_bytes, rdmm_stream_t stream,
                                 uint64_t* flops) {
  return spmm_impl<float>(rows, cols, n, nnz, row_ptr, col_idx, val, B, ldb, C,
                          ldc, 0u, workspace, workspace_bytes, stream, flops);
}

extern "C" int rdmm_spmm_csr_f64(uint32_t rows, uint32_t cols, uint32_t n,
                                 uint64_t nnz, const uint32_t* row_ptr,
                                 const uint32_t* col_idx, const double* val,
                                 const double* B, uint64_t ldb, double* C,
                                 uint64_t ldc, void* workspace,
                                 size_t workspace_bytes, rdmm_stream_t stream,
                                 uint64_t* flops) {
  return spmm_impl<double>(rows, cols, n, nnz, row_ptr, col_idx, val, B, ldb,
                           C, ldc, 0u, workspace, workspace_bytes, stream, flops);
}

extern "C" int rdmm_spmm_csr_ex(int dtype_bytes, uint32_t rows, uint32_t cols,
                                uint32_t n, uint64_t nnz,
                                const uint32_t* row_ptr,
                                const uint32_t* col_idx, const void* val,
                                const void* B, uint64_t ldb, void* C,
                                uint64_t ldc, unsigned flags, void* workspace,
                                size_t workspace_bytes, rdmm_stream_t stream,
                                uint64_t* flops) {
  if (dtype_bytes == 8)
    return spmm_impl<double>(rows, cols, n, nnz, row_ptr, col_idx,
                             static_cast<const double*>(val),
                             static_cast<const double*>(B), ldb,
                             static_cast<double*>(C), ldc, flags, workspace,
                             workspace_bytes, stream, flops);
  return spmm_impl<float>(rows, cols, n, nnz, row_ptr, col_idx,
                          static_cast<const float*>(val),
                          static_cast<const float*>(B), ldb,
                          static_cast<float*>(C), ldc, flags, workspace,
                          workspace_bytes, stream, flops);
}

extern "C" int rdmm_spmm_csr_seg(int dtype_bytes, uint32_t rows, uint32_t n,
                                 uint64_t nnz, const uint32_t* row_ptr,
                                 const uint32_t* col_idx, const void* val,
                                 const void* const* bseg, uint32_t nseg,
                                 uint32_t seg_rows, uint64_t ldb, void* C,
                                 uint64_t ldc, unsigned flags, void* workspace,
                                 size_t workspace_bytes, rdmm_stream_t stream,
                                 uint64_t* flops) {
  if (dtype_bytes == 8)
    return spmm_impl<double>(rows, nseg * seg_rows, n, nnz, row_ptr, col_idx,
                             static_cast<const double*>(val), nullptr, ldb,
                             static_cast<double*>(C), ldc, flags, workspace,
                             workspace_bytes, stream, flops,
                             reinterpret_cast<const double* const*>(bseg), nseg,
                             seg_rows);
  return spmm_impl<float>(rows, nseg * seg_rows, n, nnz, row_ptr, col_idx,
                          static_cast<const float*>(val), nullptr, ldb,
                          static_cast<float*>(C), ldc, flags, workspace,
                          workspace_bytes, stream, flops,
                          reinterpret_cast<const float* const*>(bseg), nseg, seg_rows);
}
