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
__device__ __forceinline__ float vadd(float a, float b) { return a + b; }
__device__ __forceinline__ double vadd(double a, double b) { return a + b; }
__device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) {
  return a < b ? a : b;
}
__device__ __forceinline__ uint64_t umax(uint64_t a, uint64_t b) {
  return a > b ? a : b;
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
  uint64_t ldb, ldc;
  uint64_t nnz, Q;
  uint32_t rows, nvec, nchunks, wstride;
  int prefetch;  // unused (the L2 prefetch of the next window measured slower)
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
    // row containing nonzero `lo`: largest r with rp[r] <= lo
    uint32_t l = 0, h = p.rows;
    while (h - l > 1) {
      const uint32_t m = (l + h) >> 1;
      if (__ldg(p.rp + m) <= lo)
        l = m;
      else
        h = m;
    }
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
    uint32_t l = 0, h = p.rows;
    while (h - l > 1) {
      const uint32_t m = (l + h) >> 1;
      if (__ldg(p.rp + m) <= lo)
        l = m;
      else
        h = m;
    }
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
    uint32_t l = 0, h = p.rows;
    while (h - l > 1) {
      const uint32_t m = (l + h) >> 1;
      if (__ldg(p.rp + m) <= lo)
        l = m;
      else
        h = m;
    }
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
  for (uint32_t c = worker; c < p.nchunks; c += nworkers) {
    const int32_t r = p.tail_row[c];
    if (r < 0) continue;
    const uint64_t re = p.rp[r + 1];
    V acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + G * v < p.nvec) acc[v] = tv[uint64_t(c) * ws + lane + G * v];
    for (uint32_t c2 = c + 1; c2 < p.nchunks; ++c2) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (lane + G * v < p.nvec)
          acc[v] = vadd(acc[v], hv[uint64_t(c2) * ws + lane + G * v]);
      if (re <= umin(uint64_t(c2 + 1) * p.Q, p.nnz)) break;
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (lane + G * v < p.nvec)
        Cv[uint64_t(r) * (p.ldc / VEC) + lane + G * v] = acc[v];
  }
}

// RDMM_SPMM_KERNEL=rows|stream forces a kernel (dev switch; default auto;
// narrow rows accept only "rows").
inline int kernel_variant() {
  static const int v = [] {
    const char* e = std::getenv("RDMM_SPMM_KERNEL");
    if (!e) return 0;  // auto
    return std::string(e) == "rows" ? 1 : 2;
  }();
  return v;
}

template <typename T, int VEC, int G, int NV, bool SEG>
void launch_seg(const SpmmArgs<T>& a, bool czero, int blocks, cudaStream_t s) {
  // Measured on B200 (profiles/): the nnz-stream kernel at
  // 64 registers (4 CTAs/SM) wins for one 16-B vector per lane (N=128 fp32);
  // wider rows (NV>=2) keep more gathers in flight per lane and the
  // row-oriented kernel is faster there (at the HBM gather roofline on ER);
  // narrow rows (N<128) use the whole-warp row kernel.
  // Only the (kernel, occupancy) pairs that a setting can select are
  // instantiated: narrow rows -> spmm_vec (or spmm_rows when forced);
  // G=32,NV=1 -> 4 CTAs/SM; wider -> 1 CTA/SM minimum.
  const int kv = kernel_variant();
  if constexpr (G < 32) {
    if (kv == 1) {
      if (czero) spmm_rows<T, VEC, G, NV, true, 1, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_rows<T, VEC, G, NV, false, 1, SEG><<<blocks, kThreads, 0, s>>>(a);
    } else {
      if (czero) spmm_vec<T, VEC, G, true, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_vec<T, VEC, G, false, SEG><<<blocks, kThreads, 0, s>>>(a);
    }
  } else {
    constexpr int MB = NV == 1 ? 4 : 1;
    const bool use_rows = kv == 1 || (kv == 0 && NV != 1);
    if (use_rows) {
      if (czero) spmm_rows<T, VEC, G, NV, true, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
      else spmm_rows<T, VEC, G, NV, false, MB, SEG><<<blocks, kThreads, 0, s>>>(a);
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
  spmm_fixup<T, VEC, G, NV><<<fix_blocks, kThreads, 0, s>>>(a);
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

constexpr int kMaxNV = 4;

// Panel width in vectors handled by one launch pair.
inline uint32_t panel_vecs() { return 32u * kMaxNV; }

inline uint32_t chunk_count(uint64_t nnz, uint32_t workers) {
  // ~8 chunks per resident worker for tail smoothing, >= 64 nnz each.
  uint64_t by_size = ceil_div(nnz, 64);
  uint64_t by_workers = uint64_t(workers) * 8;
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
  int VEC = 1, blocks = 0, fix_blocks = 0;
  uint32_t pv = 0, nchunks = 0, wstride = 0;
  uint64_t Q = 0;
  size_t bytes = 0;
};

template <typename T>
SpmmPlan make_plan(uint64_t nnz, uint32_t n, bool vec_ok) {
  constexpr int VV = sizeof(T) == 4 ? 4 : 2;
  SpmmPlan P;
  P.VEC = vec_ok ? VV : 1;
  const uint32_t nvec_total = n / P.VEC;
  const int sms = num_sms();
  P.pv = std::min<uint32_t>(nvec_total, panel_vecs());
  int NV = 1;
  const int G = groups_for(P.pv, &NV);
  const int blocks_max = sms * 8;  // 8 x 256 threads per SM (register bound)
  const uint32_t per_block = kThreads / G;
  const uint32_t workers = uint32_t(blocks_max) * per_block;
  const uint32_t nchunks = chunk_count(std::max<uint64_t>(nnz, 1), workers);
  P.Q = ceil_div(std::max<uint64_t>(nnz, 1), nchunks);
  P.nchunks = uint32_t(ceil_div(std::max<uint64_t>(nnz, 1), P.Q));
  P.wstride = uint32_t(ceil_div(uint64_t(P.pv) * P.VEC, 4) * 4);
  P.bytes = 2 * size_t(P.nchunks) * P.wstride * sizeof(T) +
            size_t(P.nchunks) * 4 + 256;
  P.blocks = int(std::min<uint64_t>(blocks_max, ceil_div(P.nchunks, per_block)));
  P.fix_blocks = int(std::min<uint64_t>(sms * 4, ceil_div(P.nchunks, per_block)));
  return P;
}

template <typename T>
size_t workspace_bytes_impl(uint32_t rows, uint64_t nnz, uint32_t n) {
  (void)rows;
  return std::max(make_plan<T>(nnz, n, true).bytes,
                  make_plan<T>(nnz, n, false).bytes);
}

template <typename T>
int spmm_impl(uint32_t rows, uint32_t cols, uint32_t n, uint64_t nnz,
              const uint32_t* rp, const uint32_t* ci, const T* val, const T* B,
              uint64_t ldb, T* C, uint64_t ldc, unsigned flags, void* ws,
              size_t ws_bytes, rdmm_stream_t stream, uint64_t* flops,
              const T* const* bseg = nullptr, uint32_t nseg = 0, uint32_t seg_rows = 0) {
  if (flops) *flops = 2ull * nnz * n;
  const bool czero = (flags & RDMM_SPMM_C_ZERO) != 0;
  if (ldb < n || ldc < n)
    return fail(RDMM_ERR_DIMENSION, "spmm: leading dimension smaller than n");
  if (rows == 0 || n == 0 || nnz == 0) return RDMM_OK;
  if (!rp || !ci || !val || (!B && !nseg) || !C)
    return fail(RDMM_ERR_INVALID, "spmm: null device pointer");
  cudaStream_t s = as_stream(stream);
  constexpr int VV = sizeof(T) == 4 ? 4 : 2;
  if (nseg > 16) return fail(RDMM_ERR_INVALID, "spmm: at most 16 B segments");
  bool seg_aligned = true;
  for (uint32_t q = 0; q < nseg; ++q)
    seg_aligned &= (reinterpret_cast<uintptr_t>(bseg[q]) % 16) == 0;
  const bool vec_ok = n % VV == 0 && ldb % VV == 0 && ldc % VV == 0 &&
                      (nseg ? seg_aligned : (reinterpret_cast<uintptr_t>(B) % 16) == 0) &&
                      (reinterpret_cast<uintptr_t>(C) % 16) == 0;
  const SpmmPlan P = make_plan<T>(nnz, n, vec_ok);
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
  const uint32_t nvec_total = n / P.VEC;
  KernelTimer timer(s, 1);
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
    else
      dispatch<T, VV>(a, czero, g, nvp, P.blocks, P.fix_blocks, s);
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
