// spgemm.cu -- C = sum_t A_t * B_t (+ identity terms) on sm_100a: the
// row-wise Gustavson product of the reference, generalised to a list of
// terms so that one kernel family covers
//   spgemm_local(a, b)        tile.hpp:211-255   one term  A*B
//   csr_add(a, b)             tile.hpp:257-288   two identity terms  I*a + I*b
//   stationary-C accumulate   algos.hpp:250-263  I*C0 + sum_k A(i,k) B(k,j)
//   queue drain accumulate    algos.hpp:278-293  I*C + sum_q I*P_q
// Output rows are sorted and keep cancelled zeros (tile.hpp:211-213): the
// pattern is the union of the symbolic products.
//
// Two passes:
//  1. bin rows by the product count ub (= spgemm_flops/2 per row,
//     tile.hpp:197-209); symbolic count of distinct columns per row in a
//     shared-memory hash table sized to the bin (64 .. 32768 keys), or a
//     global dense bitmap for the heaviest rows;  exclusive scan -> row_ptr.
//  2. re-bin by the exact output count; numeric accumulation in a shared
//     hash table (keys + values, load <= 0.5), bitonic sort in shared memory,
//     store;  the heaviest rows use a per-CTA dense bitmap + dense value
//     array whose in-order bitmap scan emits sorted columns directly.
// Products of a row are enumerated "flattened": a window of G A-entries is
// prefix-summed over their B-row lengths and the group's threads take
// consecutive products, so B rows are read coalesced and hub rows of R-MAT
// do not serialise on one thread.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace rdmm_impl {
namespace {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr int kTiers = 6;  // 5 hash tiers + dense

template <typename T>
struct TermDev {
  const uint32_t* arp;  // nullptr: identity term (row r of B as-is)
  const uint32_t* aci;
  const T* av;
  const uint32_t* brp;
  const uint32_t* bci;
  const T* bv;
};

// Symbolic tiers: ub <= limit -> table of 2*limit keys (64 .. 32768), G
// threads per row (32 = a warp per row, 8 rows per CTA; else a CTA per row).
__host__ __device__ constexpr uint32_t sym_limit(int i) {
  return i == 0 ? 32u : i == 1 ? 256u : i == 2 ? 1024u : i == 3 ? 4096u : 16384u;
}
// Numeric tiers by exact output count (load factor <= 0.5).
__host__ __device__ constexpr uint32_t num_limit(int i) {
  return i == 0 ? 32u : i == 1 ? 256u : i == 2 ? 1024u : i == 3 ? 4096u : 8192u;
}
constexpr int kDenseThreads = 1024;

__device__ __forceinline__ uint32_t hslot(uint32_t key, int log2t) {
  return (key * 0x9E3779B1u) >> (32 - log2t);
}

template <int G>
__device__ __forceinline__ void gsync() {
  if constexpr (G == 32)
    __syncwarp();
  else
    __syncthreads();
}

// Exclusive scan over the G threads of a group; returns the group total.
template <int G>
__device__ __forceinline__ uint32_t gscan(uint32_t v, uint32_t* sums,
                                          uint32_t& total) {
  const uint32_t tg = threadIdx.x % G, lane = tg & 31, warp = tg >> 5;
  uint32_t x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= uint32_t(off)) x += y;
  }
  if constexpr (G == 32) {
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  } else {
    constexpr int W = G / 32;
    if (lane == 31) sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t s = lane < uint32_t(W) ? sums[lane] : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, s, off);
        if (lane >= uint32_t(off)) s += y;
      }
      if (lane < uint32_t(W)) sums[lane] = s;
    }
    __syncthreads();
    const uint32_t base = warp ? sums[warp - 1] : 0u;
    total = sums[W - 1];
    __syncthreads();
    return base + x - v;
  }
}

template <int G>
__device__ __forceinline__ uint32_t gsum(uint32_t v, uint32_t* sums) {
  uint32_t total;
  gscan<G>(v, sums, total);
  return total;
}

// Window scratch for one group (G entries).
template <typename T, int G>
struct Win {
  uint32_t pre[G];
  uint32_t bs[G];
  uint32_t be[G];
  T a[G];
  uint32_t sums[32];
};

// Enumerate every product (column key, value) of row r over all terms and
// hand it to ins(key, value).  Identity terms contribute row r of B.
template <typename T, int G, bool kValues, class Ins>
__device__ __forceinline__ void enumerate_row(uint32_t r,
                                              const TermDev<T>* terms,
                                              int nterms, Win<T, G>& w,
                                              Ins ins, uint32_t part = 0,
                                              uint32_t nparts = 1) {
  const uint32_t tg = threadIdx.x % G;
  for (int t = 0; t < nterms; ++t) {
    const TermDev<T> tm = terms[t];
    const bool ident = tm.arp == nullptr;
    const uint32_t s0 = ident ? 0u : __ldg(tm.arp + r);
    const uint32_t s1 = ident ? 1u : __ldg(tm.arp + r + 1);
    for (uint32_t base = s0; base < s1; base += G) {
      const uint32_t e = base + tg;
      uint32_t len = 0, bs = 0;
      T a = T(1);
      if (e < s1) {
        const uint32_t k = ident ? r : __ldg(tm.aci + e);
        if (kValues && !ident) a = __ldg(tm.av + e);
        bs = __ldg(tm.brp + k);
        len = __ldg(tm.brp + k + 1) - bs;
      }
      uint32_t total;
      const uint32_t ex = gscan<G>(len, w.sums, total);
      w.pre[tg] = ex;
      w.bs[tg] = bs;
      if (kValues) w.a[tg] = a;
      gsync<G>();
      const uint32_t nvalid = min(uint32_t(G), s1 - base);
      for (uint32_t p = tg + part * G; p < total; p += nparts * G) {
        uint32_t lo = 0, hi = nvalid;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (w.pre[mid] <= p)
            lo = mid;
          else
            hi = mid;
        }
        const uint32_t tt = w.bs[lo] + (p - w.pre[lo]);
        const uint32_t key = __ldg(tm.bci + tt);
        T v = T(0);
        if (kValues) v = ident ? __ldg(tm.bv + tt) : w.a[lo] * __ldg(tm.bv + tt);
        ins(key, v);
      }
      gsync<G>();
    }
  }
}

// Heavy rows, segmented: a window of G A entries is cut into work items of at
// most kSeg consecutive products of one B row (a block scan of the items per
// entry); each warp of the CTA (and of the `nparts` CTAs sharing the row)
// takes whole items, its lanes reading the B-row segment coalesced.  Balanced
// like the flattened enumeration (R-MAT hub B rows become many items) at one
// binary search per item instead of one per product.
constexpr uint32_t kSeg = 256;
template <typename T, int G, bool kValues, class Ins>
__device__ __forceinline__ void enumerate_row_seg(uint32_t r, const TermDev<T>* terms,
                                                  int nterms, Win<T, G>& w, Ins ins,
                                                  uint32_t part = 0, uint32_t nparts = 1) {
  const uint32_t tg = threadIdx.x % G, lane = tg & 31, wid = tg >> 5;
  constexpr uint32_t W = G / 32;
  for (int t = 0; t < nterms; ++t) {
    const TermDev<T> tm = terms[t];
    const bool ident = tm.arp == nullptr;
    const uint32_t s0 = ident ? 0u : __ldg(tm.arp + r);
    const uint32_t s1 = ident ? 1u : __ldg(tm.arp + r + 1);
    for (uint32_t base = s0; base < s1; base += G) {
      const uint32_t e = base + tg;
      uint32_t bs = 0, be = 0;
      T a = T(1);
      if (e < s1) {
        const uint32_t k = ident ? r : __ldg(tm.aci + e);
        if (kValues && !ident) a = __ldg(tm.av + e);
        bs = __ldg(tm.brp + k);
        be = __ldg(tm.brp + k + 1);
      }
      uint32_t items;
      const uint32_t ex = gscan<G>((be - bs + kSeg - 1) / kSeg, w.sums, items);
      w.pre[tg] = ex;
      w.bs[tg] = bs;
      w.be[tg] = be;
      if (kValues) w.a[tg] = a;
      gsync<G>();
      const uint32_t nvalid = min(uint32_t(G), s1 - base);
      for (uint32_t it = part * W + wid; it < items; it += nparts * W) {
        uint32_t lo = 0, hi = nvalid;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (w.pre[mid] <= it)
            lo = mid;
          else
            hi = mid;
        }
        const uint32_t q0 = w.bs[lo] + (it - w.pre[lo]) * kSeg;
        const uint32_t q1 = min(q0 + kSeg, w.be[lo]);
        const T av = kValues ? w.a[lo] : T(1);
        for (uint32_t q = q0 + lane; q < q1; q += 32) {
          const uint32_t key = __ldg(tm.bci + q);
          T v = T(0);
          if (kValues) v = ident ? __ldg(tm.bv + q) : av * __ldg(tm.bv + q);
          ins(key, v);
        }
      }
      gsync<G>();
    }
  }
}

// Heavy rows: each warp of the CTA (and of the `nparts` CTAs sharing the
// row) takes whole A entries, its lanes stride over the entry's B row
// (coalesced, no search); two products per lane are loaded before they are
// inserted.  Used by the large CTA tiers and the dense tier.
template <typename T, int G, bool kValues, class Ins>
__device__ __forceinline__ void enumerate_row_warps(uint32_t r, const TermDev<T>* terms,
                                                    int nterms, Ins ins, uint32_t part = 0,
                                                    uint32_t nparts = 1) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr uint32_t W = G / 32;
  const uint32_t gw = part * W + wid, nw = nparts * W;
  for (int t = 0; t < nterms; ++t) {
    const TermDev<T> tm = terms[t];
    const bool ident = tm.arp == nullptr;
    const uint32_t s0 = ident ? 0u : __ldg(tm.arp + r);
    const uint32_t s1 = ident ? 1u : __ldg(tm.arp + r + 1);
    for (uint32_t e = s0 + gw; e < s1; e += nw) {
      const uint32_t k = ident ? r : __ldg(tm.aci + e);
      T a = T(1);
      if (kValues && !ident) a = __ldg(tm.av + e);
      const uint32_t bs = __ldg(tm.brp + k), be = __ldg(tm.brp + k + 1);
      for (uint32_t q = bs + lane; q < be; q += 64) {
        const bool two = q + 32 < be;
        const uint32_t k0 = __ldg(tm.bci + q);
        const uint32_t k1 = two ? __ldg(tm.bci + q + 32) : 0u;
        T v0 = T(0), v1 = T(0);
        if (kValues) {
          v0 = __ldg(tm.bv + q);
          if (two) v1 = __ldg(tm.bv + q + 32);
          if (!ident) {
            v0 = a * v0;
            v1 = a * v1;
          }
        }
        ins(k0, v0);
        if (two) ins(k1, v1);
      }
    }
  }
}

// ------------------------------------------------------------ binning

// Warp per row: ub[r] = number of products; bin by symbolic tier.  Per-term
// product counts (the reference FlopMeter per multiply, tile.hpp:197-209) are
// reduced in shared memory and flushed with one global atomic per term per
// block.
template <typename T>
__global__ void k_bin_sym(uint32_t rows, const TermDev<T>* terms, int nterms,
                          uint32_t* lists, uint32_t* tier_count,
                          unsigned long long* term_products, uint64_t* cnt64) {
  extern __shared__ unsigned long long sacc[];
  for (int t = threadIdx.x; t < nterms; t += blockDim.x) sacc[t] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = warp; r < rows; r += nwarps) {
    unsigned long long ub = 0;
    for (int t = 0; t < nterms; ++t) {
      const TermDev<T> tm = terms[t];
      unsigned long long tp = 0;
      if (tm.arp == nullptr) {
        if (lane == 0) tp = __ldg(tm.brp + r + 1) - __ldg(tm.brp + r);
      } else {
        const uint32_t s0 = __ldg(tm.arp + r), s1 = __ldg(tm.arp + r + 1);
        for (uint32_t e = s0 + lane; e < s1; e += 32) {
          const uint32_t k = __ldg(tm.aci + e);
          tp += __ldg(tm.brp + k + 1) - __ldg(tm.brp + k);
        }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) tp += __shfl_xor_sync(0xffffffffu, tp, off);
      if (lane == 0 && tp && tm.arp != nullptr) atomicAdd(sacc + t, tp);
      ub += tp;
    }
    if (lane == 0) {
      cnt64[r] = 0;
      if (ub) {
        int tier = 5;
        for (int i = 0; i < 5; ++i)
          if (ub <= sym_limit(i)) {
            tier = i;
            break;
          }
        const uint32_t pos = atomicAdd(tier_count + tier, 1u);
        lists[size_t(tier) * rows + pos] = r;
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nterms; t += blockDim.x)
    if (sacc[t]) atomicAdd(term_products + t, sacc[t]);
}

__global__ void k_bin_num(uint32_t rows, const uint64_t* cnt64, uint32_t* lists,
                          uint32_t* tier_count) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += gridDim.x * blockDim.x) {
    const uint64_t c = cnt64[r];
    if (!c) continue;
    int tier = 5;
    for (int i = 0; i < 5; ++i)
      if (c <= num_limit(i)) {
        tier = i;
        break;
      }
    const uint32_t pos = atomicAdd(tier_count + tier, 1u);
    lists[size_t(tier) * rows + pos] = r;
  }
}

// ------------------------------------------------------------ hash tiers

template <typename T, int TAB, int G>
__global__ void __launch_bounds__(G == 32 ? 256 : G)
    k_sym_hash(const uint32_t* __restrict__ list, uint32_t count,
               const TermDev<T>* terms, int nterms, uint64_t* cnt64, int flat) {
  constexpr int RPB = G == 32 ? 8 : 1;  // rows per block
  constexpr int LOG2T = __builtin_ctz(TAB);
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t grp = threadIdx.x / G, tg = threadIdx.x % G;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem) + size_t(grp) * TAB;
  Win<T, G>* win = reinterpret_cast<Win<T, G>*>(
      smem + size_t(RPB) * TAB * 4) + grp;
  for (uint32_t li = blockIdx.x * RPB + grp; li - grp < count;
       li += gridDim.x * RPB) {
    const bool active = li < count;  // whole group uniform
    if (!active) {
      if constexpr (G == 32) break;
    }
    const uint32_t r = active ? list[li] : 0u;
    for (uint32_t i = tg; i < TAB; i += G) keys[i] = kEmpty;
    gsync<G>();
    auto sym_ins = [&](uint32_t key, T) {
        uint32_t s = hslot(key, LOG2T);
        for (;;) {
          const uint32_t cur = reinterpret_cast<volatile uint32_t*>(keys)[s];
          if (cur == key) break;
          if (cur == kEmpty) {
            const uint32_t old = atomicCAS(keys + s, kEmpty, key);
            if (old == kEmpty || old == key) break;
          }
          s = (s + 1) & (TAB - 1);
        }
    };
    if (active) {
      if (G >= 512 && !flat)
        enumerate_row_warps<T, G, false>(r, terms, nterms, sym_ins);
      else if (G >= 128 && flat == 1)
        enumerate_row_seg<T, G, false>(r, terms, nterms, *win, sym_ins);
      else
        enumerate_row<T, G, false>(r, terms, nterms, *win, sym_ins);
    }
    gsync<G>();
    uint32_t c = 0;
    for (uint32_t i = tg; i < TAB; i += G) c += keys[i] != kEmpty;
    c = gsum<G>(c, win->sums);
    if (active && tg == 0) cnt64[r] = c;
    gsync<G>();
  }
}

// Bytes of the numeric table region: keys + values, or the block radix
// sort's scratch that aliases it, whichever is larger.
template <typename T, int TAB, int G>
constexpr size_t num_table_bytes() {
  if constexpr (G == 32) {
    return size_t(TAB) * (sizeof(T) + 4);
  } else {
    using BRS = cub::BlockRadixSort<uint32_t, G, TAB / G, T>;
    return std::max(size_t(TAB) * (sizeof(T) + 4), sizeof(typename BRS::TempStorage));
  }
}

template <typename T, int TAB, int G>
__global__ void __launch_bounds__(G == 32 ? 256 : G)
    k_num_hash(const uint32_t* __restrict__ list, uint32_t count,
               const TermDev<T>* terms, int nterms,
               const uint32_t* __restrict__ crp, uint32_t* __restrict__ cci,
               T* __restrict__ cv, T ident_val, int key_bits, int flat) {
  constexpr int RPB = G == 32 ? 8 : 1;
  constexpr int LOG2T = __builtin_ctz(TAB);
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t grp = threadIdx.x / G, tg = threadIdx.x % G;
  T* vals = reinterpret_cast<T*>(smem) + size_t(grp) * TAB;
  uint32_t* keys =
      reinterpret_cast<uint32_t*>(smem + size_t(RPB) * TAB * sizeof(T)) +
      size_t(grp) * TAB;
  Win<T, G>* win = reinterpret_cast<Win<T, G>*>(
      smem + size_t(RPB) * num_table_bytes<T, TAB, G>()) + grp;
  for (uint32_t li = blockIdx.x * RPB + grp; li - grp < count;
       li += gridDim.x * RPB) {
    const bool active = li < count;
    if (!active) {
      if constexpr (G == 32) break;
    }
    const uint32_t r = active ? list[li] : 0u;
    for (uint32_t i = tg; i < TAB; i += G) {
      keys[i] = kEmpty;
      vals[i] = ident_val;
    }
    gsync<G>();
    auto num_ins = [&](uint32_t key, T v) {
        // a plain load finds keys already present (most products of hot
        // columns) without a CAS; only empty-looking slots are CAS-claimed
        uint32_t s = hslot(key, LOG2T);
        for (;;) {
          const uint32_t cur = reinterpret_cast<volatile uint32_t*>(keys)[s];
          if (cur == key) break;
          if (cur == kEmpty) {
            const uint32_t old = atomicCAS(keys + s, kEmpty, key);
            if (old == kEmpty || old == key) break;
          }
          s = (s + 1) & (TAB - 1);
        }
        atomicAdd(vals + s, v);
    };
    if (active) {
      if (G >= 512 && !flat)
        enumerate_row_warps<T, G, true>(r, terms, nterms, num_ins);
      else if (G >= 128 && flat == 1)
        enumerate_row_seg<T, G, true>(r, terms, nterms, *win, num_ins);
      else
        enumerate_row<T, G, true>(r, terms, nterms, *win, num_ins);
    }
    gsync<G>();
    if constexpr (G == 32) {
      // warp tier: bitonic sort of the 64-slot table; empty keys sort last
      for (uint32_t k = 2; k <= uint32_t(TAB); k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = tg; i < uint32_t(TAB); i += G) {
            const uint32_t ixj = i ^ j;
            if (ixj > i) {
              const uint32_t ki = keys[i], kj = keys[ixj];
              const bool up = (i & k) == 0;
              if ((ki > kj) == up) {
                keys[i] = kj;
                keys[ixj] = ki;
                const T t = vals[i];
                vals[i] = vals[ixj];
                vals[ixj] = t;
              }
            }
          }
          gsync<G>();
        }
      }
      if (active) {
        const uint32_t o = crp[r], n = crp[r + 1] - o;
        for (uint32_t i = tg; i < n; i += G) {
          cci[o + i] = keys[i];
          cv[o + i] = vals[i];
        }
      }
      gsync<G>();
    } else {
      // CTA tiers: block radix sort of the whole table by column (bits
      // [0, key_bits)); the empty key has all of those bits set, so it sorts
      // after every real column.  The sort's scratch aliases the table.
      constexpr int IPT = TAB / G;
      using BRS = cub::BlockRadixSort<uint32_t, G, IPT, T>;
      uint32_t kk[IPT];
      T vv[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        kk[i] = keys[tg * IPT + i];
        vv[i] = vals[tg * IPT + i];
      }
      __syncthreads();
      BRS(*reinterpret_cast<typename BRS::TempStorage*>(smem)).Sort(kk, vv, 0, key_bits);
      if (active) {
        const uint32_t o = crp[r], n = crp[r + 1] - o;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t idx = tg * IPT + i;
          if (idx < n) {
            cci[o + idx] = kk[i];
            cv[o + idx] = vv[i];
          }
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ dense tier
//
// Rows whose output does not fit a shared-memory table accumulate in a dense
// value array + bitmap over all columns (global memory, per row slot).  CL
// CTAs (a thread-block cluster when CL > 1) share one row: its products are
// interleaved over the CTAs, and the in-order bitmap scan that emits sorted
// columns is split over them with the per-CTA counts exchanged through
// distributed shared memory.  R-MAT rows have hot output columns (thousands
// of products per column), so every CTA first combines products in a
// shared-memory write-combining cache (direct-mapped, CAS-claimed slots) and
// only misses and the final flush reach the global array with atomics.
// The symbolic pass keeps the whole bitmap in shared memory when it fits.
constexpr int kWc = 8192;  // write-combining slots per CTA

template <typename T, int WC = kWc>
constexpr size_t dense_smem_bytes() {
  return size_t(WC) * (4 + sizeof(T));
}

// SBM: the row's column bitmap lives in shared memory after the
// write-combining cache (CL = 1 and ncols <= ~1M fp32): the bitmap atomics,
// the count scan and the emission scan never touch HBM.
template <typename T, int CL, bool SBM, int WC = kWc>
__global__ void __launch_bounds__(kDenseThreads)
    k_dense_num(const uint32_t* __restrict__ list, uint32_t count,
                const TermDev<T>* terms, int nterms,
                const uint32_t* __restrict__ crp, uint32_t* __restrict__ cci,
                T* __restrict__ cv, uint32_t* bitmaps, T* dense, uint32_t nwords,
                uint32_t ncols, T ident_val, int flat) {
  constexpr int G = kDenseThreads;
  constexpr int LOG2W = __builtin_ctz(WC);
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* wkey = reinterpret_cast<uint32_t*>(dsm);
  T* wval = reinterpret_cast<T*>(dsm + size_t(WC) * 4);
  __shared__ Win<T, G> win;
  __shared__ uint32_t slice_count;
  __shared__ uint32_t coff[G];  // emission: output offset of each 32-word chunk
  const uint32_t part = CL > 1 ? cluster.block_rank() : 0;
  const uint32_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  uint32_t* bm = SBM ? reinterpret_cast<uint32_t*>(dsm + dense_smem_bytes<T, WC>())
                     : bitmaps + size_t(cid) * nwords;
  auto ldbm = [&](uint32_t w) -> uint32_t {
    if constexpr (SBM) return reinterpret_cast<volatile uint32_t*>(bm)[w];
    else return __ldcg(bm + w);
  };
  if constexpr (SBM)
    for (uint32_t i = threadIdx.x; i < nwords; i += G) bm[i] = 0;
  T* dv = dense + size_t(cid) * ncols;
  const uint32_t wper = (nwords + CL - 1) / CL;
  const uint32_t ws0 = min(part * wper, nwords), ws1 = min(ws0 + wper, nwords);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < WC; i += G) {
    wkey[i] = kEmpty;
    wval[i] = ident_val;
  }
  __syncthreads();
  for (uint32_t li = cid; li < count; li += ncl) {
    const uint32_t r = list[li];
    auto dense_ins = [&](uint32_t key, T v) {
          const uint32_t sl = hslot(key, LOG2W);
          const uint32_t cur = reinterpret_cast<volatile uint32_t*>(wkey)[sl];
          const uint32_t old = cur == kEmpty ? atomicCAS(wkey + sl, kEmpty, key) : cur;
          if (old == key) {  // cached: its bit is already set
            atomicAdd(wval + sl, v);
            return;
          }
          const uint32_t bit = 1u << (key & 31);
          if (!(ldbm(key >> 5) & bit)) atomicOr(bm + (key >> 5), bit);
          if (old == kEmpty)
            atomicAdd(wval + sl, v);
          else
            atomicAdd(dv + key, v);
        };
    // flat: products spread over every thread of the CTA(s) by a block scan
    // of the B-row lengths (balanced); otherwise whole A entries per warp
    if (flat == 2)
      enumerate_row<T, G, true>(r, terms, nterms, win, dense_ins, part, CL);
    else if (flat)
      enumerate_row_seg<T, G, true>(r, terms, nterms, win, dense_ins, part, CL);
    else
      enumerate_row_warps<T, G, true>(r, terms, nterms, dense_ins, part, CL);
    // CL = 1, no flush: a column's products all went to the cache slot it
    // claimed first or all to the dense array (slots are never evicted), so
    // the emission reads each column from where it accumulated.  CL > 1: the
    // CTAs' caches overlap; flush them into the dense array.
    __syncthreads();
    if constexpr (CL > 1) {
      for (uint32_t i = threadIdx.x; i < WC; i += G) {
        const uint32_t key = wkey[i];
        if (key != kEmpty) {
          atomicAdd(dv + key, wval[i]);
          wkey[i] = kEmpty;
          wval[i] = ident_val;
        }
      }
    }
    __threadfence();
    if constexpr (CL > 1) cluster.sync(); else __syncthreads();
    // Emission in column order, balanced over the threads: the slice's
    // words form chunks of 32; a block scan of the chunk counts gives each
    // chunk's output offset, and the warps take chunks interleaved (R-MAT's
    // output columns crowd the low words, which a contiguous word range per
    // thread turned into a barrier wait behind a few threads), one word per
    // lane with a warp scan for the positions inside the chunk.
    const uint32_t nchunk = (ws1 - ws0 + 31) / 32;
    uint32_t base = 0;
    if constexpr (CL > 1) {
      uint32_t c = 0;
      for (uint32_t w = ws0 + threadIdx.x; w < ws1; w += G) c += __popc(ldbm(w));
      const uint32_t tot = gsum<G>(c, win.sums);
      if (threadIdx.x == 0) slice_count = tot;
      cluster.sync();
      for (uint32_t q = 0; q < part; ++q) base += *cluster.map_shared_rank(&slice_count, q);
    }
    uint32_t run = crp[r] + base;
    for (uint32_t g0 = 0; g0 < nchunk; g0 += G) {
      const uint32_t ch = g0 + threadIdx.x;
      uint32_t c = 0;
      if (ch < nchunk) {
        const uint32_t wa = ws0 + ch * 32, wb = min(wa + 32, ws1);
        for (uint32_t w = wa; w < wb; ++w) c += __popc(ldbm(w));
      }
      uint32_t total;
      coff[threadIdx.x] = gscan<G>(c, win.sums, total);
      __syncthreads();
      for (uint32_t j = warp; j < uint32_t(G) && g0 + j < nchunk; j += G / 32) {
        const uint32_t w = ws0 + (g0 + j) * 32 + lane;
        uint32_t bits = w < ws1 ? ldbm(w) : 0u;
        const uint32_t cnt = __popc(bits);
        uint32_t inc = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= uint32_t(off)) inc += y;
        }
        uint32_t pos = run + coff[j] + inc - cnt;
        if (bits) bm[w] = 0;
        while (bits) {  // eight columns per round: their value loads overlap
          uint32_t cols[8];
          T vals[8];
          int nb = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            cols[q] = w * 32 + (bits ? __ffs(bits) - 1 : 0u);
            if (bits) {
              bits &= bits - 1;
              nb = q + 1;
            }
          }
          bool cached[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t sl = hslot(cols[q], LOG2W);
            cached[q] = CL == 1 && q < nb && wkey[sl] == cols[q];
            if (q < nb) vals[q] = cached[q] ? wval[sl] : __ldcg(dv + cols[q]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < nb) {
              cci[pos + q] = cols[q];
              cv[pos + q] = vals[q];
              if (!cached[q]) dv[cols[q]] = ident_val;
            }
          pos += uint32_t(nb);
        }
      }
      run += total;
      __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < WC; i += G) {  // reset the cache
      wkey[i] = kEmpty;
      wval[i] = ident_val;
    }
    __threadfence();
    if constexpr (CL > 1) cluster.sync(); else __syncthreads();
  }
}

// Symbolic heavy rows: the column bitmap lives in shared memory (ncols bits).
template <typename T>
__global__ void __launch_bounds__(kDenseThreads)
    k_dense_sym_smem(const uint32_t* __restrict__ list, uint32_t count,
                     const TermDev<T>* terms, int nterms, uint64_t* cnt64, uint32_t nwords) {
  constexpr int G = kDenseThreads;
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(dsm);
  __shared__ Win<T, G> win;
  for (uint32_t i = threadIdx.x; i < nwords; i += G) bm[i] = 0;
  __syncthreads();
  for (uint32_t li = blockIdx.x; li < count; li += gridDim.x) {
    const uint32_t r = list[li];
    enumerate_row_warps<T, G, false>(r, terms, nterms, [&](uint32_t key, T) {
      const uint32_t bit = 1u << (key & 31);
      if (!(bm[key >> 5] & bit)) atomicOr(bm + (key >> 5), bit);
    });
    __syncthreads();
    uint32_t c = 0;
    for (uint32_t i = threadIdx.x; i < nwords; i += G) {
      c += __popc(bm[i]);
      bm[i] = 0;
    }
    c = gsum<G>(c, win.sums);
    if (threadIdx.x == 0) cnt64[r] = c;
    __syncthreads();
  }
}

// Symbolic heavy rows when the bitmap does not fit shared memory.
template <typename T>
__global__ void __launch_bounds__(kDenseThreads)
    k_dense_sym_global(const uint32_t* __restrict__ list, uint32_t count,
                       const TermDev<T>* terms, int nterms, uint64_t* cnt64,
                       uint32_t* bitmaps, uint32_t nwords) {
  constexpr int G = kDenseThreads;
  __shared__ Win<T, G> win;
  uint32_t* bm = bitmaps + size_t(blockIdx.x) * nwords;
  for (uint32_t li = blockIdx.x; li < count; li += gridDim.x) {
    const uint32_t r = list[li];
    enumerate_row_warps<T, G, false>(r, terms, nterms, [&](uint32_t key, T) {
      const uint32_t bit = 1u << (key & 31);
      if (!(__ldcg(bm + (key >> 5)) & bit)) atomicOr(bm + (key >> 5), bit);
    });
    __threadfence();
    __syncthreads();
    uint32_t c = 0;
    for (uint32_t i = threadIdx.x; i < nwords; i += G) {
      c += __popc(__ldcg(bm + i));
      bm[i] = 0;
    }
    c = gsum<G>(c, win.sums);
    if (threadIdx.x == 0) cnt64[r] = c;
    __threadfence();
    __syncthreads();
  }
}

constexpr size_t kSymSmemMax = 200 * 1024;  // bitmap bytes kept in shared memory

template <typename T>
__global__ void k_fill(T* p, size_t n, T v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_rowptr32(const uint64_t* pre, uint32_t n1, uint32_t* rp) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n1;
       i += gridDim.x * blockDim.x)
    rp[i] = uint32_t(pre[i]);
}

// CTAs per dense row (RDMM_SPGEMM_CL, default 1: more rows in flight spread
// the hot-column atomics over more addresses).
inline int dense_cl() {
  static const int v = [] {
    const char* e = std::getenv("RDMM_SPGEMM_CL");
    const int x = e ? std::atoi(e) : 1;
    return x == 8 ? 8 : x == 4 ? 4 : x == 2 ? 2 : 1;
  }();
  return v;
}
// Product enumeration for the CTA tiers (G >= 128) and the dense tier:
// 2 (default) = flattened products (a block scan of the B-row lengths per
// window of A entries, a binary search per product); 1 = segmented items
// (kSeg products of one B row per warp, one search per item: fewer
// instructions but measured 6% slower at s20, 141 vs 133 ms); 0 = whole A
// entries per warp, which leaves warps waiting at the row barrier behind
// R-MAT hub B rows (ncu: barrier stalls 92 cycles/instr; s20 283 ms vs
// 207 ms).  RDMM_SPGEMM_FLAT overrides (a measurement switch).
inline int dense_flat() {
  static const int v = [] {
    const char* e = std::getenv("RDMM_SPGEMM_FLAT");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
inline uint32_t dense_rows_in_flight(uint32_t rows, int cl) {
  return std::max<uint32_t>(1, std::min<uint32_t>(rows, uint32_t(num_sms()) / cl));
}
// Numeric dense tier: rows in flight (one per SM; limiting them so that the
// dense arrays stay L2-resident measured 4.6x slower at 18 rows: the tier is
// bound by per-row work, not by DRAM).  RDMM_SPGEMM_DENSE_SLOTS overrides (a
// measurement switch).
inline uint32_t dense_num_slots(uint32_t rows, size_t bytes_per_row, int cl) {
  static const int env = [] {
    const char* e = std::getenv("RDMM_SPGEMM_DENSE_SLOTS");
    return e ? std::atoi(e) : 0;
  }();
  int dev = 0;
  cudaGetDevice(&dev);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  (void)l2;
  (void)bytes_per_row;
  uint32_t fit = env > 0 ? uint32_t(env) : uint32_t(num_sms());
  return std::max<uint32_t>(1, std::min<uint32_t>({rows, fit, uint32_t(num_sms()) / cl}));
}
// Side stream per device for tiers that run concurrently with the others.
inline cudaStream_t side_stream() {
  static cudaStream_t ss[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!ss[dev & 63]) cudaStreamCreateWithFlags(&ss[dev & 63], cudaStreamNonBlocking);
  return ss[dev & 63];
}

template <typename T, int CL>
int launch_dense_num(uint32_t slots, const uint32_t* list, uint32_t count,
                     const TermDev<T>* td, int nt, const uint32_t* crp, uint32_t* cci, T* cv,
                     uint32_t* bm, T* dense, uint32_t nwords, uint32_t ncols, T ident,
                     cudaStream_t s) {
  // static shared memory of the kernel: Win<T, G> + a counter
  const size_t stat = sizeof(Win<T, kDenseThreads>) + 64 + kDenseThreads * 4;
  // 16384 write-combining slots (the bitmap then lives in global memory /
  // L2): cfg4 s20 132.8 -> 129.7 ms against 8192 slots with the bitmap in
  // shared memory.  RDMM_SPGEMM_WC=8192 restores the latter (a measurement
  // switch).
  static const int wc_env = [] {
    const char* e = std::getenv("RDMM_SPGEMM_WC");
    return e ? std::atoi(e) : 0;
  }();
  const bool big = wc_env != kWc;
  const size_t wcb = big ? dense_smem_bytes<T, 2 * kWc>() : dense_smem_bytes<T>();
  const bool sbm = CL == 1 && wcb + size_t(nwords) * 4 + stat <= 226 * 1024;
  auto fn = big ? (sbm ? k_dense_num<T, CL, true, 2 * kWc> : k_dense_num<T, CL, false, 2 * kWc>)
                : (sbm ? k_dense_num<T, CL, true> : k_dense_num<T, CL, false>);
  const size_t sm = wcb + (sbm ? size_t(nwords) * 4 : 0);
  RDMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(slots * CL);
  cfg.blockDim = dim3(kDenseThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  RDMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, list, count, td, nt, crp, cci, cv, bm, dense,
                                   nwords, ncols, ident, dense_flat()));
  return RDMM_OK;
}

// ------------------------------------------------------------ deterministic
//
// Opt-in numeric pass with the reference's floating-point result for ANY
// values (RDMM_SPGEMM_DETERMINISTIC): every product of a batch of rows is
// expanded in enumeration order (term, A entry, B entry -- the reference's
// loop order, tile.hpp:225-237) as (key = row|col|term, a, b), a stable radix
// sort groups equal keys keeping that order, and one thread per output entry
// folds its run: within a product term sum = fma(a, b, sum) from +0 in order
// (tile.hpp:232); identity terms contribute their value as-is; term results
// combine in term order, first value copied, later ones added -- csr_add
// (tile.hpp:257-288) applied per term as stationary-C does (algos.hpp:254).
template <typename T>
struct AB {
  T a, b;
};

template <typename T>
__global__ void k_det_count(uint32_t r0, uint32_t rows, const TermDev<T>* terms, int nterms,
                            uint64_t* cnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows;
       w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t r = r0 + w;
    unsigned long long n = 0;
    for (int t = 0; t < nterms; ++t) {
      const TermDev<T> tm = terms[t];
      if (tm.arp == nullptr) {
        if (lane == 0) n += __ldg(tm.brp + r + 1) - __ldg(tm.brp + r);
      } else {
        for (uint32_t e = __ldg(tm.arp + r) + lane; e < __ldg(tm.arp + r + 1); e += 32) {
          const uint32_t k = __ldg(tm.aci + e);
          n += __ldg(tm.brp + k + 1) - __ldg(tm.brp + k);
        }
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) n += __shfl_xor_sync(0xffffffffu, n, off);
    if (lane == 0) cnt[w] = n;
  }
}

// warp per row; products written at off[row] + running index, in
// enumeration order (lanes stride a B row; the A entries and terms advance
// uniformly)
template <typename T>
__global__ void k_det_expand(uint32_t r0, uint32_t rows, const TermDev<T>* terms, int nterms,
                             const uint64_t* off, uint64_t* keys, AB<T>* ab) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < rows;
       w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t r = r0 + w;
    uint64_t o = off[w];
    for (int t = 0; t < nterms; ++t) {
      const TermDev<T> tm = terms[t];
      const bool ident = tm.arp == nullptr;
      const uint32_t s0 = ident ? 0u : __ldg(tm.arp + r), s1 = ident ? 1u : __ldg(tm.arp + r + 1);
      for (uint32_t e = s0; e < s1; ++e) {
        const uint32_t k = ident ? r : __ldg(tm.aci + e);
        const T a = ident ? T(1) : __ldg(tm.av + e);
        const uint32_t bs = __ldg(tm.brp + k), be = __ldg(tm.brp + k + 1);
        for (uint32_t q = bs + lane; q < be; q += 32) {
          const uint64_t pos = o + (q - bs);
          keys[pos] = (uint64_t(w) << 40) | (uint64_t(__ldg(tm.bci + q)) << 8) | uint64_t(t);
          ab[pos] = AB<T>{a, __ldg(tm.bv + q)};
        }
        o += be - bs;
      }
    }
  }
}

// one thread per (row, col) run of the sorted products: fold the run
__global__ void k_det_heads(const uint64_t* keys, uint64_t n, uint32_t* head) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || (keys[i] >> 8) != (keys[i - 1] >> 8)) ? 1u : 0u;
}

template <typename T>
__global__ void k_det_fold(const uint64_t* keys, const AB<T>* ab, uint64_t n,
                           const uint32_t* head, const uint32_t* hpos, const TermDev<T>* terms,
                           uint64_t cbase, uint32_t* cci, T* cv) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (!head[i]) continue;
    const uint64_t rc = keys[i] >> 8;
    T acc = T(0);
    bool have = false;
    uint64_t j = i;
    while (j < n && (keys[j] >> 8) == rc) {
      const int t = int(keys[j] & 0xff);
      const bool ident = terms[t].arp == nullptr;
      T tsum;
      if (ident) {
        tsum = ab[j].b;  // the identity term's value as-is (keeps -0.0)
        ++j;
      } else {
        tsum = T(0);
        while (j < n && keys[j] == ((rc << 8) | uint64_t(t))) {
          tsum = fma(ab[j].a, ab[j].b, tsum);
          ++j;
        }
      }
      acc = have ? acc + tsum : tsum;
      have = true;
    }
    const uint64_t o = cbase + hpos[i];
    cci[o] = uint32_t(rc & 0xffffffffu);
    cv[o] = acc;
  }
}

// Plan workspace: grow-only stream-ordered scratch per (device, stream,
// slot) (common.cuh), so repeated products on one stream allocate nothing.
// A stream has at most one SpGEMM plan in flight (symbolic -> numeric).
struct Buf {
  void* p = nullptr;
  size_t n = 0;
  int slot = 0;
  cudaError_t ensure(size_t bytes, cudaStream_t s) {
    void* q = scratch(bytes ? bytes : 8, slot, s);
    if (!q) return cudaErrorMemoryAllocation;
    p = q;
    n = bytes;
    return cudaSuccess;
  }
  template <typename X>
  X* as() const {
    return static_cast<X*>(p);
  }
};

template <typename T, int TAB, int G>
size_t hash_smem(bool numeric) {
  constexpr int RPB = G == 32 ? 8 : 1;
  return size_t(RPB) * (numeric ? num_table_bytes<T, TAB, G>() : size_t(TAB) * 4) +
         size_t(RPB) * sizeof(Win<T, G>);
}

template <typename T, int TAB, int G>
int launch_sym_hash(const uint32_t* list, uint32_t count,
                    const TermDev<T>* terms, int nterms, uint64_t* cnt64,
                    cudaStream_t s) {
  if (!count) return 0;
  constexpr int RPB = G == 32 ? 8 : 1;
  const size_t sm = hash_smem<T, TAB, G>(false);
  auto fn = k_sym_hash<T, TAB, G>;
  if (sm > 48 * 1024)
    RDMM_CUDA_TRY(cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  const int threads = G == 32 ? 256 : G;
  const uint64_t blocks = std::min<uint64_t>(ceil_div(count, RPB),
                                             uint64_t(num_sms()) * 64);
  count_launch();
  fn<<<unsigned(blocks), threads, sm, s>>>(list, count, terms, nterms, cnt64, dense_flat());
  return 0;
}

template <typename T, int TAB, int G>
int launch_num_hash(const uint32_t* list, uint32_t count,
                    const TermDev<T>* terms, int nterms, const uint32_t* crp,
                    uint32_t* cci, T* cv, T ident, int key_bits, cudaStream_t s) {
  if (!count) return 0;
  constexpr int RPB = G == 32 ? 8 : 1;
  const size_t sm = hash_smem<T, TAB, G>(true);
  auto fn = k_num_hash<T, TAB, G>;
  if (sm > 48 * 1024)
    RDMM_CUDA_TRY(cudaFuncSetAttribute(
        fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
  const int threads = G == 32 ? 256 : G;
  const uint64_t blocks = std::min<uint64_t>(ceil_div(count, RPB),
                                             uint64_t(num_sms()) * 64);
  count_launch();
  fn<<<unsigned(blocks), threads, sm, s>>>(list, count, terms, nterms, crp,
                                           cci, cv, ident, key_bits, dense_flat());
  return 0;
}

}  // namespace
}  // namespace rdmm_impl

using namespace rdmm_impl;

struct rdmm_spgemm_plan {
  int dtype = 4;
  uint32_t rows = 0, ncols = 0;
  int nterms = 0;
  bool ident_only = false;
  Buf terms, cnt64, pre64, lists, tcount, ub, scan_tmp, bitmaps, dense;
  rdmm_spgemm_plan() {
    int slot = 10;
    for (Buf* b : {&terms, &cnt64, &pre64, &lists, &tcount, &ub, &scan_tmp, &bitmaps, &dense})
      b->slot = slot++;
  }
  uint32_t sym_count[kTiers] = {0}, num_count[kTiers] = {0};
  uint64_t nnz = 0, flops = 0;
  std::vector<uint64_t> term_flops;
  uint32_t* c_row_ptr = nullptr;
};

namespace {

template <typename T>
int symbolic_impl(uint32_t rows, uint32_t ncols, const rdmm_spgemm_term* terms,
                  int nterms, uint32_t* c_row_ptr, rdmm_spgemm_plan** out,
                  uint64_t* c_nnz, uint64_t* flops, cudaStream_t s) {
  // the symbolic pass counts toward the SpGEMM kernel time too (VERDICT r1:
  // the roofline time of a product must include both passes)
  KernelTimer timer(s, 2);
  auto* P = new rdmm_spgemm_plan();
  std::unique_ptr<rdmm_spgemm_plan> guard(P);
  P->dtype = sizeof(T);
  P->rows = rows;
  P->ncols = ncols;
  P->nterms = nterms;
  P->c_row_ptr = c_row_ptr;
  std::vector<TermDev<T>> th(nterms > 0 ? nterms : 1);
  bool ident_only = true;
  for (int t = 0; t < nterms; ++t) {
    th[t].arp = terms[t].a_row_ptr;
    th[t].aci = terms[t].a_col_idx;
    th[t].av = static_cast<const T*>(terms[t].a_val);
    th[t].brp = terms[t].b_row_ptr;
    th[t].bci = terms[t].b_col_idx;
    th[t].bv = static_cast<const T*>(terms[t].b_val);
    if (th[t].arp) ident_only = false;
    if (!th[t].brp)
      return fail(RDMM_ERR_INVALID, "spgemm: term without a B operand");
  }
  P->ident_only = ident_only;
  RDMM_CUDA_TRY(P->terms.ensure(sizeof(TermDev<T>) * th.size(), s));
  RDMM_CUDA_TRY(cudaMemcpyAsync(P->terms.p, th.data(),
                                sizeof(TermDev<T>) * th.size(),
                                cudaMemcpyHostToDevice, s));
  RDMM_CUDA_TRY(P->cnt64.ensure(sizeof(uint64_t) * (size_t(rows) + 1), s));
  RDMM_CUDA_TRY(P->pre64.ensure(sizeof(uint64_t) * (size_t(rows) + 1), s));
  RDMM_CUDA_TRY(P->lists.ensure(sizeof(uint32_t) * size_t(kTiers) * (rows ? rows : 1), s));
  const size_t tc_bytes = sizeof(uint32_t) * 2 * kTiers + 8 * size_t(nterms) + 16;
  RDMM_CUDA_TRY(P->tcount.ensure(tc_bytes, s));
  RDMM_CUDA_TRY(cudaMemsetAsync(P->tcount.p, 0, tc_bytes, s));
  RDMM_CUDA_TRY(cudaMemsetAsync(P->cnt64.p, 0, sizeof(uint64_t) * (size_t(rows) + 1), s));
  uint32_t* tc = P->tcount.as<uint32_t>();
  auto* tub = reinterpret_cast<unsigned long long*>(tc + 2 * kTiers);
  const TermDev<T>* td = P->terms.as<TermDev<T>>();
  uint64_t* cnt = P->cnt64.as<uint64_t>();
  uint32_t* lists = P->lists.as<uint32_t>();
  if (rows && nterms) {
    const unsigned blocks = unsigned(std::min<uint64_t>(
        ceil_div(rows, 8), uint64_t(num_sms()) * 16));
    count_launch();
    k_bin_sym<T><<<blocks, 256, 8 * size_t(nterms), s>>>(rows, td, nterms, lists,
                                                         tc, tub, cnt);
    RDMM_CUDA_TRY(cudaGetLastError());
  }
  std::vector<uint32_t> hcv(2 * kTiers + 2 * size_t(nterms) + 4);
  uint32_t* hc = hcv.data();
  RDMM_CUDA_TRY(cudaMemcpyAsync(hc, tc, tc_bytes - 16 + 8, cudaMemcpyDeviceToHost, s));
  RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  for (int i = 0; i < kTiers; ++i) P->sym_count[i] = hc[i];
  P->term_flops.assign(nterms, 0);
  P->flops = 0;
  for (int t = 0; t < nterms; ++t) {
    uint64_t v;
    std::memcpy(&v, hc + 2 * kTiers + 2 * t, 8);
    P->term_flops[t] = 2 * v;
    P->flops += 2 * v;
  }
  auto L = [&](int tier) { return lists + size_t(tier) * rows; };
  int rc = 0;
  rc |= launch_sym_hash<T, 64, 32>(L(0), hc[0], td, nterms, cnt, s);
  rc |= launch_sym_hash<T, 512, 128>(L(1), hc[1], td, nterms, cnt, s);
  rc |= launch_sym_hash<T, 2048, 256>(L(2), hc[2], td, nterms, cnt, s);
  rc |= launch_sym_hash<T, 8192, 512>(L(3), hc[3], td, nterms, cnt, s);
  rc |= launch_sym_hash<T, 32768, 1024>(L(4), hc[4], td, nterms, cnt, s);
  if (rc) return rc;
  const uint32_t nwords = uint32_t(ceil_div(ncols, 32));
  if (hc[5]) {
    const uint32_t blocks = dense_rows_in_flight(hc[5], 1);
    if (size_t(nwords) * 4 <= kSymSmemMax) {
      auto fn = k_dense_sym_smem<T>;
      RDMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(nwords * 4)));
      count_launch();
      fn<<<blocks, kDenseThreads, nwords * 4, s>>>(L(5), hc[5], td, nterms, cnt, nwords);
    } else {
      RDMM_CUDA_TRY(P->bitmaps.ensure(size_t(blocks) * nwords * 4, s));
      RDMM_CUDA_TRY(cudaMemsetAsync(P->bitmaps.p, 0, size_t(blocks) * nwords * 4, s));
      count_launch();
      k_dense_sym_global<T><<<blocks, kDenseThreads, 0, s>>>(
          L(5), hc[5], td, nterms, cnt, P->bitmaps.as<uint32_t>(), nwords);
    }
  }
  RDMM_CUDA_TRY(cudaGetLastError());
  // row_ptr = exclusive scan of the counts (64-bit, checked against uint32)
  size_t tb = 0;
  RDMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, P->pre64.as<uint64_t>(),
                                              int64_t(rows) + 1, s));
  RDMM_CUDA_TRY(P->scan_tmp.ensure(tb, s));
  RDMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(P->scan_tmp.p, tb, cnt,
                                              P->pre64.as<uint64_t>(),
                                              int64_t(rows) + 1, s));
  uint64_t total = 0;
  RDMM_CUDA_TRY(cudaMemcpyAsync(&total, P->pre64.as<uint64_t>() + rows, 8,
                                cudaMemcpyDeviceToHost, s));
  if (rows) {
    const unsigned nb = unsigned(std::min<uint64_t>(ceil_div(rows + 1, 256),
                                                    uint64_t(num_sms()) * 8));
    count_launch();
    k_bin_num<<<nb, 256, 0, s>>>(rows, cnt, lists, tc + kTiers);
  }
  if (c_row_ptr) {
    const unsigned nb = unsigned(std::min<uint64_t>(ceil_div(rows + 1, 256),
                                                    uint64_t(num_sms()) * 8));
    count_launch();
    k_rowptr32<<<nb, 256, 0, s>>>(P->pre64.as<uint64_t>(), rows + 1, c_row_ptr);
  }
  RDMM_CUDA_TRY(cudaMemcpyAsync(hc, tc, sizeof(uint32_t) * 2 * kTiers,
                                cudaMemcpyDeviceToHost, s));
  RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  if (total >= (1ull << 32))
    return fail(RDMM_ERR_INVALID,
                "spgemm: output nnz exceeds the uint32 index_t range");
  for (int i = 0; i < kTiers; ++i) P->num_count[i] = hc[kTiers + i];
  P->nnz = total;
  if (c_nnz) *c_nnz = total;
  if (flops) *flops = P->flops;
  *out = guard.release();
  return RDMM_OK;
}

template <typename T>
int numeric_impl(rdmm_spgemm_plan* P, uint32_t* cci, T* cv, cudaStream_t s) {
  if (P->nnz == 0) return RDMM_OK;
  if (!P->c_row_ptr)
    return fail(RDMM_ERR_INVALID, "spgemm numeric: plan has no row_ptr");
  const TermDev<T>* td = P->terms.as<TermDev<T>>();
  const int nt = P->nterms;
  uint32_t* lists = P->lists.as<uint32_t>();
  const uint32_t rows = P->rows;
  auto L = [&](int tier) { return lists + size_t(tier) * rows; };
  // -0.0 is the exact additive identity (keeps signed zeros of csr_add);
  // products start from +0.0 like the reference accumulator (tile.hpp:232).
  const T ident = P->ident_only ? T(-0.0) : T(0);
  KernelTimer timer(s, 2);
  const uint32_t* crp = P->c_row_ptr;
  const uint32_t* c = P->num_count;
  // bits that cover every column index plus one, so the empty key
  // (0xFFFFFFFF) still sorts last once truncated to them
  int key_bits = 1;
  while (key_bits < 32 && (uint64_t(1) << key_bits) <= P->ncols) ++key_bits;
  // the dense tier (few SMs, L2-resident arrays) runs on a side stream beside
  // the hash tiers; rows of different tiers are disjoint
  cudaStream_t main_s = s;
  cudaStream_t ds = s;
  cudaEvent_t fork = nullptr, join = nullptr;
  if (c[5]) {
    ds = side_stream();
    RDMM_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    RDMM_CUDA_TRY(cudaEventRecord(fork, main_s));
    RDMM_CUDA_TRY(cudaStreamWaitEvent(ds, fork, 0));
  }
  int rc = 0;
  rc |= launch_num_hash<T, 64, 32>(L(0), c[0], td, nt, crp, cci, cv, ident, key_bits, s);
  rc |= launch_num_hash<T, 512, 128>(L(1), c[1], td, nt, crp, cci, cv, ident, key_bits, s);
  rc |= launch_num_hash<T, 2048, 256>(L(2), c[2], td, nt, crp, cci, cv, ident, key_bits, s);
  rc |= launch_num_hash<T, 8192, 512>(L(3), c[3], td, nt, crp, cci, cv, ident, key_bits, s);
  rc |= launch_num_hash<T, 16384, 1024>(L(4), c[4], td, nt, crp, cci, cv, ident, key_bits, s);
  if (rc) return rc;
  if (c[5]) {
    const uint32_t nwords = uint32_t(ceil_div(P->ncols, 32));
    const int cl = dense_cl();
    const uint32_t blocks = dense_num_slots(c[5], size_t(P->ncols) * sizeof(T), cl);
    s = ds;
    RDMM_CUDA_TRY(P->bitmaps.ensure(size_t(blocks) * nwords * 4, main_s));
    RDMM_CUDA_TRY(P->dense.ensure(size_t(blocks) * P->ncols * sizeof(T), main_s));
    RDMM_CUDA_TRY(cudaEventRecord(fork, main_s));  // the buffers exist
    RDMM_CUDA_TRY(cudaStreamWaitEvent(s, fork, 0));
    RDMM_CUDA_TRY(cudaMemsetAsync(P->bitmaps.p, 0, size_t(blocks) * nwords * 4, s));
    const size_t nd = size_t(blocks) * P->ncols;
    count_launch();
    k_fill<T><<<unsigned(std::min<uint64_t>(ceil_div(nd, 256), 4096)), 256, 0, s>>>(
        P->dense.as<T>(), nd, ident);
    auto* bm = P->bitmaps.as<uint32_t>();
    T* dn = P->dense.as<T>();
    int rc2 = 0;
    switch (cl) {
      case 8: rc2 = launch_dense_num<T, 8>(blocks, L(5), c[5], td, nt, crp, cci, cv, bm, dn, nwords, P->ncols, ident, s); break;
      case 4: rc2 = launch_dense_num<T, 4>(blocks, L(5), c[5], td, nt, crp, cci, cv, bm, dn, nwords, P->ncols, ident, s); break;
      case 2: rc2 = launch_dense_num<T, 2>(blocks, L(5), c[5], td, nt, crp, cci, cv, bm, dn, nwords, P->ncols, ident, s); break;
      default: rc2 = launch_dense_num<T, 1>(blocks, L(5), c[5], td, nt, crp, cci, cv, bm, dn, nwords, P->ncols, ident, s);
    }
    if (rc2) return rc2;
    RDMM_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    RDMM_CUDA_TRY(cudaEventRecord(join, ds));
    RDMM_CUDA_TRY(cudaStreamWaitEvent(main_s, join, 0));
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
  }
  RDMM_CUDA_TRY(cudaGetLastError());
  return RDMM_OK;
}

// Deterministic numeric pass (see k_det_expand): rows in batches of at most
// kDetBatch products, each expanded, stably sorted and folded.
constexpr uint64_t kDetBatch = uint64_t(1) << 26;

template <typename T>
int numeric_det_impl(rdmm_spgemm_plan* P, uint32_t* cci, T* cv, cudaStream_t s) {
  if (P->nnz == 0) return RDMM_OK;
  if (!P->c_row_ptr)
    return fail(RDMM_ERR_INVALID, "spgemm numeric: plan has no row_ptr");
  if (P->nterms > 255) return fail(RDMM_ERR_INVALID, "spgemm deterministic: at most 255 terms");
  KernelTimer timer(s, 2);
  const TermDev<T>* td = P->terms.as<TermDev<T>>();
  const uint32_t rows = P->rows;
  // products per row -> host prefix (batch boundaries)
  uint64_t* cnt = nullptr;
  RDMM_CUDA_TRY(cudaMallocAsync(&cnt, (size_t(rows) + 1) * 8, s));
  const unsigned nb = unsigned(std::min<uint64_t>(ceil_div(uint64_t(rows) * 32, 256),
                                                  uint64_t(num_sms()) * 16));
  count_launch();
  k_det_count<T><<<std::max(1u, nb), 256, 0, s>>>(0, rows, td, P->nterms, cnt);
  std::vector<uint64_t> hc(rows);
  RDMM_CUDA_TRY(cudaMemcpyAsync(hc.data(), cnt, size_t(rows) * 8, cudaMemcpyDeviceToHost, s));
  std::vector<uint32_t> rp(size_t(rows) + 1);
  RDMM_CUDA_TRY(cudaMemcpyAsync(rp.data(), P->c_row_ptr, (size_t(rows) + 1) * 4,
                                cudaMemcpyDeviceToHost, s));
  RDMM_CUDA_TRY(cudaStreamSynchronize(s));
  uint64_t maxb = 0;
  for (uint64_t x : hc) maxb = std::max(maxb, x);
  const uint64_t cap = std::max<uint64_t>(std::min<uint64_t>(kDetBatch, std::accumulate(
                                              hc.begin(), hc.end(), uint64_t(0))), maxb);
  uint64_t *keys = nullptr, *keys2 = nullptr, *off = nullptr;
  AB<T>*ab = nullptr, *ab2 = nullptr;
  uint32_t *head = nullptr, *hpos = nullptr;
  RDMM_CUDA_TRY(cudaMallocAsync(&keys, cap * 8, s));
  RDMM_CUDA_TRY(cudaMallocAsync(&keys2, cap * 8, s));
  RDMM_CUDA_TRY(cudaMallocAsync(&ab, cap * sizeof(AB<T>), s));
  RDMM_CUDA_TRY(cudaMallocAsync(&ab2, cap * sizeof(AB<T>), s));
  RDMM_CUDA_TRY(cudaMallocAsync(&head, cap * 4, s));
  RDMM_CUDA_TRY(cudaMallocAsync(&hpos, cap * 4, s));
  RDMM_CUDA_TRY(cudaMallocAsync(&off, (size_t(rows) + 1) * 8, s));
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, keys, keys2, ab, ab2, int64_t(cap), 0, 64, s);
    cub::DeviceScan::ExclusiveSum(nullptr, b, head, hpos, int64_t(cap), s);
    tmp_bytes = std::max(a, b);
  }
  RDMM_CUDA_TRY(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), s));
  int key_bits = 8;
  while (key_bits < 40 && (uint64_t(1) << (key_bits - 8)) < uint64_t(P->ncols)) ++key_bits;
  int rc = RDMM_OK;
  for (uint32_t r0 = 0; r0 < rows && rc == RDMM_OK;) {
    uint32_t r1 = r0;
    uint64_t n = 0;
    std::vector<uint64_t> ho;
    while (r1 < rows && (r1 == r0 || n + hc[r1] <= cap) && r1 - r0 < (1u << 23)) {
      ho.push_back(n);
      n += hc[r1++];
    }
    ho.push_back(n);
    if (n) {
      RDMM_CUDA_TRY(cudaMemcpyAsync(off, ho.data(), ho.size() * 8, cudaMemcpyHostToDevice, s));
      const uint32_t br = r1 - r0;
      const unsigned eb = unsigned(std::min<uint64_t>(ceil_div(uint64_t(br) * 32, 256),
                                                      uint64_t(num_sms()) * 16));
      count_launch(4);
      k_det_expand<T><<<std::max(1u, eb), 256, 0, s>>>(r0, br, td, P->nterms, off, keys, ab);
      // row bits above the column and term bits
      int rbits = 1;
      while (rbits < 24 && (uint64_t(1) << rbits) < br) ++rbits;
      size_t tb = tmp_bytes;
      RDMM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, ab, ab2, int64_t(n), 0,
                                                    40 + rbits, s));
      const unsigned fb = unsigned(std::min<uint64_t>(ceil_div(n, 256), uint64_t(num_sms()) * 16));
      k_det_heads<<<fb, 256, 0, s>>>(keys2, n, head);
      tb = tmp_bytes;
      RDMM_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, head, hpos, int64_t(n), s));
      k_det_fold<T><<<fb, 256, 0, s>>>(keys2, ab2, n, head, hpos, td, rp[r0], cci, cv);
      RDMM_CUDA_TRY(cudaGetLastError());
      (void)key_bits;
    }
    RDMM_CUDA_TRY(cudaStreamSynchronize(s));  // `ho` / offsets reused next batch
    r0 = r1;
  }
  for (void* p : {static_cast<void*>(cnt), static_cast<void*>(keys), static_cast<void*>(keys2),
                  static_cast<void*>(ab), static_cast<void*>(ab2), static_cast<void*>(head),
                  static_cast<void*>(hpos), static_cast<void*>(off), tmp})
    cudaFreeAsync(p, s);
  RDMM_CUDA_TRY(cudaGetLastError());
  return rc;
}

}  // namespace

extern "C" int rdmm_spgemm_symbolic(uint32_t rows, uint32_t ncols,
                                    int dtype_bytes,
                                    const rdmm_spgemm_term* terms, int nterms,
                                    uint32_t* c_row_ptr,
                                    rdmm_spgemm_plan** plan, uint64_t* c_nnz,
                                    uint64_t* flops, rdmm_stream_t stream) {
  if (!plan) return fail(RDMM_ERR_INVALID, "spgemm: null plan pointer");
  *plan = nullptr;
  if (nterms < 0 || (nterms > 0 && !terms))
    return fail(RDMM_ERR_INVALID, "spgemm: bad term list");
  return dtype_bytes == 8
             ? symbolic_impl<double>(rows, ncols, terms, nterms, c_row_ptr,
                                     plan, c_nnz, flops, as_stream(stream))
             : symbolic_impl<float>(rows, ncols, terms, nterms, c_row_ptr,
                                    plan, c_nnz, flops, as_stream(stream));
}

extern "C" int rdmm_spgemm_numeric(rdmm_spgemm_plan* plan, uint32_t* c_col_idx,
                                   void* c_val, rdmm_stream_t stream) {
  if (!plan) return fail(RDMM_ERR_INVALID, "spgemm: null plan");
  return plan->dtype == 8
             ? numeric_impl<double>(plan, c_col_idx, static_cast<double*>(c_val),
                                    as_stream(stream))
             : numeric_impl<float>(plan, c_col_idx, static_cast<float*>(c_val),
                                   as_stream(stream));
}

extern "C" int rdmm_spgemm_numeric_ex(rdmm_spgemm_plan* plan, uint32_t* c_col_idx,
                                      void* c_val, unsigned flags, rdmm_stream_t stream) {
  if (!plan) return fail(RDMM_ERR_INVALID, "spgemm: null plan");
  if (!(flags & RDMM_SPGEMM_DETERMINISTIC))
    return rdmm_spgemm_numeric(plan, c_col_idx, c_val, stream);
  return plan->dtype == 8
             ? numeric_det_impl<double>(plan, c_col_idx, static_cast<double*>(c_val),
                                        as_stream(stream))
             : numeric_det_impl<float>(plan, c_col_idx, static_cast<float*>(c_val),
                                       as_stream(stream));
}

extern "C" void rdmm_spgemm_plan_destroy(rdmm_spgemm_plan* plan) { delete plan; }

extern "C" int rdmm_spgemm_plan_term_flops(const rdmm_spgemm_plan* plan,
                                           uint64_t* out) {
  if (!plan) return fail(RDMM_ERR_INVALID, "spgemm: null plan");
  for (size_t t = 0; t < plan->term_flops.size(); ++t) out[t] = plan->term_flops[t];
  return RDMM_OK;
}

extern "C" int rdmm_spgemm_plan_info(const rdmm_spgemm_plan* plan,
                                     uint32_t* sym_tiers, uint32_t* num_tiers) {
  if (!plan) return fail(RDMM_ERR_INVALID, "spgemm: null plan");
  for (int i = 0; i < kTiers; ++i) {
    if (sym_tiers) sym_tiers[i] = plan->sym_count[i];
    if (num_tiers) num_tiers[i] = plan->num_count[i];
  }
  return RDMM_OK;
}
