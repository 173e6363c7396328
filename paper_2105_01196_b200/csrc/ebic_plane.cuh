// ebic_plane.cuh -- rank-plane encoding + shared-memory row-slab fitness kernel.
//
// RANK PLANE (built once per resident matrix and approx value)
//   For row r with values v_0..v_{C-1} (the store, f32 or f64) and the reference
//   threshold thr(x) = RN64(x - RN64(approx*|x|))  (trend.cpp:22,33):
//     R(r,c) = 1 + #{c' : v_c' <  v_c}                (strict rank, 1..C)
//     T(r,c) =     #{c' : v_c' <= thr(v_c)}           (threshold rank, 0..C)
//   For two values of the same row:  v_y > thr(v_x)  <=>  R(y) > T(x).
//     (if v_y > thr: every value <= thr is < v_y, so R(y)-1 >= T(x);
//      if v_y <= thr: v_y itself is counted by T(x) but not by R(y)-1, and every
//      value < v_y is <= thr, so R(y)-1 <= T(x)-1.)
//   The plane word is W = R << 16 | T (C <= 65535).  With key(W) = W << 16 | 0xFFFF
//   (mod 2^32 = T << 16 | 0xFFFF):   W_y > key(W_x)  <=>  R(y) > T(x).
//   So every consecutive-pair test of row_supports (trend.cpp:17-37), forward
//   v[k] > thr(v[k-1]) and reversed v[k-1] > thr(v[k]), is ONE unsigned integer
//   compare, exact by construction: all floating point happens in the builder,
//   in double, with the reference's two rounded operations.
//
// SLAB KERNEL (the hot path)
//   A CTA stages a tile of RT consecutive rows x ALL columns of the plane in
//   shared memory ([C][RT] words, column-major like the store), then its warps
//   sweep candidates over it: lanes own rows, each candidate column is one
//   conflict-free LDS per lane, each pair one IMAD + one ISETP, and the rows
//   supporting a candidate are counted with __ballot_sync + __popc into a
//   per-CTA shared-memory count (one owner warp per candidate, no atomics);
//   counts are flushed to global with one atomicAdd per (CTA, candidate chunk).
//   Candidates are packed into 16-byte records (7 x u16 columns + u16 length)
//   in shared memory once per chunk; longer candidates continue from the CSR.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ebic_kernels.cuh"

namespace ebic {

constexpr int kSlabWarps = 32;
constexpr int kSlabThreads = kSlabWarps * 32;
constexpr int kRecCols = 7;          // columns held in a candidate record
constexpr uint32_t kPlaneMaxCols = 8192;

__device__ __forceinline__ uint32_t plane_key(uint32_t w) { return (w << 16) | 0xFFFFu; }

// ---------------------------------------------------------------------------
// plane builder: one CTA per row (grid-stride); bitonic sort of the row in
// shared memory, then two binary searches per element.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
build_plane_kernel(const T* __restrict__ store, uint64_t ld, uint32_t n_rows, uint32_t n_cols,
                   uint32_t pow2, double approx, uint32_t* __restrict__ plane) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);
  for (uint32_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
    for (uint32_t j = threadIdx.x; j < pow2; j += blockDim.x)
      s[j] = j < n_cols ? store[(uint64_t)j * ld + row] : (T)INFINITY;
    __syncthreads();
    // bitonic sort, ascending
    for (uint32_t k = 2; k <= pow2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = threadIdx.x; i < pow2; i += blockDim.x) {
          const uint32_t p = i ^ j;
          if (p > i) {
            const T a = s[i], b = s[p];
            const bool up = (i & k) == 0;
            if ((a > b) == up) {
              s[i] = b;
              s[p] = a;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t c = threadIdx.x; c < n_cols; c += blockDim.x) {
      const T v = store[(uint64_t)c * ld + row];
      // lower_bound: #values < v
      uint32_t lo = 0, hi = n_cols;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s[mid] < v) lo = mid + 1; else hi = mid;
      }
      const uint32_t rank1 = lo + 1;
      // upper_bound of the reference threshold (double): #values <= thr(v)
      const double t = thr64((double)v, approx);
      lo = 0;
      hi = n_cols;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((double)s[mid] <= t) lo = mid + 1; else hi = mid;
      }
      plane[(uint64_t)c * ld + row] = (rank1 << 16) | lo;
    }
    __syncthreads();
  }
}

template <int RPL> struct LdsVec;
template <> struct LdsVec<1> { using V = uint32_t; };
template <> struct LdsVec<2> { using V = uint2; };
template <> struct LdsVec<4> { using V = uint4; };
__device__ __forceinline__ uint32_t vel(const uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t vel(const uint2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ uint32_t vel(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// explicit shared-space loads on 32-bit shared addresses (no generic->shared
// conversion inside the candidate loop)
__device__ __forceinline__ uint32_t lds_v(uint32_t addr, uint32_t*) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds_v(uint32_t addr, uint2*) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds_v(uint32_t addr, uint4*) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
template <typename V> __device__ __forceinline__ V lds(uint32_t addr) { return lds_v(addr, (V*)nullptr); }

struct SlabArgs {
  const uint32_t* plane;
  uint64_t ld;
  uint32_t n_rows, n_cols;
  const uint32_t* cols;   // CSR population (device)
  const uint32_t* offs;
  uint32_t n_cand;
  uint32_t chunk;         // candidates per chunk (records staged in SMEM)
  uint32_t n_chunks;
  uint32_t n_slabs;
  uint32_t* counts;
  uint32_t* mask;         // MASK: [cand][ld/32] words
  uint64_t mask_wpc;
  int* err;
  int prefetch;           // warm L2 with the next unit's slab (plane larger than L2)
  uint32_t group;         // slab_pair_kernel: CTAs per chunk group (see the kernel)
  uint32_t* out;          // slab_pair_kernel: final counts (written, not added; device-accessible)
  uint32_t* done;         // slab_pair_kernel: [n_chunks + 1] arrival counters, zero between launches
  int* err_out;           // slab_pair_kernel: where the device error flag is forwarded (== err: kept)
};

// One consecutive-pair test on RPL rows: forward needs c > thr(p), reversed p > thr(c).
template <int RPL, bool NEG, typename V>
__device__ __forceinline__ void pair_test(const V& wp, const V& wc, uint32_t& okf, uint32_t& okr) {
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const uint32_t p = vel(wp, r), c = vel(wc, r);
    if (!(c > plane_key(p))) okf &= ~(1u << r);
    if (NEG && !(p > plane_key(c))) okr &= ~(1u << r);
  }
}

// Fixed-length body: all L loads issued first (ILP), then the L-1 pair tests.
// Returns the RPL support bits of this lane's rows (before validity masking).
// u16 halves of a record word, one PRMT each
__device__ __forceinline__ uint32_t lo16(uint32_t x) { return __byte_perm(x, 0u, 0x4410); }
__device__ __forceinline__ uint32_t hi16(uint32_t x) { return __byte_perm(x, 0u, 0x4432); }

template <int L, int RPL, bool NEG, uint32_t COLSHIFT>
__device__ __forceinline__ uint32_t eval_fixed(uint32_t lane_base, const uint4& rec) {
  using V = typename LdsVec<RPL>::V;
  const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                 hi16(rec.z), lo16(rec.w), hi16(rec.w)};
  V w[L];
#pragma unroll
  for (int k = 0; k < L; ++k) w[k] = lds<V>(lane_base + (cc[k] << COLSHIFT));
  if constexpr (RPL == 1) {
    bool f = true, r = NEG;
#pragma unroll
    for (int k = 1; k < L; ++k) {
      f = f && (w[k] > plane_key(w[k - 1]));
      if (NEG) r = r && (w[k - 1] > plane_key(w[k]));
    }
    return (f || r) ? 1u : 0u;
  } else {
    uint32_t okf = (1u << RPL) - 1u, okr = NEG ? okf : 0u;
#pragma unroll
    for (int k = 1; k < L; ++k) pair_test<RPL, NEG>(w[k - 1], w[k], okf, okr);
    return okf | okr;
  }
}

// ---------------------------------------------------------------------------
// plane builder, row-tile version (the default): a CTA owns RG consecutive rows
// (one warp per row).  The tile is read from the column-major store with RG
// consecutive rows per column -- one full 32-B sector per column at RG = 8, f32
// (a warp reading a single row would touch one sector per ELEMENT) -- sorted
// per row with a warp-level bitonic network in shared memory (__syncwarp only),
// searched exactly like build_plane_kernel, and written back the same way.
// ---------------------------------------------------------------------------
// Order-preserving unsigned image of a float (sort key) and back.
__device__ __forceinline__ uint32_t f2key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// Warp bitonic sort of 32*E keys held E per lane (element g = lane*E + j):
// in-lane stages on registers, cross-lane stages with __shfl_xor_sync.
template <int E>
__device__ __forceinline__ void warp_register_sort(uint32_t (&k)[E], int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32 * E; kk <<= 1) {
#pragma unroll
    for (int d = kk >> 1; d > 0; d >>= 1) {
      if (d < E) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          if ((j & d) == 0) {
            const bool up = ((lane * E + j) & kk) == 0;
            const uint32_t a = k[j], b = k[j ^ d];
            k[j] = up ? min(a, b) : max(a, b);
            k[j ^ d] = up ? max(a, b) : min(a, b);
          }
        }
      } else {
        const int lx = d / E;
        const bool lower = (lane & lx) == 0;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const bool up = ((lane * E + j) & kk) == 0;
          const uint32_t o = __shfl_xor_sync(kFull, k[j], lx);
          k[j] = (lower == up) ? min(k[j], o) : max(k[j], o);
        }
      }
    }
  }
}

// E == 0: warp-level shared-memory bitonic sort (any C, f32 or f64);
// E > 0 : float32 rows with C <= 32*E sorted in registers (warp_register_sort).
template <typename T, int E>
__global__ void __launch_bounds__(256)
build_plane_tile_kernel(const T* __restrict__ store, uint64_t ld, uint32_t n_rows, uint32_t n_cols,
                        uint32_t pow2, uint32_t rg, double approx, uint32_t* __restrict__ plane) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t cp = n_cols + 1;                              // padded tile row (bank spread)
  T* s_val = reinterpret_cast<T*>(smem_raw);                   // [rg][cp] values, then plane words
  T* s_srt = s_val + (size_t)rg * cp;                          // [rg][pow2] sorted values
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_groups = (n_rows + rg - 1) / rg;
  for (uint32_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const uint32_t row0 = grp * rg;
    // 1. tile load: consecutive threads read consecutive rows of a column
    for (uint32_t t = threadIdx.x; t < rg * n_cols; t += blockDim.x) {
      const uint32_t c = t / rg, r = t % rg;
      s_val[r * cp + c] = row0 + r < n_rows ? store[(uint64_t)c * ld + row0 + r] : (T)0;
    }
    __syncthreads();
    for (uint32_t w = warp; w < rg; w += blockDim.x / 32) {
      T* v = s_val + (size_t)w * cp;
      T* srt = s_srt + (size_t)w * pow2;
      // 2. sort the row (ascending, padding +inf) into srt
      if constexpr (E > 0) {
        uint32_t key[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint32_t c = lane * E + j;
          key[j] = c < n_cols ? f2key((float)v[c]) : 0xFFFFFFFFu;
        }
        warp_register_sort<E>(key, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const uint32_t c = lane * E + j;
          if (c < n_cols) srt[c] = (T)key2f(key[j]);
        }
        __syncwarp();
      } else {
        for (uint32_t j = lane; j < pow2; j += 32) srt[j] = j < n_cols ? v[j] : (T)INFINITY;
        __syncwarp();
        for (uint32_t k = 2; k <= pow2; k <<= 1) {
          for (uint32_t d = k >> 1; d > 0; d >>= 1) {
            for (uint32_t i = lane; i < pow2 / 2; i += 32) {
              const uint32_t a = ((i & ~(d - 1)) << 1) | (i & (d - 1));  // lower index of the i-th pair
              const uint32_t b = a | d;
              const T x = srt[a], y = srt[b];
              if ((x > y) == ((a & k) == 0)) {
                srt[a] = y;
                srt[b] = x;
              }
            }
            __syncwarp();
          }
        }
      }
      // 3. exact ranks: R = 1 + lower_bound(v), T = upper_bound(thr64(v))
      for (uint32_t c = lane; c < n_cols; c += 32) {
        const T x = v[c];
        uint32_t lo = 0, hi = n_cols;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (srt[mid] < x) lo = mid + 1; else hi = mid;
        }
        const uint32_t rank1 = lo + 1;
        const double t = thr64((double)x, approx);
        lo = 0;
        hi = n_cols;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if ((double)srt[mid] <= t) lo = mid + 1; else hi = mid;
        }
        // the plane word replaces the value in place (low 32 bits of the element;
        // each element is read, then overwritten, by the same lane)
        *reinterpret_cast<uint32_t*>(&v[c]) = (rank1 << 16) | lo;
      }
    }
    __syncthreads();
    // 4. coalesced write-back of the plane words
    for (uint32_t t = threadIdx.x; t < rg * n_cols; t += blockDim.x) {
      const uint32_t c = t / rg, r = t % rg;
      if (row0 + r < n_rows)
        plane[(uint64_t)c * ld + row0 + r] = *reinterpret_cast<const uint32_t*>(&s_val[(size_t)r * cp + c]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// slab kernel
//   RPL : consecutive rows per lane (1, 2, 4)   -> LDS.32 / .64 / .128
//   SUB : candidates per warp (1, 2, 4)          -> 32/SUB lanes per candidate
//   RT  = (32 / SUB) * RPL rows per slab
// work unit = (candidate chunk, row slab), linearised chunk-major; CTA b owns
// units [b*U/G, (b+1)*U/G).
// ---------------------------------------------------------------------------
// Per-length record classes: class L (2..7) holds candidates of exactly L
// columns, class 1 length-1 candidates, class 8 everything longer (first 7
// columns in the record, the tail read from the CSR).  Sorting a chunk's
// records by class once lets the sweep run a branch-free, fully unrolled body
// per class instead of dispatching on the length of every candidate.
constexpr int kClasses = 9;  // 0 (invalid) .. 8

template <int RPL, int SUB, bool NEG, bool MASK, int L, uint32_t COLSHIFT>
__device__ __forceinline__ void sweep_class(const SlabArgs& a, uint32_t sa_rec, uint32_t lane_base, uint32_t* s_cnt,
                                            uint32_t n_padded, uint32_t class_base, uint32_t c_begin,
                                            uint32_t row0, uint32_t vmask, int warp, int lane, int sub, int rl) {
  // Each class list is padded to a multiple of the sweep stride with dummy
  // records (candidate slot `chunk`, a scratch count), so every (warp, sub)
  // slot has a record on every iteration: no bounds checks in the loop.
  constexpr int LPC = 32 / SUB;
  using V = typename LdsVec<RPL>::V;
  constexpr uint32_t stride = kSlabWarps * SUB;
  for (uint32_t t = warp * SUB + sub; t < n_padded; t += stride) {
    const uint4 rec = lds<uint4>(sa_rec + (class_base + t) * 16);
    const uint32_t j = lo16(rec.x);
    uint32_t ok;
    if constexpr (L == 1) {
      ok = vmask;  // no pair: every row supports (the trend.cpp:19 loop never runs)
    } else if constexpr (L < 8) {
      ok = eval_fixed<L, RPL, NEG, COLSHIFT>(lane_base, rec) & vmask;
    } else {
      // >= 8 columns: the first 7 from the record, the tail from the CSR
      uint32_t okf = vmask, okr = NEG ? vmask : 0u;
      const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                     hi16(rec.z), lo16(rec.w), hi16(rec.w)};
      V wp = lds<V>(lane_base + (cc[0] << COLSHIFT));
#pragma unroll
      for (int k = 1; k < kRecCols; ++k) {
        const V wc = lds<V>(lane_base + (cc[k] << COLSHIFT));
        pair_test<RPL, NEG>(wp, wc, okf, okr);
        wp = wc;
      }
      if (j < a.chunk) {
        // the tail in blocks of TB columns (independent index loads, then shared loads)
        constexpr int TB = RPL == 1 ? 8 : RPL == 2 ? 4 : 2;  // register budget: 64 per thread
        const uint32_t b = a.offs[c_begin + j], e = a.offs[c_begin + j + 1];
        for (uint32_t k0 = b + kRecCols; k0 < e; k0 += TB) {
          if ((okf | okr) == 0u) break;  // this lane's rows are all decided
          uint32_t idx[TB];
#pragma unroll
          for (int i = 0; i < TB; ++i) idx[i] = k0 + i < e ? __ldg(a.cols + k0 + i) : 0u;
          V wv[TB];
#pragma unroll
          for (int i = 0; i < TB; ++i) wv[i] = lds<V>(lane_base + (idx[i] << COLSHIFT));
#pragma unroll
          for (int i = 0; i < TB; ++i) {
            if (k0 + i < e) {
              pair_test<RPL, NEG>(wp, wv[i], okf, okr);
              wp = wv[i];
            }
          }
        }
      }
      ok = okf | okr;
    }
    if constexpr (MASK) {
      static_assert(!MASK || (RPL == 1 && SUB == 1), "mask output needs one row per lane");
      const uint32_t word = __ballot_sync(kFull, ok & 1u);
      if (lane == 0 && j < a.chunk) {
        a.mask[(uint64_t)(c_begin + j) * a.mask_wpc + row0 / 32] = word;
        atomicAdd(&s_cnt[j], (uint32_t)__popc(word));
      }
    } else if constexpr (RPL == 1) {
      const uint32_t b = __ballot_sync(kFull, ok & 1u);
      const uint32_t n = SUB == 1 ? __popc(b) : __popc((b >> (sub * LPC)) & ((1u << LPC) - 1u));
      if (rl == 0) atomicAdd(&s_cnt[j], n);  // sole owner of candidate j in this CTA
    } else {
      static_assert(RPL == 1 || SUB == 1, "multi-row lanes use whole warps");
      const uint32_t n = __reduce_add_sync(kFull, (uint32_t)__popc(ok));
      if (lane == 0) atomicAdd(&s_cnt[j], n);
    }
  }
}

// Warm L2 with the plane rows of the CTA's NEXT work unit while the current one
// is swept (host policy in make_slab_args: only for L2-resident planes).
template <uint32_t RT>
__device__ __forceinline__ void prefetch_next_slab(const SlabArgs& a, uint64_t u_next, uint64_t u_end) {
  if (!a.prefetch || u_next >= u_end) return;
  const uint32_t row0 = (uint32_t)(u_next % a.n_slabs) * RT;
  constexpr uint32_t LINES = (RT * 4 + 127) / 128;
  for (uint32_t t = threadIdx.x; t < a.n_cols * LINES; t += blockDim.x) {
    const uint32_t c = t / LINES, l = t % LINES;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.plane + (uint64_t)c * a.ld + row0 + l * 32));
  }
}

// Pack one chunk of the CSR population into shared-memory records
// {u16 candidate slot, 7 x u16 columns}, sorted into length classes (counting
// sort) and each class padded to a multiple of STRIDE with dummy records
// (slot = chunk, all columns 0).  Zeroes the chunk's shared counts.  Invalid
// candidates (empty, or a column >= n_cols) raise the device error flag and
// land in class 0, which is never swept (count 0).  Called by every thread.
template <uint32_t STRIDE>
__device__ void pack_chunk(const SlabArgs& a, uint32_t c_begin, uint32_t c_n, uint4* s_rec, uint32_t* s_cnt,
                           uint32_t* s_hist, uint32_t* s_base, uint32_t* s_fill) {
  auto class_of = [&](uint32_t i, uint32_t& len, bool& bad) -> uint32_t {
    const uint32_t b = a.offs[i], e = a.offs[i + 1];
    len = e > b ? e - b : 0;
    bad = len == 0;
    for (uint32_t k = b; k < e && !bad; ++k) bad |= a.cols[k] >= a.n_cols;
    return bad ? 0u : min(len, 8u);
  };
  if (threadIdx.x < kClasses) s_hist[threadIdx.x] = 0;
  __syncthreads();
  // pass 1: class histogram (+ validation)
  for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
    uint32_t len;
    bool bad;
    const uint32_t cl = class_of(c_begin + j, len, bad);
    if (bad) atomicOr(a.err, 1);
    atomicAdd(&s_hist[cl], 1u);
    s_cnt[j] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int c = 0; c < kClasses; ++c) {
      s_base[c] = acc;
      s_fill[c] = 0;
      s_hist[c] = (s_hist[c] + STRIDE - 1) / STRIDE * STRIDE;
      acc += s_hist[c];
    }
    s_cnt[a.chunk] = 0;  // scratch count of the padding records
  }
  __syncthreads();
  for (int c = 1; c < kClasses; ++c)
    for (uint32_t t = threadIdx.x; t < s_hist[c]; t += blockDim.x) s_rec[s_base[c] + t] = make_uint4(a.chunk, 0u, 0u, 0u);
  __syncthreads();
  // pass 2: records scattered by class
  for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
    uint32_t len;
    bool bad;
    const uint32_t cl = class_of(c_begin + j, len, bad);
    const uint32_t b = a.offs[c_begin + j];
    const uint32_t pos = s_base[cl] + atomicAdd(&s_fill[cl], 1u);
    uint32_t h[8] = {j, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kRecCols; ++k)
      if (!bad && (uint32_t)k < len) h[k + 1] = a.cols[b + k];
    s_rec[pos] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
  }
}

template <int RPL, int SUB, bool NEG, bool MASK>
__global__ void __launch_bounds__(kSlabThreads, 1)
slab_count_kernel(const SlabArgs a) {
  constexpr int LPC = 32 / SUB;        // lanes per candidate
  constexpr uint32_t RT = LPC * RPL;   // rows per slab
  constexpr uint32_t COLSHIFT = RT == 8 ? 5 : RT == 16 ? 6 : RT == 32 ? 7 : RT == 64 ? 8 : 9;  // log2(RT*4)
  static_assert((4u * RT) == (1u << COLSHIFT), "RT must be a power of two");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(smem_raw);               // [C][RT]
  uint4* s_rec = reinterpret_cast<uint4*>(s_slab + (size_t)a.n_cols * RT);  // [chunk], sorted by class
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_rec + a.chunk + kClasses * kSlabWarps * SUB);  // [chunk+1]
  __shared__ uint32_t s_hist[kClasses], s_base[kClasses], s_fill[kClasses];
  const uint32_t sa_slab = (uint32_t)__cvta_generic_to_shared(s_slab);
  const uint32_t sa_rec = (uint32_t)__cvta_generic_to_shared(s_rec);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPC, rl = lane % LPC;
  const uint32_t lane_base = sa_slab + rl * RPL * 4;
  const uint64_t U = (uint64_t)a.n_chunks * a.n_slabs;
  const uint64_t u_begin = blockIdx.x * U / gridDim.x, u_end = (blockIdx.x + 1) * U / gridDim.x;

  uint32_t cur_chunk = 0xffffffffu, c_begin = 0, c_n = 0;

  auto flush = [&]() {
    if (cur_chunk == 0xffffffffu) return;
    for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x)
      if (s_cnt[j]) atomicAdd(&a.counts[c_begin + j], s_cnt[j]);
  };
  for (uint64_t u = u_begin; u < u_end; ++u) {
    const uint32_t chunk = (uint32_t)(u / a.n_slabs), slab = (uint32_t)(u % a.n_slabs);
    const uint32_t row0 = slab * RT;
    __syncthreads();  // previous slab / counts fully consumed
    if (chunk != cur_chunk) {
      flush();
      cur_chunk = chunk;
      c_begin = chunk * a.chunk;
      c_n = min(a.chunk, a.n_cand - c_begin);
      pack_chunk<kSlabWarps * SUB>(a, c_begin, c_n, s_rec, s_cnt, s_hist, s_base, s_fill);
    }
    // stage the slab: rows [row0, row0+RT) of every column (RT*4 bytes contiguous per column)
    {
      constexpr uint32_t V4 = RT / 4;  // uint4 per column
      constexpr int UNR = 4;           // all loads of a round in flight before any store
      const uint32_t total = a.n_cols * V4;
      const uint4* src = reinterpret_cast<const uint4*>(a.plane);
      uint4* dst = reinterpret_cast<uint4*>(s_slab);
      const uint64_t ld4 = a.ld / 4, r4 = row0 / 4;
      for (uint32_t t0 = threadIdx.x; t0 < total; t0 += UNR * blockDim.x) {
        uint4 w[UNR];
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t t = t0 + k * blockDim.x;
          if (t < total) w[k] = __ldg(src + (uint64_t)(t / V4) * ld4 + r4 + t % V4);
        }
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t t = t0 + k * blockDim.x;
          if (t < total) dst[t] = w[k];
        }
      }
    }
    __syncthreads();
    prefetch_next_slab<RT>(a, u + 1, u_end);

    const uint32_t valid_rows = min(RT, a.n_rows - row0);
    uint32_t vmask = 0;  // validity bits of this lane's RPL rows
#pragma unroll
    for (int j = 0; j < RPL; ++j) vmask |= (rl * RPL + j < valid_rows ? 1u : 0u) << j;

#define EBIC_SWEEP(L)                                                                                   \
  sweep_class<RPL, SUB, NEG, MASK, L, COLSHIFT>(a, sa_rec, lane_base, s_cnt, s_hist[L], s_base[L], c_begin, \
                                                row0, vmask, warp, lane, sub, rl)
    EBIC_SWEEP(4);
    EBIC_SWEEP(3);
    EBIC_SWEEP(5);
    EBIC_SWEEP(2);
    EBIC_SWEEP(6);
    EBIC_SWEEP(7);
    EBIC_SWEEP(8);
    EBIC_SWEEP(1);
#undef EBIC_SWEEP
    if constexpr (MASK) {
      // invalid candidates (class 0) still need their mask words cleared: the
      // host memsets the mask before the launch, so nothing to do here.
    }
  }
  __syncthreads();
  flush();
}

}  // namespace ebic
