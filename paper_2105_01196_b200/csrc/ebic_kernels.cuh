// ebic_kernels.cuh -- sm_100a kernels for batched bicluster fitness evaluation.
//
// Reference semantics (re-stated, not translated):
//   row_supports(m, r, c, p)  trend.cpp:41-46
//     forward : for k in 1..L-1:  v[k]   > v[k-1] - approx*|v[k-1]|      (trend.cpp:17-26)
//     reversed: for k in L-2..0:  v[k]   > v[k+1] - approx*|v[k+1]|      (trend.cpp:28-37)
//     result  : forward || (negative_trends && reversed)
//   evaluate_population       trend.cpp:56-72  -> fitness_count_kernel
//   supporting_rows           trend.cpp:48-54  -> fitness_count_kernel<MASK> + scatter_rows_kernel
//
// Both directions are evaluated in ONE forward sweep over the candidate's
// columns: at pair (v[k-1], v[k]) forward needs v[k] > thr(v[k-1]) and
// reversed needs v[k-1] > thr(v[k]), where thr(x) = RN64(x - RN64(approx*|x|)).
//
// Exactness:
//   * f64 store            : thr computed with __dmul_rn/__dsub_rn -- the reference ops.
//   * approx == 0          : thr(x) == x exactly, so the test is a native compare.
//   * f32 store, approx > 0: a float32 FILTER brackets thr in [lo, hi] with a proven
//     margin (|t_f32 - thr| <= 2^-22 (1+|a|)|x| + 2^-149, bracket half-width 4x that).
//     x > hi  => pass,  x <= lo => fail,  otherwise the row is re-evaluated with the
//     exact double arithmetic (row_exact).  Uncertain rows are ~1e-6 of all rows.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ebic {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 8;                // warps per CTA (one candidate per warp)
constexpr int kThreads = kWarps * 32;
constexpr int kColChunk = 64;            // column indices staged in SMEM per warp
constexpr uint32_t kRowAlign = 256;      // ld (padded rows) is a multiple of this

enum Mode : int { kModeNative = 0, kModeFilter = 1, kModeF64 = 2 };

struct TrendArgs {
  double approx;   // the reference's approx (double)
  float a_f;       // RN32(approx)
  float kscale;    // bracket half-width scale: >= (1+|approx|) * 2^-20
  int negative;    // negative_trends
};

template <typename T> struct Vec;
template <> struct Vec<float>  { using V = float4;  static constexpr int W = 4; };
template <> struct Vec<double> { using V = double2; static constexpr int W = 2; };

__device__ __forceinline__ float  vget(const float4& v, int i)  { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ double vget(const double2& v, int i) { return i == 0 ? v.x : v.y; }

__device__ __forceinline__ float4 ldv(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ldv(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// The reference threshold, bit-exact: RN64(x - RN64(a * |x|)) (no FMA contraction).
__device__ __forceinline__ double thr64(double x, double a) {
  return __dsub_rn(x, __dmul_rn(a, fabs(x)));
}

// row_supports() re-evaluated with the reference's double arithmetic.
// `cols` are global-memory column indices (already validated).
template <typename T>
__device__ bool row_exact(const T* __restrict__ mat, uint64_t ld, uint64_t row,
                          const uint32_t* __restrict__ cols, uint32_t len, double a, bool neg) {
  bool fwd = true;
  double prev = (double)mat[(uint64_t)cols[0] * ld + row];
  for (uint32_t k = 1; k < len && fwd; ++k) {
    double cur = (double)mat[(uint64_t)cols[k] * ld + row];
    fwd = cur > thr64(prev, a);
    prev = cur;
  }
  if (fwd) return true;
  if (!neg) return false;
  prev = (double)mat[(uint64_t)cols[len - 1] * ld + row];
  for (uint32_t k = len - 1; k-- > 0;) {
    double cur = (double)mat[(uint64_t)cols[k] * ld + row];
    if (!(cur > thr64(prev, a))) return false;
    prev = cur;
  }
  return true;
}

// Half-width of the float32 bracket of thr64(x) around t = x - a_f |x|
// (|x| = ax).  x = +-0 has the exact threshold +-0 (thr64: x - a * 0), which
// t reproduces, so its bracket is empty: no row with x = 0 (common: zeros in
// expression data) takes the double test.
__device__ __forceinline__ float bracket_halfwidth(float ax, float kscale) {
  return ax > 0.f ? __fmaf_rn(kscale, ax, 0x1p-146f) : 0.f;
}

// Per-element bracket of the threshold, float32 filter mode.
__device__ __forceinline__ void bracket(float x, const TrendArgs& ta, float& lo, float& hi) {
  const float ax = fabsf(x);
  const float t = __fmaf_rn(-ta.a_f, ax, x);
  const float d = bracket_halfwidth(ax, ta.kscale);
  lo = __fsub_rn(t, d);
  hi = __fadd_rn(t, d);
}

// ---------------------------------------------------------------------------
// fitness_count_kernel
//   grid.x : candidate groups of kWarps (warp w of CTA b owns candidate b*kWarps+w)
//   grid.y : row slabs of `slab_rows` rows (slab-major order keeps the working
//            set of concurrently resident CTAs inside L2)
//   lane   : NV vectors of W consecutive rows per pass, coalesced 512 B per
//            warp-load (float32) -- rows base + 32*W*n + W*lane + i
// MASK=true additionally writes the row-membership bitmask
//   mask[cand * (ld/32) + row/32] bit (row%32)
// ---------------------------------------------------------------------------
template <typename T, int MODE, bool NEG, bool MASK>
__global__ void __launch_bounds__(kThreads)
fitness_count_kernel(const T* __restrict__ mat, uint64_t ld, uint32_t n_rows, uint32_t n_cols,
                     const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs,
                     uint32_t n_cand, uint32_t slab_rows, TrendArgs ta,
                     uint32_t* __restrict__ counts, uint32_t* __restrict__ mask,
                     int* __restrict__ err) {
  using V = typename Vec<T>::V;
  constexpr int W = Vec<T>::W;
  constexpr int NV = 2;                 // vectors per lane per pass
  constexpr int RPL = W * NV;           // rows per lane per pass
  constexpr uint32_t kPass = 32u * RPL; // rows per warp per pass
  static_assert(kRowAlign % kPass == 0, "row padding must cover a pass");
  constexpr int G = 4;                  // columns loaded ahead

  __shared__ uint32_t s_cols[kWarps][kColChunk];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cand = blockIdx.x * kWarps + warp;
  if (cand >= n_cand) return;

  const uint32_t beg = offs[cand];
  const uint32_t len = offs[cand + 1] - beg;
  const uint32_t* gcols = cols + beg;

  // validate the candidate (warp-uniform decision)
  bool bad = (len == 0) || (offs[cand + 1] < beg);
  if (!bad) {
    for (uint32_t k = lane; k < len; k += 32) bad |= (gcols[k] >= n_cols);
    bad = __any_sync(kFull, bad);
  }
  if (bad) {
    if (lane == 0) atomicOr(err, 1);
    return;
  }

  const uint32_t row0 = blockIdx.y * slab_rows;
  if (row0 >= n_rows) return;
  const uint32_t row_end = min(row0 + slab_rows, n_rows);
  const double a = ta.approx;

  // stage the first chunk of column indices
  uint32_t staged = 0xffffffffu;
  auto stage = [&](uint32_t chunk) {
    __syncwarp();
    const uint32_t cs = chunk * kColChunk;
    for (uint32_t k = lane; k < kColChunk && cs + k < len; k += 32) s_cols[warp][k] = gcols[cs + k];
    __syncwarp();
    staged = chunk;
  };

  uint32_t my_count = 0;

  for (uint32_t base = row0; base < row_end; base += kPass) {
    T prev[RPL];
    float plo[RPL], phi[RPL];   // bracket of thr(prev) (filter mode)
    double pthr[RPL];           // thr(prev) (f64 mode)
    bool okf[RPL], okr[RPL], unc[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const uint32_t r = base + 32u * W * (i / W) + W * lane + (i % W);
      okf[i] = r < row_end;
      okr[i] = NEG && okf[i];
      unc[i] = false;
    }

    const T* pbase = mat + base + W * lane;
    for (uint32_t j = 0; j < len; j += G) {
      V buf[G][NV];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t k = j + g;
        if (k < len) {
          if (k / kColChunk != staged) stage(k / kColChunk);
          const uint64_t c = s_cols[warp][k % kColChunk];
          const T* p = pbase + c * ld;
#pragma unroll
          for (int n = 0; n < NV; ++n) buf[g][n] = ldv(p + 32 * W * n);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t k = j + g;
        if (k < len) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const T cur = vget(buf[g][i / W], i % W);
            if constexpr (MODE == kModeNative) {
              if (k > 0) {
                okf[i] = okf[i] && (cur > prev[i]);
                if (NEG) okr[i] = okr[i] && (prev[i] > cur);
              }
            } else if constexpr (MODE == kModeFilter) {
              float lo, hi;
              bracket((float)cur, ta, lo, hi);
              if (k > 0) {
                const float c = (float)cur, p = (float)prev[i];
                const bool f_hi = c > phi[i], f_lo = c > plo[i];
                okf[i] = okf[i] && f_hi;
                unc[i] = unc[i] || (f_lo && !f_hi);
                if (NEG) {
                  const bool r_hi = p > hi, r_lo = p > lo;
                  okr[i] = okr[i] && r_hi;
                  unc[i] = unc[i] || (r_lo && !r_hi);
                }
              }
              plo[i] = lo;
              phi[i] = hi;
            } else {  // kModeF64
              const double t = thr64((double)cur, a);
              if (k > 0) {
                okf[i] = okf[i] && ((double)cur > pthr[i]);
                if (NEG) okr[i] = okr[i] && ((double)prev[i] > t);
              }
              pthr[i] = t;
            }
            prev[i] = cur;
          }
        }
      }
      // warp-uniform early exit: nothing left that a further column could change
      bool alive = false;
#pragma unroll
      for (int i = 0; i < RPL; ++i) alive = alive || okf[i] || okr[i];
      if (!__any_sync(kFull, alive)) break;
    }

    // resolve, count, mask
    uint32_t bits = 0;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const uint32_t r = base + 32u * W * (i / W) + W * lane + (i % W);
      bool res = okf[i] || okr[i];
      if constexpr (MODE == kModeFilter) {
        if (unc[i] && r < row_end) res = row_exact<T>(mat, ld, r, gcols, len, a, NEG);
      }
      res = res && (r < row_end);
      my_count += res ? 1u : 0u;
      bits |= (res ? 1u : 0u) << i;
    }
    if (MASK) {
      // vector n of this lane covers rows base + 32*W*n + W*lane + [0, W)
#pragma unroll
      for (int n = 0; n < NV; ++n) {
        uint32_t nib = (bits >> (n * W)) & ((1u << W) - 1u);
        constexpr int LPW = 32 / W;  // lanes contributing to one 32-row word
        uint32_t word = nib << (W * (lane % LPW));
#pragma unroll
        for (int s = 1; s < LPW; s <<= 1) word |= __shfl_xor_sync(kFull, word, s);
        if (lane % LPW == 0) {
          const uint64_t wrow = base + 32u * W * n + W * lane;  // multiple of 32
          mask[(uint64_t)cand * (ld / 32) + wrow / 32] = word;
        }
      }
    }
  }

  const uint32_t total = __reduce_add_sync(kFull, my_count);
  if (lane == 0 && total) atomicAdd(&counts[cand], total);
}

// ---------------------------------------------------------------------------
// scatter_rows_kernel: one CTA per candidate turns its bitmask into the
// ascending row list at rows_out[row_offsets[cand] ...] (stable compaction:
// block-wide exclusive scan of per-word popcounts).
// ---------------------------------------------------------------------------
constexpr int kScatterThreads = 1024;

__global__ void __launch_bounds__(kScatterThreads)
scatter_rows_kernel(const uint32_t* __restrict__ mask, uint64_t words_per_cand, uint64_t n_words_valid,
                    const uint64_t* __restrict__ row_offsets, uint64_t row_base,
                    uint32_t* __restrict__ rows_out) {
  __shared__ uint32_t s_warp[kScatterThreads / 32];
  __shared__ uint64_t s_carry;
  const uint32_t cand = blockIdx.x;
  const uint32_t* m = mask + (uint64_t)cand * words_per_cand;
  uint32_t* out = rows_out + row_offsets[cand];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint64_t w0 = 0; w0 < n_words_valid; w0 += kScatterThreads) {
    const uint64_t w = w0 + threadIdx.x;
    const uint32_t word = w < n_words_valid ? m[w] : 0u;
    const uint32_t c = __popc(word);
    // warp inclusive scan
    uint32_t x = c;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, x, s);
      if (lane >= s) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = s_warp[lane];
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, v, s);
        if (lane >= s) v += y;
      }
      s_warp[lane] = v;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t excl = s_carry + (warp ? s_warp[warp - 1] : 0u) + (x - c);
    uint32_t bitsleft = word;
    uint64_t o = excl;
    while (bitsleft) {
      const int b = __ffs(bitsleft) - 1;
      bitsleft &= bitsleft - 1;
      out[o++] = (uint32_t)(row_base + w * 32 + b);
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_warp[kScatterThreads / 32 - 1];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// overlap_popc_kernel: pairwise row-set intersections of a batch, from its
// row bitmasks -- the |rows_a n rows_b| of induced_jaccard (evolution.cpp:44-51)
// without row lists.  CTA (i, t) pairs candidate i with candidates
// [t*kOverlapTile, +kOverlapTile) at or above the diagonal; each thread ANDs
// its words of mask i with the tile's masks, then a block reduction.  Both
// inter[i*n + j] and inter[j*n + i] are written.
// ---------------------------------------------------------------------------
constexpr int kOverlapTile = 8;
constexpr int kOverlapThreads = 256;

__global__ void __launch_bounds__(kOverlapThreads)
overlap_popc_kernel(const uint32_t* __restrict__ mask, uint64_t words_per_cand, uint64_t n_words_valid,
                    uint32_t n, uint32_t* __restrict__ inter) {
  const uint32_t i = blockIdx.x, j0 = blockIdx.y * kOverlapTile;
  if (j0 + kOverlapTile <= i) return;  // the tile is wholly below the diagonal
  const uint32_t* mi = mask + (uint64_t)i * words_per_cand;
  uint32_t c[kOverlapTile] = {};
  for (uint64_t w = threadIdx.x; w < n_words_valid; w += kOverlapThreads) {
    const uint32_t a = mi[w];
#pragma unroll
    for (int t = 0; t < kOverlapTile; ++t)
      if (j0 + t < n && j0 + t >= i) c[t] += __popc(a & mask[(uint64_t)(j0 + t) * words_per_cand + w]);
  }
  __shared__ uint32_t s_part[kOverlapThreads / 32][kOverlapTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kOverlapTile; ++t) {
    const uint32_t v = __reduce_add_sync(kFull, c[t]);
    if (lane == 0) s_part[warp][t] = v;
  }
  __syncthreads();
  if (threadIdx.x < kOverlapTile) {
    const uint32_t j = j0 + threadIdx.x;
    if (j < n && j >= i) {
      uint32_t v = 0;
      for (int w = 0; w < kOverlapThreads / 32; ++w) v += s_part[w][threadIdx.x];
      inter[(uint64_t)i * n + j] = v;
      inter[(uint64_t)j * n + i] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// single (row, candidate) predicate with the reference arithmetic
// ---------------------------------------------------------------------------
template <typename T>
__global__ void row_supports_kernel(const T* __restrict__ mat, uint64_t ld, uint64_t row,
                                    const uint32_t* __restrict__ cols, uint32_t len, double a,
                                    int neg, int* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = row_exact<T>(mat, ld, row, cols, len, a, neg != 0) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// matrix store: check + transpose (row-major -> column-major, padded)
// ---------------------------------------------------------------------------
// flags bit0: a non-finite value; bit1: a value not exactly representable in float32
template <typename TI>
__global__ void check_values_kernel(const TI* __restrict__ in, uint64_t n, int* __restrict__ flags) {
  int f = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = (double)in[i];
    if (!isfinite(v)) f |= 1;
    if ((double)(float)v != v) f |= 2;
  }
  f = (int)__reduce_or_sync(kFull, (unsigned)f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

template <typename TI, typename TO>
__global__ void transpose_kernel(const TI* __restrict__ in, uint64_t n_rows, uint64_t n_cols,
                                 TO* __restrict__ out, uint64_t ld, uint64_t ld_rows_total) {
  // tile 32 (rows) x 32 (cols); block (32, 8)
  __shared__ TO tile[32][33];
  const uint64_t r0 = (uint64_t)blockIdx.y * 32, c0 = (uint64_t)blockIdx.x * 32;
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const uint64_t r = r0 + dy, c = c0 + threadIdx.x;
    tile[dy][threadIdx.x] = (r < n_rows && c < n_cols) ? (TO)in[r * n_cols + c] : (TO)0;
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    const uint64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (c < n_cols && r < ld_rows_total) out[c * ld + r] = tile[threadIdx.x][dy];
  }
}

}  // namespace ebic
