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

// ---------------------------------------------------------------------------
// slab kernel
//   RPL : consecutive rows per lane (1, 2, 4)   -> LDS.32 / .64 / .128
//   SUB : candidates per warp (1, 2, 4)          -> 32/SUB lanes per candidate
//   RT  = (32 / SUB) * RPL rows per slab
// work unit = (candidate chunk, row slab), linearised chunk-major; CTA b owns
// units [b*U/G, (b+1)*U/G).
// ---------------------------------------------------------------------------
template <int RPL> struct LdsVec;
template <> struct LdsVec<1> { using V = uint32_t; };
template <> struct LdsVec<2> { using V = uint2; };
template <> struct LdsVec<4> { using V = uint4; };
__device__ __forceinline__ uint32_t vel(const uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t vel(const uint2& v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ uint32_t vel(const uint4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

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
};

template <int RPL, int SUB, bool NEG, bool MASK>
__global__ void __launch_bounds__(kSlabThreads, 1)
slab_count_kernel(const SlabArgs a) {
  constexpr int LPC = 32 / SUB;        // lanes per candidate
  constexpr uint32_t RT = LPC * RPL;   // rows per slab
  using V = typename LdsVec<RPL>::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(smem_raw);               // [C][RT]
  uint4* s_rec = reinterpret_cast<uint4*>(s_slab + (size_t)a.n_cols * RT);  // [chunk]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_rec + a.chunk);          // [chunk]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPC, rl = lane % LPC;
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
      __syncthreads();
      cur_chunk = chunk;
      c_begin = chunk * a.chunk;
      c_n = min(a.chunk, a.n_cand - c_begin);
      // pack candidate records: 7 x u16 columns + u16 length
      for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
        const uint32_t i = c_begin + j;
        const uint32_t b = a.offs[i], e = a.offs[i + 1];
        const uint32_t len = e > b ? e - b : 0;
        uint32_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        bool bad = len == 0 || len > 0xFFFFu;
#pragma unroll
        for (int k = 0; k < kRecCols; ++k) {
          if ((uint32_t)k < len) {
            h[k] = a.cols[b + k];
            bad |= h[k] >= a.n_cols;
          }
        }
        for (uint32_t k = kRecCols; k < len && !bad; ++k) bad |= a.cols[b + k] >= a.n_cols;
        if (bad) {
          atomicOr(a.err, 1);
#pragma unroll
          for (int k = 0; k < 8; ++k) h[k] = 0;  // len 0: counted as 0
        } else {
          h[7] = len;
        }
        s_rec[j] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
        s_cnt[j] = 0;
      }
    }
    // stage the slab: rows [row0, row0+RT) of every column (RT*4 bytes contiguous per column)
    {
      constexpr uint32_t V4 = RT / 4;  // uint4 per column
      const uint64_t total = (uint64_t)a.n_cols * V4;
      const uint4* src = reinterpret_cast<const uint4*>(a.plane);
      uint4* dst = reinterpret_cast<uint4*>(s_slab);
      for (uint64_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint64_t c = t / V4, q = t % V4;
        dst[t] = __ldg(src + (c * a.ld + row0) / 4 + q);
      }
    }
    __syncthreads();

    const uint32_t valid_rows = min(RT, a.n_rows - row0);
    // per-lane row validity bits
    uint32_t vmask = 0;
#pragma unroll
    for (int j = 0; j < RPL; ++j) vmask |= (rl * RPL + j < valid_rows ? 1u : 0u) << j;

    const uint32_t n_iter = (c_n + kSlabWarps * SUB - 1) / (kSlabWarps * SUB);
    for (uint32_t it = 0; it < n_iter; ++it) {
      const uint32_t j = (it * kSlabWarps + warp) * SUB + sub;  // candidate within chunk
      const bool have = j < c_n;
      uint32_t okf = 0, okr = 0;
      if (have) {
        const uint4 rec = s_rec[j];
        const uint32_t len = rec.w >> 16;
        uint32_t cc[kRecCols] = {rec.x & 0xFFFFu, rec.x >> 16, rec.y & 0xFFFFu, rec.y >> 16,
                                 rec.z & 0xFFFFu, rec.z >> 16, rec.w & 0xFFFFu};
        const uint32_t lane_off = rl * RPL;
        V wp = *reinterpret_cast<const V*>(s_slab + cc[0] * RT + lane_off);
        okf = len ? vmask : 0u;
        okr = NEG ? okf : 0u;
#pragma unroll
        for (int k = 1; k < kRecCols; ++k) {
          if ((uint32_t)k < len) {
            const V wc = *reinterpret_cast<const V*>(s_slab + cc[k] * RT + lane_off);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const uint32_t p = vel(wp, r), c = vel(wc, r);
              okf &= ~((c > plane_key(p) ? 0u : 1u) << r);
              if (NEG) okr &= ~((p > plane_key(c) ? 0u : 1u) << r);
            }
            wp = wc;
          }
        }
        if (len > kRecCols) {
          // long candidate: continue from the CSR (rare; evolved populations have L <= ~10)
          const uint32_t* gc = a.cols + a.offs[c_begin + j];
          for (uint32_t k = kRecCols; k < len; ++k) {
            if ((okf | okr) == 0u) break;  // per-lane: nothing left to decide
            const V wc = *reinterpret_cast<const V*>(s_slab + gc[k] * RT + lane_off);
#pragma unroll
            for (int r = 0; r < RPL; ++r) {
              const uint32_t p = vel(wp, r), c = vel(wc, r);
              okf &= ~((c > plane_key(p) ? 0u : 1u) << r);
              if (NEG) okr &= ~((p > plane_key(c) ? 0u : 1u) << r);
            }
            wp = wc;
          }
        }
      }
      const uint32_t ok = okf | okr;  // RPL bits, one per row of this lane
      if (MASK) {
        static_assert(!MASK || (RPL == 1 && SUB == 1), "mask output needs one row per lane");
        const uint32_t word = __ballot_sync(kFull, ok & 1u);
        if (have && lane == 0) a.mask[(uint64_t)(c_begin + j) * a.mask_wpc + row0 / 32] = word;
        if (have && lane == 0 && word) s_cnt[j] += __popc(word);
      } else {
        uint32_t n;
        if (RPL == 1) {
          const uint32_t b = __ballot_sync(kFull, ok & 1u);
          n = SUB == 1 ? __popc(b) : __popc((b >> (sub * LPC)) & (LPC == 32 ? 0xffffffffu : ((1u << LPC) - 1u)));
        } else {
          n = __popc(ok);
          // reduce within the lanes of this candidate
#pragma unroll
          for (int s = LPC / 2; s > 0; s >>= 1) n += __shfl_xor_sync(kFull, n, s);
        }
        if (have && rl == 0 && n) s_cnt[j] += n;
      }
    }
  }
  __syncthreads();
  flush();
}

}  // namespace ebic
