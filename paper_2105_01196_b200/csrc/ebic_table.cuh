// ebic_table.cuh -- the pair-trend index: every consecutive-pair test of the
// matrix, precomputed once per (matrix, approx) as row bitsets.
//
// For an ordered column pair (a, b), bit r of the pair vector B(a, b) is the
// reference's per-pair test for row r (trend.cpp:22, forward step a -> b):
//     B(a, b)[r] = [ v_r(b) > v_r(a) - approx*|v_r(a)| ]  =  [ R_r(b) > T_r(a) ]
// (the exact rank-plane identity, ebic_plane.cuh).  The reversed step of
// trend.cpp:33 is B(b, a).  A candidate c_0..c_{L-1} is then supported by
// exactly the rows of
//     AND_k B(c_{k-1}, c_k)   |   AND_k B(c_k, c_{k-1})   (negatives only)
// so evaluate_population (trend.cpp:56-72) becomes L-1 (or 2(L-1)) streaming
// reads of R/8 bytes per candidate, ANDs and a popcount -- an HBM-bound kernel
// with no shared-memory gathers.  supporting_rows (trend.cpp:48-54) is the same
// AND, written out as the row mask (bit r = row r, natural order).
//
// Layout: table[(a * C + b) * wp + w], w < wp = round_up(ceil(R / 32), 32)
// words per pair (every vector starts on a 128-byte line); bits of rows >= R
// are zero.  Size
// C^2 * wp * 4 bytes: 2.5 GB at 20k x 1000 -- it is used when it fits the
// context's memory budget, otherwise the slab kernels run.
#pragma once
#include <cstdint>

#include "ebic_plane.cuh"

namespace ebic {

constexpr int kTableBuildWarps = 32;   // a-columns per builder CTA
constexpr int kTableRowsPerCta = 1024;  // rows per builder CTA (32 words)

// Builder: CTA (row block rb, a-tile) -- warp w owns column a = a0 + w and keeps
// the threshold keys of its 1024 rows in registers (lane l, i: row 32 i + l);
// the CTA streams W_b blocks of every column b through shared memory (two
// columns per barrier, the next two already loading into registers).  Word i
// of B(a, b) is one ballot over the warp; lane i keeps it, so
// the 32 words of a pair vector leave as one coalesced 128-byte store.
__global__ void __launch_bounds__(kTableBuildWarps * 32)
build_pair_table_kernel(const uint32_t* __restrict__ plane, uint64_t ld, uint32_t n_rows, uint32_t n_cols,
                        uint32_t wp, uint32_t* __restrict__ table) {
  __shared__ uint32_t s_wb[2][2][kTableRowsPerCta];  // [iteration parity][column of the pair][row]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r0 = blockIdx.x * kTableRowsPerCta;
  const uint32_t a = blockIdx.y * kTableBuildWarps + warp;
  const bool a_ok = a < n_cols;
  uint32_t ka[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t r = r0 + 32 * i + lane;
    // rows past the matrix never pass: no 32-bit word exceeds 0xFFFFFFFF
    ka[i] = (a_ok && r < n_rows) ? plane_key(__ldg(plane + (uint64_t)a * ld + r)) : 0xFFFFFFFFu;
  }
  // W_b blocks, two columns per barrier, register double-buffered: the loads
  // of the next two columns are in flight while the current two are compared
  const uint32_t r = r0 + threadIdx.x;
  auto fetch = [&](uint32_t b) -> uint32_t {
    return (b < n_cols && r < n_rows) ? __ldg(plane + (uint64_t)b * ld + r) : 0u;
  };
  const uint32_t w0 = r0 / 32;  // first word of this row block
  uint32_t n0 = fetch(0), n1 = fetch(1);
  int par = 0;
  for (uint32_t b = 0; b < n_cols; b += 2, par ^= 1) {
    // one barrier per two columns: the buffers alternate between iterations,
    // so writing this pair never races the previous pair's readers
    s_wb[par][0][threadIdx.x] = n0;
    s_wb[par][1][threadIdx.x] = n1;
    __syncthreads();
    n0 = fetch(b + 2);
    n1 = fetch(b + 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (b + h < n_cols) {
        const uint32_t* wb = s_wb[par][h];
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint32_t bits = __ballot_sync(kFull, wb[32 * i + lane] > ka[i]);
          if (lane == i) word = bits;
        }
        if (a_ok && w0 + lane < wp) table[((uint64_t)a * n_cols + b + h) * wp + w0 + lane] = word;
      }
    }
  }
}

// Evaluator: one CTA per candidate (grid-stride over candidates).  Thread t
// owns the uint4 slices t, t + T, ... of every pair vector (J = ceil(nv / T)
// of them, T = blockDim.x = min(1024, nv rounded up to a warp)), so a pair
// vector is read by the whole CTA in one coalesced sweep, and the loads of G
// pairs (G x J <= 4 slices per thread) are issued before they are combined:
// one HBM round trip per G pairs per candidate, with many candidates' CTAs in
// flight per SM.
// Counts are WRITTEN (out may be the device alias of page-locked host memory);
// MASK also writes the row-mask words.  Invalid candidates count 0 and store a
// code in *err_out: 1 = column >= n_cols, 2 = empty candidate / offsets not
// increasing / past n_idx.
template <int J, bool NEG, bool MASK>
__global__ void __launch_bounds__(1024)
table_count_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                   const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                   uint32_t n_idx, uint32_t* __restrict__ out, int* err_out, uint32_t* __restrict__ mask,
                   uint64_t mask_wpc) {
  constexpr int G = J >= 4 ? 1 : 4 / J;  // pairs whose loads are in flight together (G x J slices)
  __shared__ uint32_t s_part[2][32];
  const uint32_t T = blockDim.x, t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5, n_warps = (T + 31) >> 5;
  const uint32_t nv = wp / 4;  // uint4 per pair vector
  const uint4* t4 = reinterpret_cast<const uint4*>(table);
  int parity = 0;
  for (uint32_t i = blockIdx.x; i < n_cand; i += gridDim.x, parity ^= 1) {
    const uint32_t b = __ldg(offs + i), e = __ldg(offs + i + 1);
    const bool bad_offs = e <= b || e > n_idx;
    const uint32_t L = bad_offs ? 0 : e - b;
    bool badc = false;
    for (uint32_t k = t; k < L; k += T) badc |= __ldg(cols + b + k) >= n_cols;
    if (__syncthreads_or(bad_offs || badc)) {
      if (t == 0) {
        out[i] = 0;
        *err_out = bad_offs ? 2 : 1;
      }
      continue;
    }
    uint32_t n = 0;
    for (uint32_t v0 = 0; v0 < nv; v0 += T * J) {
      uint4 f[J], r[J];
#pragma unroll
      for (int u = 0; u < J; ++u) {
        // valid-row bits of the four words of slice v (word w covers rows [32 w, 32 w + 32))
        const uint32_t v = v0 + u * T + t;
        uint32_t m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t r0 = 32 * (4 * v + q);
          m[q] = (v < nv && r0 < n_rows) ? (n_rows - r0 >= 32 ? 0xFFFFFFFFu : (1u << (n_rows - r0)) - 1u) : 0u;
        }
        f[u] = make_uint4(m[0], m[1], m[2], m[3]);
        r[u] = NEG ? f[u] : make_uint4(0u, 0u, 0u, 0u);
      }
      uint32_t cp = __ldg(cols + b);
      for (uint32_t k0 = 1; k0 < L; k0 += G) {
        uint4 x[G][J], y[G][J];
        uint32_t pc[G + 1];
        pc[0] = cp;
#pragma unroll
        for (int g = 0; g < G; ++g) pc[g + 1] = k0 + g < L ? __ldg(cols + b + k0 + g) : 0u;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool live = k0 + g < L;
          const uint4* fwd = t4 + ((uint64_t)pc[g] * n_cols + pc[g + 1]) * nv;
          const uint4* rev = t4 + ((uint64_t)pc[g + 1] * n_cols + pc[g]) * nv;
#pragma unroll
          for (int u = 0; u < J; ++u) {
            // unconditional loads (see table_count_warp_kernel): a dead pair
            // re-reads the live pair-0 vector and its result is discarded
            const uint32_t v = min(v0 + u * T + t, nv - 1);
            const uint4* src = live ? fwd : t4 + ((uint64_t)pc[0] * n_cols + pc[1]) * nv;
            const uint4* srr = live ? rev : t4 + ((uint64_t)pc[1] * n_cols + pc[0]) * nv;
            const uint4 a = __ldg(src + v);
            x[g][u] = live ? a : make_uint4(~0u, ~0u, ~0u, ~0u);
            if (NEG) {
              const uint4 c = __ldg(srr + v);
              y[g][u] = live ? c : make_uint4(~0u, ~0u, ~0u, ~0u);
            }
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
          for (int u = 0; u < J; ++u) {
            f[u].x &= x[g][u].x; f[u].y &= x[g][u].y; f[u].z &= x[g][u].z; f[u].w &= x[g][u].w;
            if (NEG) {
              r[u].x &= y[g][u].x; r[u].y &= y[g][u].y; r[u].z &= y[g][u].z; r[u].w &= y[g][u].w;
            }
          }
        }
        {
          const uint32_t last = L - k0 < (uint32_t)G ? L - k0 : (uint32_t)G;  // pairs of this group
#pragma unroll
          for (int g = 1; g <= G; ++g)
            if ((uint32_t)g == last) cp = pc[g];  // (no dynamic register-array index)
        }
      }
#pragma unroll
      for (int u = 0; u < J; ++u) {
        const uint32_t v = v0 + u * T + t;
        const uint4 s = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
        n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
        if (MASK && v < nv) {
          uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
          const uint32_t words[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * v + q < mask_wpc) mw[q] = words[q];
        }
      }
    }
    // block sum: per-warp REDUX, then one thread; the partials alternate between
    // two buffers so one barrier per candidate suffices
    n = __reduce_add_sync(kFull, n);
    if (lane == 0) s_part[parity][warp] = n;
    __syncthreads();
    if (t < 32) {
      uint32_t x = t < (uint32_t)n_warps ? s_part[parity][t] : 0u;
      x = __reduce_add_sync(kFull, x);
      if (t == 0) out[i] = x;
    }
  }
}

// Evaluator for short pair vectors (nv <= 256 slices, i.e. up to 32K rows):
// one WARP per candidate, lane l owns the uint4 slices l, l + 32, ... (J =
// ceil(nv / 32) of them, a template parameter so the accumulators live in
// registers) and issues all J loads of a pair before combining them.  Same
// outputs and error codes as table_count_kernel.  (Measured on B200: batching
// several candidates per warp, several pairs' loads in flight, or prefetching
// the next candidate cost more in registers / occupancy than they gain; the
// kernel runs at 70-90% of the random-2.5-KB-chunk read ceiling measured by
// scripts/microbench/random_chunks.cu.)
template <int J, bool NEG, bool MASK, bool MULTI = false>
__global__ void __launch_bounds__(256)
table_count_warp_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                        const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                        uint32_t n_idx, uint32_t* __restrict__ out, int* err_out, uint32_t* __restrict__ mask,
                        uint64_t mask_wpc) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint32_t nv = wp / 4;  // uint4 per pair vector (== 32 J unless MULTI or J == 1)
  const uint4* t4 = reinterpret_cast<const uint4*>(table);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_cand; i += warps) {
    const uint32_t b = __ldg(offs + i), e = __ldg(offs + i + 1);
    const bool bad_offs = e <= b || e > n_idx;
    const uint32_t L = bad_offs ? 0 : e - b;
    bool badc = false;
    for (uint32_t k = b + lane; k < b + L; k += 32) badc |= __ldg(cols + k) >= n_cols;
    if (__any_sync(kFull, bad_offs || badc)) {
      if (lane == 0) {
        out[i] = 0;
        *err_out = bad_offs ? 2 : 1;
      }
      continue;
    }
    // the candidate's columns, 32 at a time in lane registers (shuffled out per pair)
    const uint32_t c_lane = lane < L ? __ldg(cols + b + lane) : 0u;
    uint32_t n = 0;
    // MULTI: vectors longer than 32 J slices are swept in passes of 32 J
    for (uint32_t v0 = 0; v0 < (MULTI ? nv : 1u); v0 += 32 * J) {
      uint4 f[J], r[J];
#pragma unroll
      for (int u = 0; u < J; ++u) {
        // valid-row bits of the four words of slice v (word w covers rows [32 w, 32 w + 32))
        const uint32_t v = v0 + u * 32 + lane;
        uint32_t m[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t r0 = 32 * (4 * v + q);
          m[q] = (v < nv && r0 < n_rows) ? (n_rows - r0 >= 32 ? 0xFFFFFFFFu : (1u << (n_rows - r0)) - 1u) : 0u;
        }
        f[u] = make_uint4(m[0], m[1], m[2], m[3]);
        r[u] = NEG ? f[u] : make_uint4(0u, 0u, 0u, 0u);
      }
      uint32_t cp = __shfl_sync(kFull, c_lane, 0);
      for (uint32_t k = 1; k < L; ++k) {
        const uint32_t cc = k < 32 ? __shfl_sync(kFull, c_lane, k & 31) : __ldg(cols + b + k);
        // all J loads unconditional, at immediate offsets from one base, so they
        // issue back to back (a predicated load lets ptxas reuse one destination
        // register and serialise the J round trips).  The host pads vectors of
        // more than 32 slices to a multiple of 32 (nv == 32 J); below that the
        // lanes past the vector re-read its last slice (same line; their
        // accumulators start at 0).  MULTI clamps every slice index instead.
        const uint4* fwd = t4 + ((uint64_t)cp * n_cols + cc) * nv;
        const uint4* rev = t4 + ((uint64_t)cc * n_cols + cp) * nv;
        uint4 x[J], y[J];
        if constexpr (MULTI) {
#pragma unroll
          for (int u = 0; u < J; ++u) {
            const uint32_t v = min(v0 + u * 32 + lane, nv - 1);
            x[u] = __ldg(fwd + v);
            if (NEG) y[u] = __ldg(rev + v);
          }
        } else {
          const uint32_t lv = J == 1 ? min((uint32_t)lane, nv - 1) : (uint32_t)lane;
#pragma unroll
          for (int u = 0; u < J; ++u) {
            x[u] = __ldg(fwd + lv + u * 32);
            if (NEG) y[u] = __ldg(rev + lv + u * 32);
          }
        }
#pragma unroll
        for (int u = 0; u < J; ++u) {
          f[u].x &= x[u].x; f[u].y &= x[u].y; f[u].z &= x[u].z; f[u].w &= x[u].w;
          if (NEG) {
            r[u].x &= y[u].x; r[u].y &= y[u].y; r[u].z &= y[u].z; r[u].w &= y[u].w;
          }
        }
        cp = cc;
      }
#pragma unroll
      for (int u = 0; u < J; ++u) {
        const uint32_t v = v0 + u * 32 + lane;
        const uint4 s = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
        n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
        if (MASK && v < nv) {
          uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
          const uint32_t words[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * v + q < mask_wpc) mw[q] = words[q];
        }
      }
    }
    n = __reduce_add_sync(kFull, n);
    if (lane == 0) out[i] = n;
  }
}

}  // namespace ebic
