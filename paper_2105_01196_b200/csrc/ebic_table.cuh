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
// Layout: table[(a * C + b) * wp + w]; word w covers rows 32 w .. 32 w + 31
// (byte-interleaved even / odd rows: index_bit_row, index_valid_bits);
// wp = ceil(R / 32) rounded up to 4 words, or to 128 above 128 words; bits of
// rows >= R are zero.  Size
// C^2 * wp * 4 bytes: 2.5 GB at 20k x 1000 -- it is used when it fits the
// context's memory budget, otherwise the slab kernels run.
#pragma once
#include <cstdint>

#include "ebic_plane.cuh"
#include "ebic_index.cuh"
#include "ebic_lazy.cuh"

namespace ebic {

constexpr int kTableBuildWarps = 32;   // a-columns per builder CTA
constexpr int kTableRowsPerCta = 1024;  // rows per builder CTA (32 words)

// Sign-replicating byte permute: byte k of the result is 0xFF or 0x00 by
// bit 15 (k = 0) / 31 (k = 1) of lo and bit 15 (k = 2) / 31 (k = 3) of hi.
__device__ __forceinline__ uint32_t prmt_sign15_31(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0xFDB9;" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ uint2 ldg_u2(const uint32_t* p) {
  return __ldg(reinterpret_cast<const uint2*>(p));
}

// Builder: CTA = (row block of 1024 rows, tile of 32 columns a).  Warp w owns
// column a = a0 + w; lane l owns the 32 rows of word l of the block and keeps
// their negated thresholds as 16 packed row pairs (NT, as in the slab kernel:
// 0 - (T_even | T_odd << 16) - 0x00010001).  The CTA streams every column b's
// guarded ranks (Rg = R | 0x8000 per row, two rows per word) through shared
// memory, two columns per barrier, the next two already loading (one 8-byte
// load per row pair).  For a pair word, D = Rg(b) + NT(a) has bit 15 set iff
// R_b > T_a for the even row and bit 31 for the odd row (ebic_simd.cuh), so
// one IADD tests two rows; pairs j and j + 8 are filed together by one
// sign-replicating PRMT (four bytes of 0x00 / 0xFF) and one LOP3 (bit j of
// each byte): 16 IADD + 8 PRMT + 8 LOP3 per index word, and the warp's 32
// words leave as one coalesced 128-byte store.  Shared layout: pair j of word
// l at j * 33 + l -- conflict-free reads at immediate offsets (lane l reads
// word l of row j), at most 2-way conflicts for the staging stores.
//
// A = a-columns per warp: with A = 2 a warp keeps the thresholds of columns
// a and a + 16 (32 packed registers) and every shared-memory read of a column
// b pair feeds two IADDs, so a CTA of 16 warps still covers 32 columns a.
template <int A>
__global__ void __launch_bounds__(kTableBuildWarps / A * 32, A)
build_pair_table_kernel(const uint32_t* __restrict__ plane, uint64_t ld, uint32_t n_rows, uint32_t n_cols,
                        uint32_t wp, uint32_t* __restrict__ table, uint32_t b_per_z) {
  // blockIdx.z: this CTA's slice [b_begin, b_end) of the columns b (even
  // length; slices only balance the waves -- every (a, b) is built once)
  const uint32_t b_begin = blockIdx.z * b_per_z, b_end = min(n_cols, b_begin + b_per_z);
  constexpr int T = kTableBuildWarps / A * 32;                 // threads
  constexpr int PAIRS = kTableRowsPerCta / 2;                  // row pairs of the block
  constexpr int SW = 33;                                       // words per staged pair row j (32 + 1 pad)
  constexpr uint32_t COLB = 16 * SW * 4;                       // bytes per staged column
  __shared__ uint32_t s_rg[2][2][16 * SW];  // [iteration parity][column of the pair][pair j * SW + word]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r0 = blockIdx.x * kTableRowsPerCta;
  const uint32_t w0 = r0 / 32;  // first word of this row block
  uint32_t ac[A];
  bool a_ok[A];
  // this lane's 32 rows of each column a -> 16 negated threshold pairs
  uint32_t nt[A][16];
#pragma unroll
  for (int q = 0; q < A; ++q) {
    ac[q] = blockIdx.y * kTableBuildWarps + warp + q * (kTableBuildWarps / A);
    a_ok[q] = ac[q] < n_cols;
    const uint32_t rl = r0 + 32 * lane;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t re = rl + 2 * j;  // (re < n_rows keeps re + 1 inside the column's ld rows)
      const uint2 v = (a_ok[q] && re < n_rows) ? ldg_u2(plane + (uint64_t)ac[q] * ld + re) : make_uint2(0u, 0u);
      nt[q][j] = 0u - __byte_perm(v.x, v.y, 0x5410) - 0x00010001u;  // T_even | T_odd << 16, negated
    }
  }
  const uint32_t valid = index_valid_bits(n_rows, w0 + lane);
  // staging: each thread packs PER row pairs of columns b and b + 1
  constexpr int PER = 2 * PAIRS / T;  // pairs staged per thread per iteration (2 with A = 1, 4 with A = 2)
  uint32_t nxt[PER];
  auto fetch = [&](uint32_t b) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t idx = threadIdx.x + k * T;  // 0 .. 2 PAIRS - 1
      const uint32_t col = b + idx / PAIRS, tp = idx % PAIRS;
      const uint32_t re = r0 + 2 * tp;
      const uint2 v = (col < n_cols && re < n_rows) ? ldg_u2(plane + (uint64_t)col * ld + re) : make_uint2(0u, 0u);
      nxt[k] = __byte_perm(v.x, v.y, 0x7632) | 0x80008000u;  // guarded ranks Rg of the pair
    }
  };
  auto stage = [&](int par) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t idx = threadIdx.x + k * T;
      const uint32_t tp = idx % PAIRS;
      s_rg[par][idx / PAIRS][(tp & 15) * SW + (tp >> 4)] = nxt[k];  // pair j = tp & 15 of word tp >> 4
    }
  };
  fetch(b_begin);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(&s_rg[0][0][0]) + 4 * lane;
  // this lane's output word of pair (a_0, b): advanced by wp per column b; the
  // other a-columns of the warp are kTableBuildWarps / A columns further on
  const bool st_ok = w0 + lane < wp;
  uint32_t* trow = table + ((uint64_t)ac[0] * n_cols + b_begin) * wp + w0 + lane;
  const uint64_t qstride = (uint64_t)(kTableBuildWarps / A) * n_cols * wp;
  int par = 0;
  for (uint32_t b = b_begin; b < b_end; b += 2, par ^= 1, trow += 2 * wp) {
    // one barrier per two columns: the buffers alternate between iterations,
    // so writing this pair never races the previous pair's readers
    stage(par);
    __syncthreads();
    fetch(b + 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (b + h < b_end) {
        const uint32_t base = sbase + (uint32_t)(2 * par + h) * COLB;
        uint32_t x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x[j]) : "r"(base + j * SW * 4));
        uint32_t word[A];
#pragma unroll
        for (int q = 0; q < A; ++q) word[q] = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
          for (int q = 0; q < A; ++q)
            word[q] |= prmt_sign15_31(x[j] + nt[q][j], x[j + 8] + nt[q][j + 8]) & (0x01010101u << j);
        }
#pragma unroll
        for (int q = 0; q < A; ++q)
          if (st_ok && a_ok[q]) trow[h * wp + q * qstride] = word[q] & valid;
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
    if (L == 1) {  // no pair: every row supports (the trend.cpp:19 loop never runs)
      if (t == 0) out[i] = n_rows;
      if (MASK)
        for (uint32_t w = t; w < mask_wpc; w += T)
          mask[(uint64_t)i * mask_wpc + w] = index_to_natural(index_valid_bits(n_rows, w));
      continue;
    }
    uint32_t n = 0;
    for (uint32_t v0 = 0; v0 < nv; v0 += T * J) {
      // accumulators start all-ones: the index has no bits past the last row
      uint4 f[J], r[J];
#pragma unroll
      for (int u = 0; u < J; ++u) {
        f[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
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
        const uint4 o = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
        const uint4 s = v < nv ? o : make_uint4(0u, 0u, 0u, 0u);  // (threads past the vector re-read its end)
        n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
        if (MASK && v < nv) {
          uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
          const uint32_t words[4] = {index_to_natural(s.x), index_to_natural(s.y), index_to_natural(s.z),
                                     index_to_natural(s.w)};
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
template <int J, bool NEG, bool MASK>
__global__ void __launch_bounds__(256)
table_count_warp_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                        const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                        uint32_t n_idx, uint32_t* __restrict__ out, int* err_out, uint32_t* __restrict__ mask,
                        uint64_t mask_wpc) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint32_t nv = wp / 4;  // uint4 per pair vector (<= 32 J)
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
    if (L == 1) {  // no pair: every row supports (the trend.cpp:19 loop never runs)
      if (lane == 0) out[i] = n_rows;
      if (MASK)
        for (uint32_t w = lane; w < mask_wpc; w += 32) mask[(uint64_t)i * mask_wpc + w] =
            index_to_natural(index_valid_bits(n_rows, w));
      continue;
    }
    // the candidate's columns, 32 at a time in lane registers (shuffled out per pair)
    const uint32_t c_lane = lane < L ? __ldg(cols + b + lane) : 0u;
    // accumulators start all-ones: the index has no bits past the last row, so
    // after the first pair they hold exactly the supporting rows
    uint4 f[J], r[J];
#pragma unroll
    for (int u = 0; u < J; ++u) {
      f[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
      r[u] = NEG ? f[u] : make_uint4(0u, 0u, 0u, 0u);
    }
    const uint32_t lv = J == 1 ? min((uint32_t)lane, nv - 1) : (uint32_t)lane;
    if constexpr (!NEG) {
      // software-pipelined: pair k + 1's J loads are in flight while pair k is
      // combined (as in the multi-pass kernel)
      auto col = [&](uint32_t j) -> uint32_t { return j < 32 ? __shfl_sync(kFull, c_lane, j & 31) : __ldg(cols + b + j); };
      auto vec = [&](uint32_t k) -> const uint4* {
        return t4 + ((uint64_t)col(k - 1) * n_cols + col(k)) * nv + lv;
      };
      uint4 xa[J];
      {
        const uint4* p0 = vec(1);
#pragma unroll
        for (int u = 0; u < J; ++u) xa[u] = __ldg(p0 + u * 32);
      }
      for (uint32_t k = 1; k + 1 < L; ++k) {
        const uint4* pn = vec(k + 1);
        uint4 xb[J];
#pragma unroll
        for (int u = 0; u < J; ++u) xb[u] = __ldg(pn + u * 32);
#pragma unroll
        for (int u = 0; u < J; ++u) {
          f[u].x &= xa[u].x; f[u].y &= xa[u].y; f[u].z &= xa[u].z; f[u].w &= xa[u].w;
          xa[u] = xb[u];
        }
      }
#pragma unroll
      for (int u = 0; u < J; ++u) {
        f[u].x &= xa[u].x; f[u].y &= xa[u].y; f[u].z &= xa[u].z; f[u].w &= xa[u].w;
      }
    } else {
    uint32_t cp = __shfl_sync(kFull, c_lane, 0);
    for (uint32_t k = 1; k < L; ++k) {
      const uint32_t cc = k < 32 ? __shfl_sync(kFull, c_lane, k & 31) : __ldg(cols + b + k);
      // all J loads unconditional, at immediate offsets from one base, so they
      // issue back to back (a predicated load lets ptxas reuse one destination
      // register and serialise the J round trips).  The host pads vectors of
      // more than 32 slices to a multiple of 32 (nv == 32 J); below that the
      // lanes past the vector re-read its last slice (same line; their
      // accumulators start at 0)
      const uint4* fwd = t4 + ((uint64_t)cp * n_cols + cc) * nv + lv;
      const uint4* rev = t4 + ((uint64_t)cc * n_cols + cp) * nv + lv;
      uint4 x[J], y[J];
#pragma unroll
      for (int u = 0; u < J; ++u) {
        x[u] = __ldg(fwd + u * 32);
        if (NEG) y[u] = __ldg(rev + u * 32);
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
    }
    uint32_t n = 0;
#pragma unroll
    for (int u = 0; u < J; ++u) {
      const uint32_t v = u * 32 + lane;
      const uint4 o = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
      // (J == 1: lanes past the vector re-read its last slice -- drop them)
      const uint4 s = (J > 1 || v < nv) ? o : make_uint4(0u, 0u, 0u, 0u);
      n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
      if (MASK && v < nv) {
        uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
        const uint32_t words[4] = {index_to_natural(s.x), index_to_natural(s.y), index_to_natural(s.z),
                                   index_to_natural(s.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (4 * v + q < mask_wpc) mw[q] = words[q];
      }
    }
    n = __reduce_add_sync(kFull, n);
    if (lane == 0) out[i] = n;
  }
}

// Programmatic dependent launch (PDL).  The count kernels let the next kernel
// of their stream launch as soon as they start (their CTAs are persistent, so
// the next grid's CTAs only fill SM slots as this grid's CTAs retire: the
// tail of batch k overlaps the start of batch k+1), and wait for the previous
// grid before their first global store (a back-to-back batch may write the
// same output buffer).  The count kernels read nothing an earlier count
// kernel writes; kernels whose output they do read (the index builders, the
// lazy pair builder) never trigger early, so the count kernel starts after
// them as usual.  Both instructions are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Long vectors (> 256 slices) with many candidates: the same warp-per-
// candidate scheme sweeping the vectors in passes of 32 J slices (every slice
// index clamped, loads still unconditional).  A separate kernel so that the
// single-pass kernel above keeps its register allocation and load schedule.
//
// LAZY (long vectors only, MULTI): the vectors come from the lazy index's
// pool, built ahead of this kernel by lazy_claim_kernel / lazy_build_kernel
// (ebic_lazy.cuh).  A candidate with a pair whose slot is not ready (the pool
// was full, or another stream's batch is still building it) is deferred to
// lazy_deferred_kernel, which computes such pairs from the value store -- the
// same bits either way -- so this kernel keeps the register budget of the
// plain index kernel.  (A persistent, software-pipelined variant of this
// kernel -- the next candidate's offsets, columns and slots fetched during the
// current one's passes -- measured 0.70 vs 0.44 ms at C4 and was dropped.)
template <int J, bool NEG, bool MASK, bool MULTI = true, bool LAZY = false>
__global__ void __launch_bounds__(256)
table_count_warp_multi_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                        const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                        uint32_t n_idx, uint32_t* __restrict__ out, int* err_out, uint32_t* __restrict__ mask,
                        uint64_t mask_wpc, const LazyArgs la) {
  static_assert(!LAZY || MULTI, "the lazy index runs the multi-pass kernel");
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint32_t nv = wp / 4;  // uint4 per pair vector (== 32 J unless MULTI or J == 1)
  const uint4* t4 = reinterpret_cast<const uint4*>(LAZY ? la.pool : table);
  // programmatic dependent launch (pdl_trigger): wait for the previous grid
  // only before this warp's first global store
  pdl_trigger();
  bool dep_done = false;
  auto before_store = [&]() {
    if (!dep_done) {
      pdl_wait();
      dep_done = true;
    }
  };
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_cand; i += warps) {
    const uint32_t b = __ldg(offs + i), e = __ldg(offs + i + 1);
    const bool bad_offs = e <= b || e > n_idx;
    const uint32_t L = bad_offs ? 0 : e - b;
    bool badc = false;
    for (uint32_t k = b + lane; k < b + L; k += 32) badc |= __ldg(cols + k) >= n_cols;
    if (__any_sync(kFull, bad_offs || badc)) {
      before_store();
      if (lane == 0) {
        out[i] = 0;
        *err_out = bad_offs ? 2 : 1;
      }
      continue;
    }
    if (L == 1) {  // no pair: every row supports (the trend.cpp:19 loop never runs)
      before_store();
      if (lane == 0) out[i] = n_rows;
      if (MASK)
        for (uint32_t w = lane; w < mask_wpc; w += 32)
          mask[(uint64_t)i * mask_wpc + w] = index_to_natural(index_valid_bits(n_rows, w));
      continue;
    }
    // the candidate's columns, 32 at a time in lane registers (shuffled out per pair)
    const uint32_t c_lane = lane < L ? __ldg(cols + b + lane) : 0u;
    // LAZY: pool slots of the candidate's first 31 forward / reversed pairs
    // (pair lane -> lane + 1), looked up once for all passes
    uint32_t sf_lane = kSlotEmpty, sr_lane = kSlotEmpty;
    if (LAZY) {
      // the slots lazy_claim_kernel recorded for the first 31 pairs (claimed
      // ones are built by now); the later pairs are looked up in the map
      bool ready = true;
      if (lane < 31 && (uint32_t)lane + 1 < L) {
        sf_lane = __ldg(la.pslot + (uint64_t)i * 64 + lane);
        if (NEG) sr_lane = __ldg(la.pslot + (uint64_t)i * 64 + 32 + lane);
        ready = slot_ready(sf_lane) && (!NEG || slot_ready(sr_lane));
      }
      for (uint32_t k = 32 + lane; k < L; k += 32) {  // pairs past the lanes
        const uint32_t x = __ldg(cols + b + k - 1), y = __ldg(cols + b + k);
        ready = ready && slot_ready(lazy_lookup(la, (uint64_t)x * n_cols + y)) &&
                (!NEG || slot_ready(lazy_lookup(la, (uint64_t)y * n_cols + x)));
      }
      if (!NEG) ready = ready && L <= 32;  // (the pipelined loop takes every slot from a lane register)
      if (!__all_sync(kFull, ready)) {
        before_store();
        if (lane == 0) la.defer[1 + atomicAdd(la.defer, 1u)] = i;
        continue;
      }
    }
    if constexpr (MULTI && !NEG) {
      // Software-pipelined over the candidate's pairs: pair k + 1's J loads are
      // in flight while pair k is combined.  (The plain loop below kept only
      // ~3 of its 8 loads in flight when fed from lazy pool slots -- ptxas
      // reused their registers -- and ran C4 at 0.58 ms; pipelined, the lazy
      // pool runs at 0.41 ms.)
      // base of pair k's vector (pair k joins columns k - 1 and k)
      auto col = [&](uint32_t j) -> uint32_t { return j < 32 ? __shfl_sync(kFull, c_lane, j & 31) : __ldg(cols + b + j); };
      auto vec = [&](uint32_t k) -> const uint4* {
        if constexpr (LAZY) return t4 + (uint64_t)__shfl_sync(kFull, sf_lane, (k - 1) & 31) * nv;
        else return t4 + ((uint64_t)col(k - 1) * n_cols + col(k)) * nv;
      };
      uint32_t n = 0;
      for (uint32_t v0 = 0; v0 < nv; v0 += 32 * J) {
        uint32_t vv[J];
#pragma unroll
        for (int u = 0; u < J; ++u) vv[u] = min(v0 + u * 32 + lane, nv - 1);
        uint4 f[J], xa[J];
#pragma unroll
        for (int u = 0; u < J; ++u) f[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
        {
          const uint4* p0 = vec(1);
#pragma unroll
          for (int u = 0; u < J; ++u) xa[u] = __ldg(p0 + vv[u]);
        }
        for (uint32_t k = 1; k + 1 < L; ++k) {
          const uint4* pn = vec(k + 1);
          uint4 xb[J];
#pragma unroll
          for (int u = 0; u < J; ++u) xb[u] = __ldg(pn + vv[u]);
#pragma unroll
          for (int u = 0; u < J; ++u) {
            f[u].x &= xa[u].x; f[u].y &= xa[u].y; f[u].z &= xa[u].z; f[u].w &= xa[u].w;
            xa[u] = xb[u];
          }
        }
        before_store();
#pragma unroll
        for (int u = 0; u < J; ++u) {
          f[u].x &= xa[u].x; f[u].y &= xa[u].y; f[u].z &= xa[u].z; f[u].w &= xa[u].w;
          const uint32_t v = v0 + u * 32 + lane;
          const uint4 s = v < nv ? f[u] : make_uint4(0u, 0u, 0u, 0u);
          n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
          if (MASK && v < nv) {
            uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
            const uint32_t words[4] = {index_to_natural(s.x), index_to_natural(s.y), index_to_natural(s.z),
                                       index_to_natural(s.w)};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (4 * v + q < mask_wpc) mw[q] = words[q];
          }
        }
      }
      n = __reduce_add_sync(kFull, n);
      if (lane == 0) out[i] = n;
      continue;
    }
    uint32_t n = 0;
    // MULTI: vectors longer than 32 J slices are swept in passes of 32 J
    for (uint32_t v0 = 0; v0 < (MULTI ? nv : 1u); v0 += 32 * J) {
      uint4 f[J], r[J];  // all-ones: the index has no bits past the last row
#pragma unroll
      for (int u = 0; u < J; ++u) {
        f[u] = make_uint4(~0u, ~0u, ~0u, ~0u);
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
        if constexpr (LAZY) {
          uint32_t sf = k - 1 < 31 ? __shfl_sync(kFull, sf_lane, (k - 1) & 31)
                                   : lazy_lookup(la, (uint64_t)cp * n_cols + cc);
          uint32_t sr = !NEG ? 0u : k - 1 < 31 ? __shfl_sync(kFull, sr_lane, (k - 1) & 31)
                                              : lazy_lookup(la, (uint64_t)cc * n_cols + cp);
          sf = __shfl_sync(kFull, sf, 0);  // one view per warp
          sr = __shfl_sync(kFull, sr, 0);
#pragma unroll
          for (int u = 0; u < J; ++u) {
            const uint32_t v = min(v0 + u * 32 + lane, nv - 1);
            // (every pair is ready: checked above.  A slot's bits never change
            // while it is ready, so the read-only path is safe for them.)
            x[u] = __ldg(t4 + (uint64_t)sf * nv + v);
            if (NEG) y[u] = __ldg(t4 + (uint64_t)sr * nv + v);
          }
        } else if constexpr (MULTI) {
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
      before_store();
#pragma unroll
      for (int u = 0; u < J; ++u) {
        const uint32_t v = v0 + u * 32 + lane;
        const uint4 o = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
        const uint4 s = v < nv ? o : make_uint4(0u, 0u, 0u, 0u);  // (clamped re-reads past the vector)
        n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
        if (MASK && v < nv) {
          uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
          const uint32_t words[4] = {index_to_natural(s.x), index_to_natural(s.y), index_to_natural(s.z),
                                     index_to_natural(s.w)};
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


// Tiny vectors (nv <= 32 uint4 slices: R <= 4096 rows): a GROUP of GL lanes
// per candidate (32 / GL candidates per warp), lane s of the group owning
// slices s, s + GL, ... (J of them) of every pair vector.  A 128-B vector
// (R = 1000) is then one 16-B load per lane instead of a whole warp's bulk
// copy and mbarrier round trip; U pairs' loads are issued before they are
// combined, and the next candidate's offsets load while this one runs.  The
// index is small enough to sit in L2 (64^2 x 128 B = 512 KB at 1000 rows), so
// the kernel is bound by L2 latency and issue, not HBM.  Counts and error
// codes as table_count_kernel; no masks, no lazy index.
template <int GL, int J, int U, bool NEG>
__global__ void __launch_bounds__(256)
table_count_group_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                         const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                         uint32_t n_idx, uint32_t* __restrict__ out, int* err_out) {
  static_assert(GL >= 1 && GL <= 32 && (GL & (GL - 1)) == 0, "group size is a power of two");
  constexpr int CPW = 32 / GL;  // candidates per warp
  const int lane = threadIdx.x & 31, s = lane % GL;
  const uint32_t nv = wp / 4;
  uint32_t sl[J];
#pragma unroll
  for (int j = 0; j < J; ++j) sl[j] = min((uint32_t)(s + j * GL), nv - 1);  // past the vector: re-read (dropped)
  const uint4* t4 = reinterpret_cast<const uint4*>(table);
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x / 32) * CPW;
  uint64_t i0 = ((uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * CPW;
  auto load_offs = [&](uint64_t i, uint32_t& b, uint32_t& e) {
    b = i < n_cand ? __ldg(offs + i) : 0u;
    e = i < n_cand ? __ldg(offs + i + 1) : 0u;
  };
  uint32_t b, e;
  load_offs(i0 + lane / GL, b, e);
  pdl_trigger();
  bool dep_done = false;  // griddepcontrol.wait issued (before this warp's first store)
  for (; i0 < n_cand; i0 += stride) {
    const uint64_t i = i0 + lane / GL;
    const bool live = i < n_cand;
    uint32_t bn, en;  // the next candidate's offsets, in flight during this one
    load_offs(i + stride, bn, en);
    const bool bad_offs = live && (e <= b || e > n_idx);
    const uint32_t L = (live && !bad_offs) ? e - b : 0u;
    uint4 f[J], r[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      f[j] = make_uint4(~0u, ~0u, ~0u, ~0u);
      r[j] = NEG ? f[j] : make_uint4(0u, 0u, 0u, 0u);
    }
    bool badc = false;
    uint32_t cp = L ? __ldg(cols + b) : 0u;
    badc |= L && cp >= n_cols;
    // the warp runs to its longest candidate; shorter groups are predicated off
    uint32_t Lmax = L;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) Lmax = max(Lmax, __shfl_xor_sync(kFull, Lmax, o));
    for (uint32_t k0 = 1; k0 < Lmax; k0 += U) {
      uint32_t cc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cc[u] = k0 + u < L ? __ldg(cols + b + k0 + u) : 0u;
      uint4 x[U][J], y[U][J];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t a = u == 0 ? cp : cc[u - 1];
        const bool ok = k0 + u < L && a < n_cols && cc[u] < n_cols;
        badc |= k0 + u < L && cc[u] >= n_cols;
        const uint64_t pf = ok ? (uint64_t)a * n_cols + cc[u] : 0u, pr = ok ? (uint64_t)cc[u] * n_cols + a : 0u;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          x[u][j] = __ldg(t4 + pf * nv + sl[j]);
          if (NEG) y[u][j] = __ldg(t4 + pr * nv + sl[j]);
          if (!ok) {
            x[u][j] = make_uint4(~0u, ~0u, ~0u, ~0u);
            y[u][j] = x[u][j];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          f[j].x &= x[u][j].x; f[j].y &= x[u][j].y; f[j].z &= x[u][j].z; f[j].w &= x[u][j].w;
          if (NEG) {
            r[j].x &= y[u][j].x; r[j].y &= y[u][j].y; r[j].z &= y[u][j].z; r[j].w &= y[u][j].w;
          }
        }
      }
      cp = cc[U - 1];  // (past the candidate's end the pairs are predicated off)
    }
    uint32_t n = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint4 o = NEG ? make_uint4(f[j].x | r[j].x, f[j].y | r[j].y, f[j].z | r[j].z, f[j].w | r[j].w) : f[j];
      if ((uint32_t)(s + j * GL) < nv) n += __popc(o.x) + __popc(o.y) + __popc(o.z) + __popc(o.w);
    }
#pragma unroll
    for (int w = GL / 2; w >= 1; w >>= 1) n += __shfl_xor_sync(kFull, n, w);
    if (!dep_done) {
      pdl_wait();
      dep_done = true;
    }
    if (live && s == 0) {
      if (bad_offs || badc) {  // (every lane of a group loads the same columns: same flags)
        out[i] = 0;
        *err_out = bad_offs ? 2 : 1;
      } else {
        out[i] = L == 1 ? n_rows : n;
      }
    }
    b = bn;
    e = en;
  }
}

// TMA variant of the warp-per-candidate kernel (short vectors, nv <= 256
// slices).  One elected lane issues a bulk copy (cp.async.bulk, the TMA
// engine) per pair vector -- S pairs at a time, into the warp's shared-memory
// slots -- that completes on the warp's mbarrier; the lanes then read their
// slices from shared memory.  The HBM requests of all S pairs are in flight at
// once with no registers tied up (the register-load version is at the mercy
// of ptxas interleaving its loads with the ANDs), and a 2.5-KB pair vector is
// one copy instruction instead of 160 vector loads.
constexpr int kTmaWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}


// LAZY: the vectors come from the lazy index (ebic_lazy.cuh) -- the pair's
// slot is looked up in la.map (for a candidate's first 31 pairs, one lookup
// per lane, prefetched with the candidate's columns); a ready slot is copied
// from la.pool by TMA like a full-index vector; a missing one is built by the
// warp straight into its shared-memory slot (and, if the warp wins the pool
// slot, written to the pool and published for every later candidate).
template <int J, int S, bool NEG, bool MASK, bool LAZY = false>
__global__ void __launch_bounds__(kTmaWarps * 32)
table_count_tma_kernel(const uint32_t* __restrict__ table, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                       const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs, uint32_t n_cand,
                       uint32_t n_idx, uint32_t* __restrict__ out, int* err_out, uint32_t* __restrict__ mask,
                       uint64_t mask_wpc, LazyArgs la) {
  extern __shared__ __align__(128) unsigned char smem[];  // [warp][S (x2 with NEG)][pair vector]
  __shared__ __align__(8) uint64_t s_bar[kTmaWarps];    // "full": the slots' bulk copies have landed
  __shared__ __align__(8) uint64_t s_empty[kTmaWarps];  // "empty": all 32 lanes are done reading the slots
  constexpr int NS = NEG ? 2 * S : S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nv = wp / 4, slot = wp * 4;  // uint4 / bytes per pair vector
  const uint32_t my = smem_u32(smem) + (uint32_t)warp * NS * slot;
  const uint32_t bar = smem_u32(&s_bar[warp]), empty = smem_u32(&s_empty[warp]);
  const uint32_t* vec_base = LAZY ? la.pool : table;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init(empty, 32);
  }
  if (LAZY && la.count_out && blockIdx.x == 0 && threadIdx.x == 0) {  // the host's lagged view of the pool's fill
    la.count_out[0] = *(volatile uint32_t*)la.count;
    __threadfence_system();
    la.count_out[1] = la.seq;
  }
  __syncwarp();
  pdl_trigger();
  bool dep_done = false;  // griddepcontrol.wait issued (before this warp's first store)
  auto before_store = [&]() {
    if (!dep_done) {
      pdl_wait();
      dep_done = true;
    }
  };
  // LAZY: slots of pair (position lane -> lane + 1) of a candidate, looked up
  // as soon as its columns are known (clamped: columns are validated later)
  auto lookup = [&](uint32_t c_l, uint32_t L, uint32_t& sf, uint32_t& sr) {
    sf = sr = kSlotEmpty;
    if (!LAZY) return;
    const uint32_t c_n = __shfl_down_sync(kFull, c_l, 1);
    if (lane < 31 && lane + 1 < L) {
      const uint32_t x = min(c_l, n_cols - 1), y = min(c_n, n_cols - 1);
      sf = lazy_lookup(la, (uint64_t)x * n_cols + y);
      if (NEG) sr = lazy_lookup(la, (uint64_t)y * n_cols + x);
    }
  };
  uint32_t phase = 0, ephase = 0;
  // Persistent warps, software-pipelined over candidates: the next candidate's
  // offsets are loaded at the top of an iteration and its columns once the
  // first bulk copies have landed, so the offsets -> columns -> pair vectors
  // chain of one candidate overlaps the previous candidate's copies.
  const uint32_t warps = gridDim.x * kTmaWarps;
  uint32_t i = blockIdx.x * kTmaWarps + warp;
  uint32_t b = 0, e = 0, c_lane = 0, sf_lane = kSlotEmpty, sr_lane = kSlotEmpty;
  if (i < n_cand) {
    b = __ldg(offs + i);
    e = __ldg(offs + i + 1);
    const uint32_t L0 = (e > b && e <= n_idx) ? e - b : 0u;
    c_lane = lane < L0 ? __ldg(cols + b + lane) : 0u;
    lookup(c_lane, L0, sf_lane, sr_lane);
  }
  for (; i < n_cand; i += warps) {
    const uint32_t inext = i + warps;
    uint32_t bn = 0, en = 0, cn = 0, sfn = kSlotEmpty, srn = kSlotEmpty;
    bool next_cols = false;
    if (inext < n_cand) {  // in flight while this candidate is processed
      bn = __ldg(offs + inext);
      en = __ldg(offs + inext + 1);
    }
    auto fetch_next_cols = [&]() {
      if (next_cols) return;
      next_cols = true;
      const uint32_t Ln = (inext < n_cand && en > bn && en <= n_idx) ? en - bn : 0u;
      cn = lane < Ln ? __ldg(cols + bn + lane) : 0u;
      lookup(cn, Ln, sfn, srn);
    };
    do {  // one candidate; `break` = done with it
    const bool bad_offs = e <= b || e > n_idx;
    const uint32_t L = bad_offs ? 0 : e - b;
    bool badc = lane < L && c_lane >= n_cols;
    for (uint32_t k = b + 32 + lane; k < b + L; k += 32) badc |= __ldg(cols + k) >= n_cols;
    if (__any_sync(kFull, bad_offs || badc)) {
      before_store();
      if (lane == 0) {
        out[i] = 0;
        *err_out = bad_offs ? 2 : 1;
      }
      break;
    }
    if (L == 1) {  // no pair: every row supports (the trend.cpp:19 loop never runs)
      before_store();
      if (lane == 0) out[i] = n_rows;
      if (MASK)
        for (uint32_t w = lane; w < mask_wpc; w += 32)
          mask[(uint64_t)i * mask_wpc + w] = index_to_natural(index_valid_bits(n_rows, w));
      break;
    }
    uint4 f[J], r[J];
#pragma unroll
    for (int u = 0; u < J; ++u) {
      f[u] = make_uint4(~0u, ~0u, ~0u, ~0u);  // the index has no bits past the last row
      r[u] = NEG ? f[u] : make_uint4(0u, 0u, 0u, 0u);
    }
    uint32_t cp = __shfl_sync(kFull, c_lane, 0);
    for (uint32_t k0 = 1; k0 < L; k0 += S) {
      const uint32_t g = min((uint32_t)S, L - k0);  // pairs in this group (warp-uniform)
      uint32_t pc[S + 1];
      pc[0] = cp;
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t k = k0 + q;
        pc[q + 1] = k < 32 ? __shfl_sync(kFull, c_lane, k & 31) : (k < L ? __ldg(cols + b + k) : 0u);
      }
      // vector index of each pair of the group: a*C + b (full index) or the
      // pool slot (LAZY; kSlotEmpty / busy = build it here)
      uint32_t vf[S], vr[S];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t k = k0 + q;
        if (LAZY) {
          const bool in_lane = k - 1 < 31;
          const uint32_t x = __shfl_sync(kFull, sf_lane, (k - 1) & 31);
          const uint32_t y = __shfl_sync(kFull, sr_lane, (k - 1) & 31);
          vf[q] = in_lane ? x : (k < L ? lazy_lookup(la, (uint64_t)pc[q] * n_cols + pc[q + 1]) : 0u);
          vr[q] = !NEG ? 0u : in_lane ? y : (k < L ? lazy_lookup(la, (uint64_t)pc[q + 1] * n_cols + pc[q]) : 0u);
          // one view per warp: lanes loading the same entry while another warp
          // publishes it could disagree, and the code below is warp-collective
          vf[q] = __shfl_sync(kFull, vf[q], 0);
          vr[q] = __shfl_sync(kFull, vr[q], 0);
        } else {
          vf[q] = pc[q] * n_cols + pc[q + 1];
          vr[q] = pc[q + 1] * n_cols + pc[q];
        }
      }
      if (lane == 0) {
        uint32_t bytes = 0;
#pragma unroll
        for (int q = 0; q < S; ++q)
          if ((uint32_t)q < g) bytes += (slot_ready(vf[q]) || !LAZY ? slot : 0u) + (NEG && (slot_ready(vr[q]) || !LAZY) ? slot : 0u);
        if (LAZY) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic writes to the slots
        mbar_expect_tx(bar, bytes);
#pragma unroll
        for (int q = 0; q < S; ++q) {
          if ((uint32_t)q < g) {
            if (!LAZY || slot_ready(vf[q])) bulk_g2s(my + q * slot, vec_base + (uint64_t)vf[q] * wp, slot, bar);
            if (NEG && (!LAZY || slot_ready(vr[q])))
              bulk_g2s(my + (S + q) * slot, vec_base + (uint64_t)vr[q] * wp, slot, bar);
          }
        }
      }
      if (LAZY) {
        // vectors not in the pool yet: built by the warp into their slots
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          const bool rev = q >= S;
          const int qq = rev ? q - S : q;
          if ((uint32_t)qq >= g) continue;
          const uint32_t v = rev ? vr[qq] : vf[qq];
          if (slot_ready(v)) continue;
          const uint32_t pa = rev ? pc[qq + 1] : pc[qq], pb = rev ? pc[qq] : pc[qq + 1];
          const uint64_t key = (uint64_t)pa * n_cols + pb;
          uint32_t cl = kSlotEmpty;
          if (v == kSlotEmpty && lane == 0) cl = lazy_claim(la, key);
          cl = __shfl_sync(kFull, cl, 0);
          const uint32_t dst = my + q * slot;
          build_pair_vector_warp(la, n_rows, pa, pb, wp, lane, [&](uint32_t w, uint32_t word) { sts_u32(dst + 4 * w, word); });
          if (cl != kSlotEmpty) {  // this warp owns the pool slot: copy the vector there and publish it
            const uint32_t sl = cl & ~kSlotBusy;
            __syncwarp();
            uint4* dst_g = reinterpret_cast<uint4*>(la.pool + (uint64_t)sl * wp);
            for (uint32_t t = lane; t < nv; t += 32) dst_g[t] = lds<uint4>(dst + 16 * t);
            lazy_publish(la, key, sl, lane);
          }
        }
        __syncwarp();
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
      fetch_next_cols();  // the next candidate's offsets have arrived by now
#pragma unroll
      for (int q = 0; q < S; ++q) {
        if ((uint32_t)q < g) {
#pragma unroll
          for (int u = 0; u < J; ++u) {
            // (the last group of slices: lanes past the vector re-read its
            // last slice instead of another slot; their result is dropped)
            const uint32_t v = u == J - 1 ? min((uint32_t)(u * 32 + lane), nv - 1) : u * 32 + lane;
            const uint4 x = lds<uint4>(my + q * slot + v * 16);
            f[u].x &= x.x; f[u].y &= x.y; f[u].z &= x.z; f[u].w &= x.w;
            if (NEG) {
              const uint4 y = lds<uint4>(my + (S + q) * slot + v * 16);
              r[u].x &= y.x; r[u].y &= y.y; r[u].z &= y.z; r[u].w &= y.w;
            }
          }
        }
      }
#pragma unroll
      for (int q = 1; q <= S; ++q)
        if ((uint32_t)q == g) cp = pc[q];
      // release the slots: every lane arrives once its reads are done; the
      // issuing lane waits for all 32 before the next bulk copies refill them
      // (the canonical consumer-release / producer-acquire handshake)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty) : "memory");
      if (lane == 0) mbar_wait(empty, ephase);
      ephase ^= 1u;
      __syncwarp();
    }
    uint32_t n = 0;
    before_store();
#pragma unroll
    for (int u = 0; u < J; ++u) {
      const uint32_t v = u * 32 + lane;
      const uint4 o = NEG ? make_uint4(f[u].x | r[u].x, f[u].y | r[u].y, f[u].z | r[u].z, f[u].w | r[u].w) : f[u];
      const uint4 s = v < nv ? o : make_uint4(0u, 0u, 0u, 0u);  // (lanes past a short vector)
      n += __popc(s.x) + __popc(s.y) + __popc(s.z) + __popc(s.w);
      if (MASK && v < nv) {
        uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
        const uint32_t words[4] = {index_to_natural(s.x), index_to_natural(s.y), index_to_natural(s.z),
                                   index_to_natural(s.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (4 * v + q < mask_wpc) mw[q] = words[q];
      }
    }
    n = __reduce_add_sync(kFull, n);
    if (lane == 0) out[i] = n;
    } while (false);
    fetch_next_cols();
    b = bn;
    e = en;
    c_lane = cn;
    sf_lane = sfn;
    sr_lane = srn;
  }
}

// The candidates the count kernel deferred (a pair not ready in the pool):
// a warp per candidate, one uint4 slice per lane at a time, ready pairs from
// the pool and the others computed from the value store (pair_slice_thread).
// Rare (a full pool, or batches on several streams sharing pairs), so simple.
template <bool NEG, bool MASK>
__global__ void __launch_bounds__(256)
lazy_deferred_kernel(const LazyArgs la, uint32_t n_cols, uint32_t wp, uint32_t n_rows,
                     const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs,
                     uint32_t* __restrict__ out, uint32_t* __restrict__ mask, uint64_t mask_wpc) {
  const uint32_t n_def = *(volatile uint32_t*)la.defer;
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint32_t nv = wp / 4;
  const uint4* p4 = reinterpret_cast<const uint4*>(la.pool);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n_def; d += warps) {
    const uint32_t i = la.defer[1 + d];
    const uint32_t b = __ldg(offs + i), L = __ldg(offs + i + 1) - b;  // (validated by the count kernel)
    uint32_t n = 0;
    for (uint32_t v0 = 0; v0 < nv; v0 += 32) {
      const uint32_t v = min(v0 + lane, nv - 1);
      uint4 f = make_uint4(~0u, ~0u, ~0u, ~0u), r = NEG ? f : make_uint4(0u, 0u, 0u, 0u);
      uint32_t cp = __ldg(cols + b);
      for (uint32_t k = 1; k < L; ++k) {
        const uint32_t cc = __ldg(cols + b + k);
        const uint32_t sf = lazy_lookup(la, (uint64_t)cp * n_cols + cc);
        const uint4 x = slot_ready(sf) ? __ldcg(p4 + (uint64_t)sf * nv + v) : pair_slice_thread(la, n_rows, cp, cc, v);
        f.x &= x.x; f.y &= x.y; f.z &= x.z; f.w &= x.w;
        if (NEG) {
          const uint32_t sr = lazy_lookup(la, (uint64_t)cc * n_cols + cp);
          const uint4 y = slot_ready(sr) ? __ldcg(p4 + (uint64_t)sr * nv + v) : pair_slice_thread(la, n_rows, cc, cp, v);
          r.x &= y.x; r.y &= y.y; r.z &= y.z; r.w &= y.w;
        }
        cp = cc;
      }
      const uint4 o = NEG ? make_uint4(f.x | r.x, f.y | r.y, f.z | r.z, f.w | r.w) : f;
      if (v0 + lane < nv) {
        n += __popc(o.x) + __popc(o.y) + __popc(o.z) + __popc(o.w);
        if (MASK) {
          uint32_t* mw = mask + (uint64_t)i * mask_wpc + 4 * v;
          const uint32_t words[4] = {index_to_natural(o.x), index_to_natural(o.y), index_to_natural(o.z),
                                     index_to_natural(o.w)};
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
