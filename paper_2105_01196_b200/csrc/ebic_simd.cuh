// ebic_simd.cuh -- two rows per 32-bit word: the packed-rank-pair helpers of
// the slab kernel (slab_pair_kernel, ebic_pair.cuh).
//
// Same rank-plane test as slab_count_kernel (R(y) > T(x) <=> v_y > thr(v_x),
// see ebic_plane.cuh), but each slab column is restaged as 16-bit row PAIRS:
//   Rg[i] = (R(2i) | 0x8000) | (R(2i+1) | 0x8000) << 16        ("guarded" ranks)
//   NT[i] = 0 - (T(2i) | T(2i+1) << 16) - 0x00010001            (negated thresholds)
// For a consecutive pair (p, c) of a candidate, D = Rg[c] + NT[p] (mod 2^32)
// = Rg - T - 0x00010001 has bit 15 set iff R_lo(c) > T_lo(p) and bit 31 set
// iff R_hi(c) > T_hi(p): the guard bit absorbs the borrow, so the halves never
// interact (R, T <= C <= 8192 < 2^15).  One IADD tests two rows; AND-ing the
// D's of all pairs and keeping bits 15/31 gives the verdict of both rows.
//
// Lane mapping: LPC = 32/SUB lanes per candidate, each lane owns P row pairs
// (2P rows), so a slab holds RT = LPC * 2P rows:
//   SUB=4, P=1: RT = 16  (C <= 2048)  four candidates per warp instruction
//   SUB=2, P=1: RT = 32  (C <= 1024)  two candidates per warp instruction
//   SUB=1, P=1: RT = 64  (C <= 512)
//   SUB=1, P=2: RT = 128 (C <= 256)
// Shared memory: one line per column with the row pairs interleaved,
// [Rg_0 NT_0 Rg_1 NT_1 ...] at P=1, [Rg_0 Rg_1 NT_0 NT_1 ...] per lane at P=2
// (see stage_pairs; 4 B per element, the same footprint as the u32
// plane).  A lane fetches both words of its row pair(s) of a column with ONE
// LDS.64 (P=1) / LDS.128 (P=2).  At SUB=2 each half-warp reads one whole,
// aligned 128-B line per load: 2 wavefronts for 256 B, the minimum -- no bank
// conflicts for any pair of columns.
#pragma once
#include <cstdint>

#include "ebic_plane.cuh"

namespace ebic {

// Per-lane slab data: P row pairs x (Rg, NT) words; per-lane verdict: P words.
template <int P> struct PairVec;
template <> struct PairVec<1> { using V = uint2; using M = uint32_t; };
template <> struct PairVec<2> { using V = uint4; using M = uint2; };

__device__ __forceinline__ uint32_t& wref(uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t& wref(uint2& v, int q) { return q ? v.y : v.x; }
__device__ __forceinline__ uint32_t wget(const uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t wget(const uint2& v, int q) { return q ? v.y : v.x; }
__device__ __forceinline__ uint32_t wget(const uint4& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

// D = Rg + NT (two rows at once); keep the guard bits 15/31
__device__ __forceinline__ uint32_t sum2(uint32_t a, uint32_t b) { return (a + b) & 0x80008000u; }

// A lane's slab words for one column: P = 1: (Rg, NT); P = 2: (Rg_0, Rg_1,
// NT_0, NT_1) -- same-kind words adjacent, so that the first column of a
// candidate (NT only) and the last (Rg only) are one aligned 8-byte LDS each
// when ptxas narrows the 16-byte load, not two strided 4-byte ones (which
// would cost twice the shared-memory wavefronts).
// acc[q] &= Rg_q(rg_src) + NT_q(nt_src)
template <int P, typename M, typename V>
__device__ __forceinline__ void and_pair(M& acc, const V& rg_src, const V& nt_src) {
#pragma unroll
  for (int q = 0; q < P; ++q) wref(acc, q) &= sum2(wget(rg_src, q), wget(nt_src, P + q));
}

// Stage one uint4 of plane words (4 consecutive rows of a column) as slab
// words: two row pairs (Rg, NT) per pair for P = 1, (Rg, Rg, NT, NT) for P = 2.
template <int P>
__device__ __forceinline__ uint4 stage_pairs(const uint4& w) {
  const uint32_t rg0 = __byte_perm(w.x, w.y, 0x7632) | 0x80008000u;
  const uint32_t nt0 = 0u - __byte_perm(w.x, w.y, 0x5410) - 0x00010001u;
  const uint32_t rg1 = __byte_perm(w.z, w.w, 0x7632) | 0x80008000u;
  const uint32_t nt1 = 0u - __byte_perm(w.z, w.w, 0x5410) - 0x00010001u;
  return P == 1 ? make_uint4(rg0, nt0, rg1, nt1) : make_uint4(rg0, rg1, nt0, nt1);
}

template <int P, typename M>
__device__ __forceinline__ void or_into(M& acc, const M& x) {
#pragma unroll
  for (int q = 0; q < P; ++q) wref(acc, q) |= wget(x, q);
}

template <int P, typename M>
__device__ __forceinline__ uint32_t popc_words(const M& v) {
  uint32_t n = 0;
#pragma unroll
  for (int q = 0; q < P; ++q) n += __popc(wget(v, q));
  return n;
}

}  // namespace ebic
