// ebic_simd.cuh -- two rows per 32-bit word: the packed-rank slab kernel.
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

// Fixed-length body: L vector loads (both words of every column), then the
// L-1 forward tests Rg(c_k) + NT(c_{k-1}) (and reversed Rg(c_{k-1}) + NT(c_k)).
// Returns the guard bits of the lane's row pairs that support the candidate.
template <int L, int P, bool NEG, uint32_t COLSHIFT>
__device__ __forceinline__ typename PairVec<P>::M simd_eval(uint32_t lane_base, const uint4& rec,
                                                          typename PairVec<P>::M vmask) {
  using V = typename PairVec<P>::V;
  using M = typename PairVec<P>::M;
  const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                 hi16(rec.z), lo16(rec.w), hi16(rec.w)};
  V w[L];
#pragma unroll
  for (int k = 0; k < L; ++k) w[k] = lds<V>(lane_base + (cc[k] << COLSHIFT));
  M f = vmask;
#pragma unroll
  for (int k = 1; k < L; ++k) and_pair<P>(f, w[k], w[k - 1]);
  if constexpr (NEG) {
    M r = vmask;
#pragma unroll
    for (int k = 1; k < L; ++k) and_pair<P>(r, w[k - 1], w[k]);
    or_into<P>(f, r);
  }
  return f;
}

template <int P, int SUB, bool NEG, int L, uint32_t COLSHIFT>
__device__ __forceinline__ void simd_sweep_class(const SlabArgs& a, uint32_t sa_rec, uint32_t lane_base,
                                                 uint32_t* s_cnt, uint32_t n_padded, uint32_t class_base,
                                                 uint32_t c_begin, typename PairVec<P>::M vmask, int warp,
                                                 int lane, int sub) {
  using V = typename PairVec<P>::V;
  using M = typename PairVec<P>::M;
  constexpr int LPC = 32 / SUB;
  constexpr uint32_t stride = kSlabWarps * SUB;
  for (uint32_t t = warp * SUB + sub; t < n_padded; t += stride) {
    const uint4 rec = lds<uint4>(sa_rec + (class_base + t) * 16);
    const uint32_t j = lo16(rec.x);
    M ok;
    if constexpr (L == 1) {
      ok = vmask;  // no pair: every row supports (the trend.cpp:19 loop never runs)
    } else if constexpr (L < 8) {
      ok = simd_eval<L, P, NEG, COLSHIFT>(lane_base, rec, vmask);
    } else {
      // >= 8 columns: first 7 from the record, the tail from the CSR
      const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                     hi16(rec.z), lo16(rec.w), hi16(rec.w)};
      M f = vmask, r = NEG ? vmask : M{};
      V wp = lds<V>(lane_base + (cc[0] << COLSHIFT));
      auto step = [&](uint32_t col) {
        const V wc = lds<V>(lane_base + (col << COLSHIFT));
        and_pair<P>(f, wc, wp);
        if (NEG) and_pair<P>(r, wp, wc);
        wp = wc;
      };
#pragma unroll
      for (int k = 1; k < kRecCols; ++k) step(cc[k]);
      if (j < a.chunk) {
        // the tail in blocks of TB columns: TB independent index loads, then TB
        // shared loads, then the pair tests (no load-to-load dependency chain)
        constexpr int TB = P == 1 ? 8 : (NEG ? 2 : 4);  // register budget: 64 per thread
        const uint32_t b = a.offs[c_begin + j], e = a.offs[c_begin + j + 1];
        for (uint32_t k0 = b + kRecCols; k0 < e; k0 += TB) {
          uint32_t any = 0;
#pragma unroll
          for (int q = 0; q < P; ++q) any |= wget(f, q) | wget(r, q);
          if (!any) break;  // this lane's rows are all decided
          uint32_t idx[TB];
#pragma unroll
          for (int i = 0; i < TB; ++i) idx[i] = k0 + i < e ? __ldg(a.cols + k0 + i) : 0u;
          V wv[TB];
#pragma unroll
          for (int i = 0; i < TB; ++i) wv[i] = lds<V>(lane_base + (idx[i] << COLSHIFT));
#pragma unroll
          for (int i = 0; i < TB; ++i) {
            if (k0 + i < e) {
              and_pair<P>(f, wv[i], wp);
              if (NEG) and_pair<P>(r, wp, wv[i]);
              wp = wv[i];
            }
          }
        }
      }
      if (NEG) or_into<P>(f, r);
      ok = f;
    }
    // count: per-lane popcount, summed per candidate with ONE REDUX for all SUB
    // candidates of the warp: candidate `sub` owns bit field [sub*FW, (sub+1)*FW)
    // (a slab count is <= RT = 2*P*LPC rows, which fits its field)
    constexpr uint32_t FW = 32 / SUB;
    static_assert(SUB == 1 || (2u * P * LPC) < (1u << FW), "count field too narrow");
    const uint32_t n = popc_words<P>(ok) << (FW * sub);
    const uint32_t tot = __reduce_add_sync(kFull, n);
    if (lane % LPC == 0)
      atomicAdd(&s_cnt[j], SUB == 1 ? tot : (tot >> (FW * sub)) & ((1u << (FW % 32)) - 1u));
  }
}

template <int P, int SUB, bool NEG>
__global__ void __launch_bounds__(kSlabThreads, 1)
slab_simd_kernel(const SlabArgs a) {
  using M = typename PairVec<P>::M;
  constexpr int LPC = 32 / SUB;
  constexpr uint32_t RT = LPC * 2 * P;             // rows per slab
  constexpr uint32_t CW = RT;                      // words per column line: RT/2 x (Rg, NT)
  constexpr uint32_t COLSHIFT = CW == 16 ? 6 : CW == 32 ? 7 : CW == 64 ? 8 : CW == 128 ? 9 : 10;  // log2(CW*4)
  static_assert((1u << COLSHIFT) == CW * 4, "column stride must be a power of two");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(smem_raw);               // [C][RT/2 x (Rg, NT)]
  uint4* s_rec = reinterpret_cast<uint4*>(s_slab + (size_t)a.n_cols * CW);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_rec + a.chunk + kClasses * kSlabWarps * SUB);
  __shared__ uint32_t s_hist[kClasses], s_base[kClasses], s_fill[kClasses];
  const uint32_t sa_slab = (uint32_t)__cvta_generic_to_shared(s_slab);
  const uint32_t sa_rec = (uint32_t)__cvta_generic_to_shared(s_rec);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPC, rl = lane % LPC;
  const uint32_t lane_base = sa_slab + rl * P * 8;  // this lane's (Rg, NT) pair(s) in column 0
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
    __syncthreads();
    if (chunk != cur_chunk) {
      flush();
      cur_chunk = chunk;
      c_begin = chunk * a.chunk;
      c_n = min(a.chunk, a.n_cand - c_begin);
      pack_chunk<kSlabWarps * SUB>(a, c_begin, c_n, s_rec, s_cnt, s_hist, s_base, s_fill);
    }
    // stage + repack: each thread takes 4 consecutive rows (one uint4 of plane
    // words) of one column -> 2 row pairs -> 4 words (Rg, NT, Rg, NT) of the line;
    // a round of UNR loads is in flight before any store
    {
      constexpr uint32_t Q = RT / 4;  // uint4 per column
      constexpr int UNR = 4;
      const uint32_t total = a.n_cols * Q;
      const uint4* src = reinterpret_cast<const uint4*>(a.plane);
      const uint64_t ld4 = a.ld / 4, r4 = row0 / 4;
      for (uint32_t t0 = threadIdx.x; t0 < total; t0 += UNR * blockDim.x) {
        uint4 w[UNR];
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t t = t0 + k * blockDim.x;
          if (t < total) w[k] = __ldg(src + (uint64_t)(t / Q) * ld4 + r4 + t % Q);
        }
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t t = t0 + k * blockDim.x;
          if (t < total) {
            const uint32_t c = t / Q, q = t % Q;
            *reinterpret_cast<uint4*>(s_slab + (size_t)c * CW + 4 * q) = stage_pairs<P>(w[k]);
          }
        }
      }
    }
    __syncthreads();
    prefetch_next_slab<RT>(a, u + 1, u_end);

    // validity guard bits of this lane's row pairs (rows beyond n_rows never count)
    const uint32_t valid_rows = min(RT, a.n_rows - row0);
    M vmask;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint32_t r = (rl * P + q) * 2;
      wref(vmask, q) = (r < valid_rows ? 0x8000u : 0u) | (r + 1 < valid_rows ? 0x80000000u : 0u);
    }

#define EBIC_SIMD_SWEEP(L)                                                                                      \
  simd_sweep_class<P, SUB, NEG, L, COLSHIFT>(a, sa_rec, lane_base, s_cnt, s_hist[L], s_base[L], c_begin, vmask, \
                                             warp, lane, sub)
    EBIC_SIMD_SWEEP(4);
    EBIC_SIMD_SWEEP(3);
    EBIC_SIMD_SWEEP(5);
    EBIC_SIMD_SWEEP(2);
    EBIC_SIMD_SWEEP(6);
    EBIC_SIMD_SWEEP(7);
    EBIC_SIMD_SWEEP(8);
    EBIC_SIMD_SWEEP(1);
#undef EBIC_SIMD_SWEEP
  }
  __syncthreads();
  flush();
}

}  // namespace ebic
