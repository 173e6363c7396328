// ebic_simd.cuh -- two rows per 32-bit word: the packed-rank slab kernel.
//
// Same rank-plane test as slab_count_kernel (R(y) > T(x) <=> v_y > thr(v_x),
// see ebic_plane.cuh), but the slab is restaged as two 16-bit planes:
//   Rg[c][i] = (R(2i)   | 0x8000) | (R(2i+1) | 0x8000) << 16   ("guarded" ranks)
//   T [c][i] =  T(2i)             |  T(2i+1)           << 16
// so one 32-bit word holds a row PAIR.  For a consecutive pair (p, c) of a
// candidate, D = Rg[c] - T[p] - 0x00010001 has bit 15 set iff R_lo(c) > T_lo(p)
// and bit 31 set iff R_hi(c) > T_hi(p): the guard bit absorbs the borrow, so
// the halves never interact (R, T <= C <= 8192 < 2^15).  One IADD3 tests two
// rows; AND-ing the D's of all pairs (LOP3, 3 inputs) and keeping bits 15/31
// gives the forward verdict of both rows.  Reversed uses Rg[p] - T[c].
//
// Lane mapping: LPC = 32/SUB lanes per candidate, each lane owns P pair-words
// (2P rows), so a slab holds RT = LPC * 2P rows:
//   SUB=4, P=1: RT = 16  (C <= 2048)  four candidates per warp instruction
//   SUB=2, P=1: RT = 32  (C <= 1024)  two candidates per warp instruction
//   SUB=1, P=1: RT = 64  (C <= 512)
//   SUB=1, P=2: RT = 128 (C <= 256)
// Shared memory: an Rg plane [C][RT/2 words] and a T plane [C][RT/2 words]
// (== 4 B per element, the same as the u32 plane), so the slab footprint is
// unchanged while each lane does half the instructions per row.  Separate
// planes (rather than one [Rg|T] line per column, which would put every
// candidate's Rg in the same banks) make the SUB candidates of one LDS collide
// only when their columns share a bank group: ~1.5 wavefronts per load at
// SUB=2, ~2 at SUB=4.
#pragma once
#include <cstdint>

#include "ebic_plane.cuh"

namespace ebic {

template <int P> struct PairVec;
template <> struct PairVec<1> { using V = uint32_t; };
template <> struct PairVec<2> { using V = uint2; };
template <> struct PairVec<4> { using V = uint4; };

// D = Rg - T - 0x00010001 word-wise; keep the guard bits (15, 31)
__device__ __forceinline__ uint32_t gt2(uint32_t rg, uint32_t t) { return (rg - t - 0x00010001u) & 0x80008000u; }

__device__ __forceinline__ uint32_t& wref(uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t& wref(uint2& v, int q) { return q ? v.y : v.x; }
__device__ __forceinline__ uint32_t& wref(uint4& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }
__device__ __forceinline__ uint32_t wget(const uint32_t& v, int) { return v; }
__device__ __forceinline__ uint32_t wget(const uint2& v, int q) { return q ? v.y : v.x; }
__device__ __forceinline__ uint32_t wget(const uint4& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }

template <int P, typename V>
__device__ __forceinline__ void and_gt(V& acc, const V& rg, const V& t) {
#pragma unroll
  for (int q = 0; q < P; ++q) wref(acc, q) &= gt2(wget(rg, q), wget(t, q));
}

template <int P, typename V>
__device__ __forceinline__ void or_into(V& acc, const V& x) {
#pragma unroll
  for (int q = 0; q < P; ++q) wref(acc, q) |= wget(x, q);
}

template <int P, typename V>
__device__ __forceinline__ uint32_t popc_words(const V& v) {
  uint32_t n = 0;
#pragma unroll
  for (int q = 0; q < P; ++q) n += __popc(wget(v, q));
  return n;
}

// Fixed-length body.  Loads T(c0), Rg(c1), T(c1), ..., Rg(c_{L-1}) (forward) and
// additionally Rg(c0) / T(c_{L-1}) for the reversed direction.  TOFF is the
// byte distance from a column's Rg words to its T words.  Returns the guard bits of
// the lane's row pairs that support the candidate.
template <int L, int P, bool NEG, uint32_t COLSHIFT>
__device__ __forceinline__ typename PairVec<P>::V simd_eval(uint32_t lane_rg, uint32_t TOFF, const uint4& rec,
                                                          typename PairVec<P>::V vmask) {
  using V = typename PairVec<P>::V;
  const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                 hi16(rec.z), lo16(rec.w), hi16(rec.w)};
  uint32_t addr[L];
#pragma unroll
  for (int k = 0; k < L; ++k) addr[k] = lane_rg + (cc[k] << COLSHIFT);
  V rg[L], t[L];
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const bool need_rg = NEG || k > 0, need_t = NEG || k + 1 < L;
    if (need_rg) rg[k] = lds<V>(addr[k]);
    if (need_t) t[k] = lds<V>(addr[k] + TOFF);
  }
  V f = vmask;
#pragma unroll
  for (int k = 1; k < L; ++k) and_gt<P>(f, rg[k], t[k - 1]);
  if constexpr (NEG) {
    V r = vmask;
#pragma unroll
    for (int k = 1; k < L; ++k) and_gt<P>(r, rg[k - 1], t[k]);
    or_into<P>(f, r);
  }
  return f;
}

template <int P, int SUB, bool NEG, int L, uint32_t COLSHIFT>
__device__ __forceinline__ void simd_sweep_class(const SlabArgs& a, uint32_t sa_rec, uint32_t lane_rg, uint32_t TOFF,
                                                 uint32_t* s_cnt, uint32_t n_padded, uint32_t class_base,
                                                 uint32_t c_begin, typename PairVec<P>::V vmask, int warp,
                                                 int lane, int sub) {
  using V = typename PairVec<P>::V;
  constexpr int LPC = 32 / SUB;
  constexpr uint32_t stride = kSlabWarps * SUB;
  for (uint32_t t = warp * SUB + sub; t < n_padded; t += stride) {
    const uint4 rec = lds<uint4>(sa_rec + (class_base + t) * 16);
    const uint32_t j = lo16(rec.x);
    V ok;
    if constexpr (L == 1) {
      ok = vmask;  // no pair: every row supports (the trend.cpp:19 loop never runs)
    } else if constexpr (L < 8) {
      ok = simd_eval<L, P, NEG, COLSHIFT>(lane_rg, TOFF, rec, vmask);
    } else {
      // >= 8 columns: first 7 from the record, the tail from the CSR
      const uint32_t cc[kRecCols] = {hi16(rec.x), lo16(rec.y), hi16(rec.y), lo16(rec.z),
                                     hi16(rec.z), lo16(rec.w), hi16(rec.w)};
      V f = vmask, r = NEG ? vmask : V{};
      uint32_t ap = lane_rg + (cc[0] << COLSHIFT);
      V rgp = NEG ? lds<V>(ap) : V{}, tp = lds<V>(ap + TOFF);
      auto step = [&](uint32_t col) {
        const uint32_t ac = lane_rg + (col << COLSHIFT);
        const V rgc = lds<V>(ac), tc = lds<V>(ac + TOFF);
        and_gt<P>(f, rgc, tp);
        if (NEG) and_gt<P>(r, rgp, tc);
        rgp = rgc;
        tp = tc;
      };
#pragma unroll
      for (int k = 1; k < kRecCols; ++k) step(cc[k]);
      if (j < a.chunk) {
        const uint32_t b = a.offs[c_begin + j], e = a.offs[c_begin + j + 1];
        for (uint32_t k = b + kRecCols; k < e; ++k) {
          uint32_t any = 0;
#pragma unroll
          for (int q = 0; q < P; ++q) any |= wget(f, q) | wget(r, q);
          if (!any) break;  // this lane's rows are all decided
          step(__ldg(a.cols + k));
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
  using V = typename PairVec<P>::V;
  constexpr int LPC = 32 / SUB;
  constexpr uint32_t RT = LPC * 2 * P;             // rows per slab
  constexpr uint32_t CWP = RT / 2;                 // words per column per plane
  constexpr uint32_t COLSHIFT = CWP == 8 ? 5 : CWP == 16 ? 6 : CWP == 32 ? 7 : CWP == 64 ? 8 : 9;  // log2(CWP*4)
  static_assert((1u << COLSHIFT) == CWP * 4, "column stride must be a power of two");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // T plane offset: Rg plane size rounded so that T(c) sits 16 banks away from Rg(c)
  const uint32_t rg_words = a.n_cols * CWP;
  const uint32_t t_words = rg_words + ((48u - rg_words % 32u) % 32u);  // == 16 (mod 32)
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(smem_raw);               // Rg plane, then T plane
  uint4* s_rec = reinterpret_cast<uint4*>(s_slab + t_words + rg_words + 16);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_rec + a.chunk + kClasses * kSlabWarps * SUB);
  __shared__ uint32_t s_hist[kClasses], s_base[kClasses], s_fill[kClasses];
  const uint32_t sa_slab = (uint32_t)__cvta_generic_to_shared(s_slab);
  const uint32_t sa_rec = (uint32_t)__cvta_generic_to_shared(s_rec);
  const uint32_t TOFF = t_words * 4;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPC, rl = lane % LPC;
  const uint32_t lane_rg = sa_slab + rl * P * 4;
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
    // words) of one column and writes 2 pair-words to each 16-bit half-plane
    {
      constexpr uint32_t Q = RT / 4;  // uint4 per column
      const uint32_t total = a.n_cols * Q;
      const uint4* src = reinterpret_cast<const uint4*>(a.plane);
      const uint64_t ld4 = a.ld / 4, r4 = row0 / 4;
#pragma unroll 4
      for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint32_t c = t / Q, q = t % Q;
        const uint4 w = __ldg(src + c * ld4 + r4 + q);
        const uint2 rg = make_uint2(__byte_perm(w.x, w.y, 0x7632) | 0x80008000u,
                                    __byte_perm(w.z, w.w, 0x7632) | 0x80008000u);
        const uint2 tt = make_uint2(__byte_perm(w.x, w.y, 0x5410), __byte_perm(w.z, w.w, 0x5410));
        *reinterpret_cast<uint2*>(s_slab + c * CWP + 2 * q) = rg;
        *reinterpret_cast<uint2*>(s_slab + t_words + c * CWP + 2 * q) = tt;
      }
    }
    __syncthreads();

    // validity guard bits of this lane's row pairs (rows beyond n_rows never count)
    const uint32_t valid_rows = min(RT, a.n_rows - row0);
    V vmask;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const uint32_t r = (rl * P + q) * 2;
      wref(vmask, q) = (r < valid_rows ? 0x8000u : 0u) | (r + 1 < valid_rows ? 0x80000000u : 0u);
    }

#define EBIC_SIMD_SWEEP(L)                                                                                  \
  simd_sweep_class<P, SUB, NEG, L, COLSHIFT>(a, sa_rec, lane_rg, TOFF, s_cnt, s_hist[L], s_base[L], c_begin, \
                                             vmask, warp, lane, sub)
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
