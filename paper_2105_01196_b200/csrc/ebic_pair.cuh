// ebic_pair.cuh -- the hot kernel: packed rank pairs over a shared-memory row
// slab, with position-indexed counts.
//
// The packed-pair test of ebic_simd.cuh: a slab column line
// holds interleaved 16-bit row pairs (stage_pairs) and one IADD
// tests two rows.  What changes is the per-candidate bookkeeping, which on
// B200 is what competes with the column loads for the shared-memory pipe:
//
//   * Counts are indexed by the candidate's POSITION in the chunk's class-
//     sorted record list, not by its slot.  Warp w visits the same positions
//     in every slab (class lists are padded to the sweep stride, so every warp
//     runs the same K iterations per slab), so iteration g's warp-reduced
//     count is parked in lane (g & 31)'s `pending` register and written to the
//     warp's shared accumulator row once every 32 iterations (one LDS+STS per
//     lane and candidate-per-warp) -- no per-candidate shared atomic.  The
//     position -> slot map is applied once per chunk, in the flush.
//   * Records carry columns only: 8 bytes (4 x u16) for candidates of <= 4
//     columns -- one 8-byte LDS per iteration instead of a 16-byte one, i.e.
//     one shared-memory wavefront instead of two for the two (or four)
//     records of a warp instruction -- and 16 bytes (7 x u16 + the u16 slot,
//     needed for the CSR tail of candidates longer than 7 columns) otherwise.
//   * The next record is loaded before the current candidate is evaluated
//     (software pipelining), taking one shared-memory round trip off the
//     dependency chain of every iteration.
//
// Reference: trend.cpp:56-72 (evaluate_population), predicate trend.cpp:17-46.
#pragma once
#include <cstdint>
#include <type_traits>

#include "ebic_simd.cuh"

namespace ebic {

// class sweep order, most common lengths first (must match the EBIC_PAIR_SWEEP sequence)
__host__ __device__ constexpr int sweep_order(int q) {
  return q == 0 ? 4 : q == 1 ? 3 : q == 2 ? 5 : q == 3 ? 2 : q == 4 ? 6 : q == 5 ? 7 : q == 6 ? 8 : 1;
}
constexpr uint32_t kDummySlot = 0xFFFFu;

__host__ __device__ constexpr uint32_t pair_rec_bytes(int L) { return L <= 4 ? 8u : 16u; }
// shared bytes per chunk position: worst-case record + u32 count + u16 slot
constexpr uint32_t kPairPosBytes = 16 + 4 + 2;

struct PairBook {             // shared-memory bookkeeping of the staged chunk
  uint32_t real[kClasses];    // candidates per class
  uint32_t npad[kClasses];    // positions per class (padded to the sweep stride)
  uint32_t pbase[kClasses];   // first position of the class
  uint32_t rbyte[kClasses];   // byte offset of the class's records
  uint32_t gbase[kClasses];   // first per-warp sweep iteration of the class
  uint32_t fill[kClasses];
  uint32_t K;                 // sweep iterations per warp per slab
  uint32_t npos;              // positions in the chunk
};

// Pack candidates [c_begin, c_begin + c_n) into class-sorted column records,
// the position -> slot map and zeroed accumulators.  Invalid candidates
// (empty, or a column >= n_cols) raise the device error flag and get no
// position (count 0).  Called by every thread of the CTA.
template <uint32_t STRIDE>
__device__ void pack_chunk_pos(const SlabArgs& a, uint32_t c_begin, uint32_t c_n, unsigned char* s_rec,
                               uint32_t* s_acc, uint16_t* s_perm, PairBook& bk) {
  auto class_of = [&](uint32_t i, uint32_t& b, uint32_t& len) -> uint32_t {
    b = a.offs[i];
    const uint32_t e = a.offs[i + 1];
    len = e > b ? e - b : 0;
    bool bad = len == 0;
    for (uint32_t k = b; k < e && !bad; ++k) bad |= a.cols[k] >= a.n_cols;
    return bad ? 0u : min(len, 8u);
  };
  if (threadIdx.x < kClasses) bk.real[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
    uint32_t b, len;
    const uint32_t cl = class_of(c_begin + j, b, len);
    if (cl == 0) atomicOr(a.err, 1);
    else atomicAdd(&bk.real[cl], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t pos = 0, byte = 0, g = 0;
    bk.npad[0] = bk.pbase[0] = bk.rbyte[0] = bk.gbase[0] = bk.fill[0] = 0;
    for (int q = 0; q < kClasses - 1; ++q) {
      const int c = sweep_order(q);
      const uint32_t np = (bk.real[c] + STRIDE - 1) / STRIDE * STRIDE;
      bk.npad[c] = np;
      bk.pbase[c] = pos;
      bk.rbyte[c] = byte;
      bk.gbase[c] = g;
      bk.fill[c] = 0;
      pos += np;
      byte += np * pair_rec_bytes(c);
      g += np / STRIDE;
    }
    bk.K = g;
    bk.npos = pos;
  }
  __syncthreads();
  // padding positions: column-0 records of the dummy slot, zeroed accumulators
  for (uint32_t p = threadIdx.x; p < bk.npos; p += blockDim.x) s_acc[p] = 0;
  for (int q = 0; q < kClasses - 1; ++q) {
    const int c = sweep_order(q);
    const uint32_t rb = pair_rec_bytes(c);
    for (uint32_t t = bk.real[c] + threadIdx.x; t < bk.npad[c]; t += blockDim.x) {
      s_perm[bk.pbase[c] + t] = (uint16_t)kDummySlot;
      if (rb == 8) *reinterpret_cast<uint2*>(s_rec + bk.rbyte[c] + t * 8) = make_uint2(0u, 0u);
      else *reinterpret_cast<uint4*>(s_rec + bk.rbyte[c] + t * 16) = make_uint4(0u, 0u, 0u, kDummySlot << 16);
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
    uint32_t b, len;
    const uint32_t cl = class_of(c_begin + j, b, len);
    if (cl == 0) continue;
    const uint32_t t = atomicAdd(&bk.fill[cl], 1u);
    s_perm[bk.pbase[cl] + t] = (uint16_t)j;
    uint32_t h[8] = {0, 0, 0, 0, 0, 0, 0, j};
#pragma unroll
    for (int k = 0; k < kRecCols; ++k)
      if ((uint32_t)k < len) h[k] = a.cols[b + k];
    if (cl <= 4) {
      *reinterpret_cast<uint2*>(s_rec + bk.rbyte[cl] + t * 8) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
    } else {
      *reinterpret_cast<uint4*>(s_rec + bk.rbyte[cl] + t * 16) =
          make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
    }
  }
}

// Record -> column list (u16 halves, one PRMT each).
__device__ __forceinline__ void rec_cols(const uint2& r, uint32_t (&cc)[kRecCols]) {
  cc[0] = lo16(r.x); cc[1] = hi16(r.x); cc[2] = lo16(r.y); cc[3] = hi16(r.y);
  cc[4] = cc[5] = cc[6] = 0;
}
__device__ __forceinline__ void rec_cols(const uint4& r, uint32_t (&cc)[kRecCols]) {
  cc[0] = lo16(r.x); cc[1] = hi16(r.x); cc[2] = lo16(r.y); cc[3] = hi16(r.y);
  cc[4] = lo16(r.z); cc[5] = hi16(r.z); cc[6] = lo16(r.w);
}

// Park this iteration's warp-reduced count in lane (g & 31); every 32
// iterations each lane adds its parked count to the warp's accumulator row
// (unpacking the SUB candidate fields).  acc_w = this warp's row: [K][SUB].
template <int SUB>
__device__ __forceinline__ void park_count(uint32_t tot, uint32_t& g, uint32_t& pending, uint32_t* acc_w, int lane) {
  if (lane == (int)(g & 31u)) pending = tot;
  if ((g & 31u) == 31u) {
    uint32_t* dst = acc_w + (g - 31u + lane) * SUB;
    constexpr uint32_t FW = 32 / SUB;
#pragma unroll
    for (int s = 0; s < SUB; ++s) dst[s] += SUB == 1 ? pending : (pending >> (FW * s)) & ((1u << (FW % 32)) - 1u);
  }
  ++g;
}

template <int SUB>
__device__ __forceinline__ void park_flush_tail(uint32_t g, uint32_t pending, uint32_t* acc_w, int lane) {
  const uint32_t g0 = g & ~31u;
  if (g0 + lane < g) {
    uint32_t* dst = acc_w + (g0 + lane) * SUB;
    constexpr uint32_t FW = 32 / SUB;
#pragma unroll
    for (int s = 0; s < SUB; ++s) dst[s] += SUB == 1 ? pending : (pending >> (FW * s)) & ((1u << (FW % 32)) - 1u);
  }
}

template <int P, int SUB, bool NEG, int L, uint32_t COLSHIFT>
__device__ __forceinline__ void pair_sweep_class(const SlabArgs& a, uint32_t sa_recs, uint32_t lane_base, uint32_t nk,
                                                 uint32_t c_begin, typename PairVec<P>::M vmask, int warp, int lane,
                                                 int sub, uint32_t& g, uint32_t& pending, uint32_t* acc_w) {
  using V = typename PairVec<P>::V;
  using M = typename PairVec<P>::M;
  using R = typename std::conditional<(L <= 4), uint2, uint4>::type;
  constexpr uint32_t RB = pair_rec_bytes(L);
  constexpr uint32_t stride = kSlabWarps * SUB;
  constexpr uint32_t FW = 32 / SUB;
  if (nk == 0) return;
  uint32_t addr = sa_recs + (warp * SUB + sub) * RB;
  const uint32_t last = sa_recs + ((nk - 1) * stride + warp * SUB + sub) * RB;
  R rec{};
  if constexpr (L > 1) rec = lds<R>(addr);
  for (uint32_t k = 0; k < nk; ++k) {
    R nxt{};
    if constexpr (L > 1) nxt = lds<R>(min(addr + stride * RB, last));  // next record, in flight during this one
    M ok;
    if constexpr (L == 1) {
      ok = vmask;  // no pair: every row supports (the trend.cpp:19 loop never runs)
    } else {
      uint32_t cc[kRecCols];
      rec_cols(rec, cc);
      if constexpr (L < 8 && P == 1 && SUB == 2 && !NEG) {
        // The first column contributes only NT words (odd banks of its line)
        // and the last only Rg words (even banks).  Half-warp 0 fetches its
        // first column while half-warp 1 fetches its last, then the other way
        // round: each LDS.32 puts 16 odd-bank and 16 even-bank words in one
        // wavefront (two ordinary 4-byte loads of the same kind would collide
        // pairwise across the half-warps and take two).  The middle columns
        // are LDS.64s of one aligned 128-byte line per half-warp, as before.
        const uint32_t a_first = lane_base + (cc[0] << COLSHIFT) + 4, a_last = lane_base + (cc[L - 1] << COLSHIFT);
        const uint32_t x0 = lds<uint32_t>(sub ? a_last : a_first);
        const uint32_t x1 = lds<uint32_t>(sub ? a_first : a_last);
        V w[L];
#pragma unroll
        for (int q = 1; q < L - 1; ++q) w[q] = lds<V>(lane_base + (cc[q] << COLSHIFT));
        w[0].y = sub ? x1 : x0;      // NT of the first column
        w[L - 1].x = sub ? x0 : x1;  // Rg of the last column
        M f = vmask;
#pragma unroll
        for (int q = 1; q < L; ++q) and_pair<P>(f, w[q], w[q - 1]);
        ok = f;
      } else if constexpr (L < 8) {
        V w[L];
#pragma unroll
        for (int q = 0; q < L; ++q) w[q] = lds<V>(lane_base + (cc[q] << COLSHIFT));
        M f = vmask;
#pragma unroll
        for (int q = 1; q < L; ++q) and_pair<P>(f, w[q], w[q - 1]);
        if constexpr (NEG) {
          M r = vmask;
#pragma unroll
          for (int q = 1; q < L; ++q) and_pair<P>(r, w[q - 1], w[q]);
          or_into<P>(f, r);
        }
        ok = f;
      } else {
        // >= 8 columns: the first 7 from the record, the tail from the CSR
        M f = vmask, r = NEG ? vmask : M{};
        V wp = lds<V>(lane_base + (cc[0] << COLSHIFT));
#pragma unroll
        for (int q = 1; q < kRecCols; ++q) {
          const V wc = lds<V>(lane_base + (cc[q] << COLSHIFT));
          and_pair<P>(f, wc, wp);
          if (NEG) and_pair<P>(r, wp, wc);
          wp = wc;
        }
        const uint32_t j = hi16(rec.w);
        if (j != kDummySlot) {
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
    }
    // candidate `sub` owns bit field [sub*FW, (sub+1)*FW) of the warp sum
    static_assert(SUB == 1 || (2u * P * (32 / SUB)) < (1u << FW), "count field too narrow");
    const uint32_t tot = __reduce_add_sync(kFull, popc_words<P>(ok) << (FW * sub));
    park_count<SUB>(tot, g, pending, acc_w, lane);
    rec = nxt;
    addr += stride * RB;
  }
}

template <int P, int SUB, bool NEG>
__global__ void __launch_bounds__(kSlabThreads, 1)
slab_pair_kernel(const SlabArgs a) {
  using M = typename PairVec<P>::M;
  constexpr int LPC = 32 / SUB;
  constexpr uint32_t RT = LPC * 2 * P;             // rows per slab
  constexpr uint32_t CW = RT;                      // words per column line: RT/2 x (Rg, NT)
  constexpr uint32_t COLSHIFT = CW == 16 ? 6 : CW == 32 ? 7 : CW == 64 ? 8 : CW == 128 ? 9 : 10;  // log2(CW*4)
  static_assert((1u << COLSHIFT) == CW * 4, "column stride must be a power of two");
  constexpr uint32_t STRIDE = kSlabWarps * SUB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_slab = reinterpret_cast<uint32_t*>(smem_raw);                 // [C][RT/2 x (Rg, NT)]
  const uint32_t max_pos = a.chunk + (kClasses - 1) * STRIDE;
  unsigned char* s_rec = reinterpret_cast<unsigned char*>(s_slab + (size_t)a.n_cols * CW);  // <= 16 B per position
  uint32_t* s_acc = reinterpret_cast<uint32_t*>(s_rec + (size_t)max_pos * 16);               // [32 warps][K][SUB]
  uint16_t* s_perm = reinterpret_cast<uint16_t*>(s_acc + max_pos);                           // position -> slot
  __shared__ PairBook bk;
  const uint32_t sa_slab = (uint32_t)__cvta_generic_to_shared(s_slab);
  const uint32_t sa_rec = (uint32_t)__cvta_generic_to_shared(s_rec);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPC, rl = lane % LPC;
  const uint32_t lane_base = sa_slab + rl * P * 8;  // this lane's (Rg, NT) pair(s) in column 0
  // Work: chunk groups of a.group CTAs.  CTA b sweeps slab range b % group of
  // chunks b / group, b / group + n_groups, ...; CTA i of every group sweeps
  // the same slab range, so the groups read each slab of the plane at about
  // the same time (one pass over the plane from DRAM when it exceeds L2).
  const uint32_t n_groups = gridDim.x / a.group, gi = blockIdx.x % a.group;
  const uint32_t s_begin = (uint32_t)((uint64_t)gi * a.n_slabs / a.group);
  const uint32_t s_end = (uint32_t)((uint64_t)(gi + 1) * a.n_slabs / a.group);
  __shared__ uint32_t s_last;

  for (uint32_t chunk = blockIdx.x / a.group; chunk < a.n_chunks; chunk += n_groups) {
    const uint32_t c_begin = chunk * a.chunk, c_n = min(a.chunk, a.n_cand - c_begin);
    __syncthreads();  // the previous chunk's records / bookkeeping are no longer read
    pack_chunk_pos<STRIDE>(a, c_begin, c_n, s_rec, s_acc, s_perm, bk);
    for (uint32_t slab = s_begin; slab < s_end; ++slab) {
      const uint32_t row0 = slab * RT;
      __syncthreads();  // previous slab fully consumed (and the pack done)
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
      prefetch_next_slab<RT>(a, (uint64_t)chunk * a.n_slabs + slab + 1, (uint64_t)chunk * a.n_slabs + s_end);

      const uint32_t valid_rows = min(RT, a.n_rows - row0);
      M vmask;
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const uint32_t r = (rl * P + q) * 2;
        wref(vmask, q) = (r < valid_rows ? 0x8000u : 0u) | (r + 1 < valid_rows ? 0x80000000u : 0u);
      }
      uint32_t g = 0, pending = 0;
      uint32_t* acc_w = s_acc + (size_t)warp * bk.K * SUB;
#define EBIC_PAIR_SWEEP(L)                                                                                   \
    pair_sweep_class<P, SUB, NEG, L, COLSHIFT>(a, sa_rec + bk.rbyte[L], lane_base, bk.npad[L] / STRIDE, c_begin, \
                                               vmask, warp, lane, sub, g, pending, acc_w)
      EBIC_PAIR_SWEEP(4);
      EBIC_PAIR_SWEEP(3);
      EBIC_PAIR_SWEEP(5);
      EBIC_PAIR_SWEEP(2);
      EBIC_PAIR_SWEEP(6);
      EBIC_PAIR_SWEEP(7);
      EBIC_PAIR_SWEEP(8);
      EBIC_PAIR_SWEEP(1);
#undef EBIC_PAIR_SWEEP
      park_flush_tail<SUB>(g, pending, acc_w, lane);
    }  // slabs
    __syncthreads();
    // position-indexed accumulators -> the chunk's global partial counts
    for (uint32_t p = threadIdx.x; p < bk.npos; p += blockDim.x) {
      const uint32_t slot = s_perm[p];
      if (slot >= c_n) continue;
      int c = sweep_order(0);
#pragma unroll
      for (int q = 1; q < kClasses - 1; ++q)
        if (p >= bk.pbase[sweep_order(q)]) c = sweep_order(q);
      const uint32_t t = p - bk.pbase[c];
      const uint32_t w = (t % STRIDE) / SUB, s = t % SUB, g = bk.gbase[c] + t / STRIDE;
      const uint32_t cnt = s_acc[(w * bk.K + g) * SUB + s];
      if (cnt) atomicAdd(&a.counts[c_begin + slot], cnt);
    }
    // the last CTA of the chunk group publishes the chunk's counts to a.out
    // (device memory, or page-locked host memory written over the bus: no
    // separate D2H copy) and re-zeroes the accumulators for the next launch
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&a.done[chunk], 1u) == a.group - 1;
    __syncthreads();
    if (s_last) {
      // (writes to page-locked host memory are visible to the host once the
      // kernel has completed: no system-scope fence needed here)
      __threadfence();
      for (uint32_t j = threadIdx.x; j < c_n; j += blockDim.x) {
        a.out[c_begin + j] = __ldcg(&a.counts[c_begin + j]);
        a.counts[c_begin + j] = 0;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        a.done[chunk] = 0;
        // the last chunk to be published forwards the device error flag
        if (atomicAdd(&a.done[a.n_chunks], 1u) == a.n_chunks - 1) {
          if (a.err_out != a.err) {
            *a.err_out = *(volatile int*)a.err;
            *a.err = 0;
          }
          a.done[a.n_chunks] = 0;
        }
      }
    }
  }  // chunks
}

}  // namespace ebic
