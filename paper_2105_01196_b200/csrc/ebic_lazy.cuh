// ebic_lazy.cuh -- the lazy pair-trend index: pair vectors built on first use.
//
// The full index (ebic_table.cuh) holds the pair vector B(a, b) of EVERY
// ordered column pair: C^2 x R/8 bytes (2.5 GB at 20k x 1000, 100 GB at
// 200k x 2000), built before the first evaluation.  A GA population touches
// only a small part of it (a C3 population of 16384 candidates, about 49K of
// the 1M pairs), so the lazy index builds a pair vector the first time a
// candidate needs it and keeps it in a pool for every later batch:
//
//   map[a * C + b]   uint32 per ordered pair: kSlotEmpty, the pool slot s of
//                    a ready vector, or s | kSlotBusy while its builder runs
//   pool[s * wp ...] the vector of slot s, same word layout as the full index
//                    (even rows in the low half of a word, odd rows in the high
//                    half: index_valid_bits / index_to_natural)
//   count            slots handed out so far (may exceed the capacity: a
//                    failed allocation still counts, so the host sees a full
//                    pool and grows or resets it before the next batch)
//
// The count kernels resolve and build inside the evaluation (no extra kernel
// per batch): a warp looks up its candidate's pairs in the map; ready vectors
// are read from the pool exactly like full-index vectors; a missing vector is
// built by the warp from the value store (the reference's own test,
// trend.cpp:22: v_r(b) > v_r(a) - approx*|v_r(a)| in double with two rounded
// ops, thr64), used directly, and -- if the warp won the slot (atomicCAS
// kSlotEmpty -> s | kSlotBusy) -- written to the pool and published (release:
// fence, then map[p] = s).  A warp that finds a vector busy (another warp is
// building it) or the pool full builds a private copy instead of waiting, so
// no warp ever spins on another.  Exactness does not depend on the cache: a
// built vector is the same bits the full-index builder produces.
#pragma once
#include <cstdint>

#include "ebic_kernels.cuh"

namespace ebic {

constexpr uint32_t kSlotEmpty = 0xFFFFFFFFu;
constexpr uint32_t kSlotBusy = 0x80000000u;  // high bit: claimed, vector not yet published

struct LazyArgs {
  uint32_t* map;        // C x C slots
  uint32_t* pool;       // cap x wp words
  uint32_t* count;      // slots handed out
  uint32_t* count_out;  // (optional, host-mapped) {count at kernel start, seq}: the host's lagged view of the fill
  uint32_t cap;         // slots in the pool
  uint32_t seq;         // batch sequence number (written with the count)
  const void* mat;      // value store (column-major, ld rows per column)
  uint64_t ld;
  int f64;              // store is double
  double approx;
};

__device__ __forceinline__ bool slot_ready(uint32_t s) { return s < kSlotBusy; }

__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Row of a 32-row word evaluated by `lane`: with lane l on row perm(l), a
// ballot over the warp is the index word itself (bit j < 16: row 2j, bit
// 16 + j: row 2j + 1).
__device__ __forceinline__ uint32_t index_row_of_lane(int lane) {
  return lane < 16 ? 2u * lane : 2u * (lane - 16) + 1u;
}

// One row's bit of B(a, b): trend.cpp:22 in double, two rounded ops (thr64).
template <typename T>
__device__ __forceinline__ bool pair_row_bit(const T* __restrict__ ca, const T* __restrict__ cb, uint32_t r,
                                             double approx) {
  return (double)__ldg(cb + r) > thr64((double)__ldg(ca + r), approx);
}

// The warp builds the wp-word vector B(a, b) and hands word w to `emit(w, word)`
// on lane w % 32 (one call per 32-word chunk per lane).  Loads are clamped to
// valid rows and issued unconditionally (8 words in flight per lane).
template <typename T, typename Emit>
__device__ __forceinline__ void build_pair_vector_warp_t(const T* __restrict__ mat, uint64_t ld, uint32_t n_rows,
                                                         uint32_t a, uint32_t b, double approx, uint32_t wp, int lane,
                                                         Emit emit) {
  const T* ca = mat + (uint64_t)a * ld;
  const T* cb = mat + (uint64_t)b * ld;
  const uint32_t rl = index_row_of_lane(lane);
  const uint32_t last = n_rows - 1;
  for (uint32_t w0 = 0; w0 < wp; w0 += 32) {
    uint32_t mine = 0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const uint32_t r = 32u * (w0 + j) + rl;
      const bool ok = r < n_rows;
      const bool bit = pair_row_bit(ca, cb, ok ? r : last, approx) && ok;
      const uint32_t word = __ballot_sync(kFull, bit);
      mine = lane == j ? word : mine;
    }
    if (w0 + lane < wp) emit(w0 + lane, mine);
  }
}

template <typename Emit>
__device__ __forceinline__ void build_pair_vector_warp(const LazyArgs& la, uint32_t n_rows, uint32_t a, uint32_t b,
                                                       uint32_t wp, int lane, Emit emit) {
  if (la.f64)
    build_pair_vector_warp_t(static_cast<const double*>(la.mat), la.ld, n_rows, a, b, la.approx, wp, lane, emit);
  else
    build_pair_vector_warp_t(static_cast<const float*>(la.mat), la.ld, n_rows, a, b, la.approx, wp, lane, emit);
}

// uint4 slice v (words 4v .. 4v + 3, rows 128 v .. 128 v + 127) of B(a, b),
// by one thread -- the slow path of the long-vector kernels for a vector that
// another warp is still building (or that found the pool full).
template <typename T>
__device__ uint4 pair_slice_thread_t(const T* __restrict__ mat, uint64_t ld, uint32_t n_rows, uint32_t a, uint32_t b,
                                     uint32_t v, double approx) {
  const T* ca = mat + (uint64_t)a * ld;
  const T* cb = mat + (uint64_t)b * ld;
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t word = 0;
    const uint32_t r0 = 128u * v + 32u * q;
    for (int j = 0; j < 32; ++j) {
      const uint32_t r = r0 + index_row_of_lane(j);
      if (r < n_rows && pair_row_bit(ca, cb, r, approx)) word |= 1u << j;
    }
    w[q] = word;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ uint4 pair_slice_thread(const LazyArgs& la, uint32_t n_rows, uint32_t a, uint32_t b,
                                                   uint32_t v) {
  return la.f64 ? pair_slice_thread_t(static_cast<const double*>(la.mat), la.ld, n_rows, a, b, v, la.approx)
                : pair_slice_thread_t(static_cast<const float*>(la.mat), la.ld, n_rows, a, b, v, la.approx);
}

// Claim the slot of pair p for this warp (lane 0 calls; result broadcast by
// the caller).  Returns the slot with kSlotBusy set when this warp must build
// and publish it, kSlotEmpty when it must build a private copy (lost the race
// or the pool is full).
__device__ __forceinline__ uint32_t lazy_claim(const LazyArgs& la, uint64_t p) {
  const uint32_t t = atomicAdd(la.count, 1u);
  if (t >= la.cap) return kSlotEmpty;
  const uint32_t old = atomicCAS(la.map + p, kSlotEmpty, t | kSlotBusy);
  return old == kSlotEmpty ? (t | kSlotBusy) : kSlotEmpty;  // (a lost race leaves slot t unused)
}

// Publish a vector the warp has written to pool[slot]: every lane makes its
// own stores visible at device scope (and to the TMA engine, which reads the
// pool through the async proxy), the warp synchronises, then lane 0 releases
// the map entry.  All 32 lanes call.
__device__ __forceinline__ void lazy_publish(const LazyArgs& la, uint64_t p, uint32_t slot, int lane) {
  __threadfence();
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
  if (lane == 0) atomicExch(la.map + p, slot);
}

// Map lookup (relaxed, device scope: entries published during this kernel are seen).
__device__ __forceinline__ uint32_t lazy_lookup(const LazyArgs& la, uint64_t p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(la.map + p) : "memory");
  return v;
}

}  // namespace ebic
