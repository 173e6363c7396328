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
//                    (index_bit_row / index_valid_bits / index_to_natural)
//   count            slots handed out so far (may exceed the capacity: a
//                    failed allocation still counts, so the host sees a full
//                    pool and grows or resets it before the next batch)
//
// Warm batches resolve and build inside the count kernel (no extra kernel per
// batch); cold batches -- the pool still filling fast -- and long vectors run
// claim / build / publish kernels first (lazy_slab_build_kernel, below).
// Inside the count kernel a warp looks up its candidate's pairs in the map; ready vectors
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
#include <type_traits>

#include "ebic_kernels.cuh"
#include "ebic_index.cuh"

namespace ebic {

constexpr uint32_t kSlotEmpty = 0xFFFFFFFFu;
constexpr uint32_t kSlotBusy = 0x80000000u;  // high bit: claimed, vector not yet published

struct LazyArgs {
  uint32_t* map;        // C x C slots
  // claim / build / publish kernels (long vectors, cold batches): per pool
  // slot, the pair it was claimed for and the claiming batch's tag
  // (kSlotEmpty: not waiting to be built), the 32-word chunks still to build
  // (lazy_build_kernel), and a ring of batch windows: start[seq % ring] = the
  // count before the batch's claims, start[ring + seq % ring] = after them
  uint32_t* keys;
  uint32_t* left;
  const uint32_t* start;
  uint32_t* defer;      // [0]: candidates deferred by the count kernel, [1..]: their indices
  uint32_t* pslot;      // [i * 64 + k (+ 32)]: slot of candidate i's k-th forward (reversed) pair, k < 31
  uint32_t* pool;       // cap x wp words
  uint32_t* count;      // slots handed out
  uint32_t* count_out;  // (optional, host-mapped) {count at kernel start, seq}: the host's lagged view of the fill
  uint32_t cap;         // slots in the pool
  uint32_t seq;         // batch sequence number (written with the count)
  const void* mat;      // value store (column-major, ld rows per column)
  uint64_t ld;
  int f64;              // store is double
  double approx;
  float a_f, kscale;    // float32 bracket of the threshold (ebic_kernels.cuh bracket / make_args)
  int cold;             // host: the pool is still filling fast -- build the batch's pairs first
                        // (lazy_slab_build_kernel) instead of inside the count kernel
};

// The per-row test's parameters: the reference threshold in double, and a
// float32 bracket of it that decides all but the near-threshold rows of a
// float32 store without float64 arithmetic.
struct PairThr {
  double approx;
  float a_f, kscale;
};
__device__ __forceinline__ PairThr pair_thr(const LazyArgs& la) { return PairThr{la.approx, la.a_f, la.kscale}; }

__device__ __forceinline__ bool slot_ready(uint32_t s) { return s < kSlotBusy; }

__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// One row's bit of B(a, b): trend.cpp:22 in double, two rounded ops (thr64).
__device__ __forceinline__ bool pair_bit(double x, double y, const PairThr& th) { return y > thr64(x, th.approx); }
// float32 store: y > thr64(x) decided by the float32 bracket [t - d, t + d]
// of the threshold (the value kernels' filter mode); the double test runs
// only for y inside it
__device__ __forceinline__ bool pair_bit(float x, float y, const PairThr& th) {
  const float ax = fabsf(x);
  const float t = __fmaf_rn(-th.a_f, ax, x);
  const float d = bracket_halfwidth(ax, th.kscale);
  if (y > __fadd_rn(t, d)) return true;
  if (y <= __fsub_rn(t, d)) return false;
  return (double)y > thr64((double)x, th.approx);
}
template <typename T>
__device__ __forceinline__ bool pair_row_bit(const T* __restrict__ ca, const T* __restrict__ cb, uint32_t r,
                                             const PairThr& th) {
  return pair_bit(__ldg(ca + r), __ldg(cb + r), th);
}

// Word w of B(a, b) (rows 32 w .. 32 w + 31) by one thread: its 32 rows of
// both columns are read as 16-byte vectors (8 rows of each column in flight
// at a time) and tested with no cross-lane traffic, so a warp fills 32 words
// at once (round 2 used a ballot per word: ~41 warp-instructions per word,
// 31 ms for C4's 98K first-visit vectors).
// Rows past the column's allocation (ld) are not read; rows >= n_rows are
// masked out.
template <typename T>
__device__ __forceinline__ uint32_t pair_word_lane(const T* __restrict__ ca, const T* __restrict__ cb, uint32_t n_rows,
                                                   uint64_t ld, uint32_t w, const PairThr& th) {
  constexpr int VW = 16 / sizeof(T);  // rows per 16-byte vector
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const uint32_t r0 = 32u * w;
  const bool whole = (uint64_t)r0 + 32 <= ld;
  uint32_t word = 0;
#pragma unroll
  for (int g = 0; g < 32; g += 8) {
    T x[8], y[8];
    if (whole) {
#pragma unroll
      for (int q = 0; q < 8; q += VW) {
        const V va = __ldg(reinterpret_cast<const V*>(ca + r0 + g + q));
        const V vb = __ldg(reinterpret_cast<const V*>(cb + r0 + g + q));
        const T* pa = reinterpret_cast<const T*>(&va);
        const T* pb = reinterpret_cast<const T*>(&vb);
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          x[q + e] = pa[e];
          y[q + e] = pb[e];
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t r = r0 + g + j;
        x[j] = r < n_rows ? __ldg(ca + r) : (T)0;
        y[j] = r < n_rows ? __ldg(cb + r) : (T)0;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (pair_bit(x[j], y[j], th)) word |= 1u << index_row_bit((uint32_t)(g + j));
  }
  return word & index_valid_bits(n_rows, w);
}

// Words w0 .. w0 + 31 of B(a, b) for a float32 store, lane l returning word
// w0 + l, through shared memory: the warp reads the chunk's 1024 rows of both
// columns with coalesced 16-byte loads into `st` (2 x 32 x 33 floats, row r
// at (r / 32) * 33 + r % 32: conflict-free both ways), then each lane tests
// its own 32 rows.  (pair_word_lane reads a lane's 128-B row runs directly;
// with 64 warps per SM those lines leave L1 before their 8 loads are done.)
constexpr uint32_t kStageFloats = 2 * 32 * 33;
__device__ __forceinline__ uint32_t pair_word_staged(const float* __restrict__ ca, const float* __restrict__ cb,
                                                     uint32_t n_rows, uint64_t ld, uint32_t w0, const PairThr& th,
                                                     int lane, float* st) {
  float* sx = st;
  float* sy = st + 32 * 33;
  const uint32_t r0 = 32u * w0;
  if ((uint64_t)r0 + 1024 <= ld) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t r = 128u * k + 4u * lane;  // 4 rows per lane per k
      const float4 va = __ldg(reinterpret_cast<const float4*>(ca + r0 + r));
      const float4 vb = __ldg(reinterpret_cast<const float4*>(cb + r0 + r));
      const uint32_t o = (r >> 5) * 33u + (r & 31u);
      sx[o] = va.x; sx[o + 1] = va.y; sx[o + 2] = va.z; sx[o + 3] = va.w;
      sy[o] = vb.x; sy[o + 1] = vb.y; sy[o + 2] = vb.z; sy[o + 3] = vb.w;
    }
  } else {  // the column's last chunk: rows past ld are not read
    for (uint32_t r = lane; r < 1024; r += 32) {
      const uint32_t o = (r >> 5) * 33u + (r & 31u);
      sx[o] = r0 + r < n_rows ? __ldg(ca + r0 + r) : 0.f;
      sy[o] = r0 + r < n_rows ? __ldg(cb + r0 + r) : 0.f;
    }
  }
  __syncwarp();
  // branch-free float32 bracket per row (bit set above it, `unc` inside it);
  // the rare rows inside the bracket get the exact double test afterwards
  uint32_t word = 0, unc = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float x = sx[lane * 33 + j], y = sy[lane * 33 + j];
    const float ax = fabsf(x);
    const float t = __fmaf_rn(-th.a_f, ax, x);
    const float d = bracket_halfwidth(ax, th.kscale);
    const uint32_t bit = 1u << index_row_bit((uint32_t)j);
    word |= y > __fadd_rn(t, d) ? bit : 0u;
    unc |= (y > __fsub_rn(t, d) && !(y > __fadd_rn(t, d))) ? (1u << j) : 0u;
  }
  while (unc) {
    const int j = __ffs(unc) - 1;
    unc &= unc - 1;
    const float x = sx[lane * 33 + j], y = sy[lane * 33 + j];
    if ((double)y > thr64((double)x, th.approx)) word |= 1u << index_row_bit((uint32_t)j);
  }
  __syncwarp();  // (the stage is refilled by the warp's next unit)
  return word & index_valid_bits(n_rows, w0 + lane);
}

// The warp builds the wp-word vector B(a, b) and hands word w to `emit(w, word)`
// on lane w % 32 (one call per 32-word chunk per lane).
template <typename T, typename Emit>
__device__ __forceinline__ void build_pair_vector_warp_t(const T* __restrict__ mat, uint64_t ld, uint32_t n_rows,
                                                         uint32_t a, uint32_t b, const PairThr& th, uint32_t wp, int lane,
                                                         Emit emit) {
  const T* ca = mat + (uint64_t)a * ld;
  const T* cb = mat + (uint64_t)b * ld;
  for (uint32_t w0 = 0; w0 < wp; w0 += 32) {
    const uint32_t mine = pair_word_lane(ca, cb, n_rows, ld, w0 + lane, th);
    if (w0 + lane < wp) emit(w0 + lane, mine);
  }
}

template <typename Emit>
__device__ __forceinline__ void build_pair_vector_warp(const LazyArgs& la, uint32_t n_rows, uint32_t a, uint32_t b,
                                                       uint32_t wp, int lane, Emit emit) {
  if (la.f64)
    build_pair_vector_warp_t(static_cast<const double*>(la.mat), la.ld, n_rows, a, b, pair_thr(la), wp, lane, emit);
  else
    build_pair_vector_warp_t(static_cast<const float*>(la.mat), la.ld, n_rows, a, b, pair_thr(la), wp, lane, emit);
}

// uint4 slice v (words 4v .. 4v + 3, rows 128 v .. 128 v + 127) of B(a, b),
// by one thread -- the slow path of the long-vector kernels for a vector that
// another warp is still building (or that found the pool full).
template <typename T>
__device__ __noinline__ uint4 pair_slice_thread_t(const T* __restrict__ mat, uint64_t ld, uint32_t n_rows, uint32_t a, uint32_t b,
                                     uint32_t v, const PairThr& th) {
  const T* ca = mat + (uint64_t)a * ld;
  const T* cb = mat + (uint64_t)b * ld;
  uint32_t w[4];
#pragma unroll 1
  for (int q = 0; q < 4; ++q) w[q] = pair_word_lane(ca, cb, n_rows, ld, 4u * v + q, th);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ uint4 pair_slice_thread(const LazyArgs& la, uint32_t n_rows, uint32_t a, uint32_t b,
                                                   uint32_t v) {
  return la.f64 ? pair_slice_thread_t(static_cast<const double*>(la.mat), la.ld, n_rows, a, b, v, pair_thr(la))
                : pair_slice_thread_t(static_cast<const float*>(la.mat), la.ld, n_rows, a, b, v, pair_thr(la));
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

// ---------------------------------------------------------------------------
// Long pair vectors (more than 256 uint4 slices: rows > 32768, e.g. 200k x
// 2000).  A 25-KB vector is too big for a warp to build inside the count
// kernel, so a batch runs three kernels:
//   lazy_claim_kernel  every pair of the batch not in the map is claimed: a
//                      pool slot t (count), map[p] = t | kSlotBusy (CAS),
//                      keys[t] = p, left[t] = the vector's 32-word chunks;
//                      each candidate's first 31 pair slots go to pslot;
//   lazy_build_kernel  the slots claimed since the batch started ([*start,
//                      count)) are built, one warp per (chunk, slot) unit,
//                      chunk-major: the units in flight at once all read the
//                      same 1024-row slice of the matrix (8 MB at 2000
//                      columns), which stays in L2; the warp that finishes a
//                      slot's last chunk publishes it (map[p] = t);
//   table_count_warp_multi_kernel<..., LAZY>  reads the vectors from the
//                      pool (slots from pslot, loaded with the columns) and
//                      defers a candidate with any pair not available (pool
//                      full, or busy in another stream's batch) to
//                      lazy_deferred_kernel, which computes such pairs from
//                      the value store.
// ---------------------------------------------------------------------------
// Batches may run on several streams at once (the device API takes the
// caller's stream), so a build kernel's slot window [start, count) can hold
// slots another batch claimed: a slot's key carries the claiming batch's tag
// (seq mod 63, bits 26..31; pair keys are < 2^26 since C <= 8192) and a build
// kernel builds only its own; the last chunk's warp clears the key again, so
// a key is set only between its batch's claim and build.
constexpr uint32_t kLazyKeyBits = 26;
constexpr uint32_t kLazyStartRing = 64;
// start[kLazyStartRing + seq % kLazyStartRing]: the count right after the
// batch's claim kernel (copied on the stream).  Every CTA of the build and
// publish kernels uses this one window end: other streams keep claiming while
// they run, and CTAs that each read the live count would partition the window
// differently (units never built, slots never published).
__device__ __forceinline__ uint32_t lazy_window_end(const LazyArgs& la) {
  return min(la.start[kLazyStartRing + la.seq % kLazyStartRing], la.cap);
}
__host__ __device__ __forceinline__ uint32_t lazy_tag(uint32_t seq) { return seq % 63u; }

// Did this batch claim slot s for pair p?  (A claim's key is written right
// after its CAS: a reader that comes too early answers "no", which only
// defers the candidate to lazy_deferred_kernel.)
__device__ __forceinline__ bool lazy_own_claim(const LazyArgs& la, uint32_t s, uint64_t p) {
  uint32_t k;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(k) : "l"(la.keys + s) : "memory");
  return k == ((uint32_t)p | (lazy_tag(la.seq) << kLazyKeyBits));
}

// The slot this batch will find pair p in once its build kernel has run:
// a ready slot, a slot this batch claims now (or claimed already, in another
// warp), or kSlotEmpty -- the pool is full, or another stream's batch is
// building p -- which defers the candidate.
__device__ __forceinline__ uint32_t lazy_claim_pair(const LazyArgs& la, uint64_t p, uint32_t n_chunks) {
  uint32_t v = lazy_lookup(la, p);
  if (v == kSlotEmpty) {
    const uint32_t t = atomicAdd(la.count, 1u);
    if (t >= la.cap) return kSlotEmpty;  // pool full
    v = atomicCAS(la.map + p, kSlotEmpty, t | kSlotBusy);
    if (v == kSlotEmpty) {  // ours (otherwise another thread claimed p first: slot t stays unused)
      la.left[t] = n_chunks;
      __threadfence();  // left before the key: the build kernel reads the key first
      la.keys[t] = (uint32_t)p | (lazy_tag(la.seq) << kLazyKeyBits);
      return t;
    }
  }
  if (slot_ready(v)) return v;
  const uint32_t s = v & ~kSlotBusy;
  return lazy_own_claim(la, s, p) ? s : kSlotEmpty;
}

// Claims the batch's missing pairs and records, per candidate, the slots of
// its first 31 forward (and reversed) pairs: pslot[i * 64 + k] (+ 32), so the
// count kernel loads them next to the columns instead of looking them up
// after the columns arrive (one dependent round trip less per candidate).
__global__ void __launch_bounds__(256)
lazy_claim_kernel(const LazyArgs la, const uint32_t* __restrict__ cols, const uint32_t* __restrict__ offs,
                  uint32_t n_cand, uint32_t n_idx, uint32_t n_cols, uint32_t n_chunks, int neg) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (la.defer) la.defer[0] = 0;  // (read by this batch's count kernel, which runs after this one)
    if (la.count_out) {  // the host's lagged view of the pool's fill
      la.count_out[0] = *(volatile uint32_t*)la.count;
      __threadfence_system();
      la.count_out[1] = la.seq;
    }
  }
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_cand; i += warps) {
    const uint32_t b = __ldg(offs + i), e = __ldg(offs + i + 1);
    if (e <= b || e > n_idx) continue;  // (reported by the count kernel)
    for (uint32_t k = b + 1 + lane; k < e; k += 32) {
      const uint32_t x = __ldg(cols + k - 1), y = __ldg(cols + k);
      if (x >= n_cols || y >= n_cols) continue;  // (reported by the count kernel)
      const uint32_t sf = lazy_claim_pair(la, (uint64_t)x * n_cols + y, n_chunks);
      const uint32_t sr = neg ? lazy_claim_pair(la, (uint64_t)y * n_cols + x, n_chunks) : kSlotEmpty;
      const uint32_t q = k - b - 1;  // pair index
      if (la.pslot && q < 31) {  // (no pslot: lazy_slab_build_kernel's batches count with the TMA kernel)
        la.pslot[(uint64_t)i * 64 + q] = sf;
        if (neg) la.pslot[(uint64_t)i * 64 + 32 + q] = sr;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
lazy_build_kernel(const LazyArgs la, uint32_t n_rows, uint32_t n_cols, uint32_t wp) {
  const uint32_t start = la.start[la.seq % kLazyStartRing];
  const uint32_t end = lazy_window_end(la);
  const uint32_t tag = lazy_tag(la.seq);
  if (end <= start) return;
  const uint32_t n_jobs = end - start, n_chunks = (wp + 31) / 32;
  const uint64_t total = (uint64_t)n_jobs * n_chunks;
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const T* mat = static_cast<const T*>(la.mat);
  extern __shared__ float stage[];  // float stores: kStageFloats per warp (pair_word_staged)
  for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < total; u += warps) {
    const uint32_t chunk = (uint32_t)(u / n_jobs), t = start + (uint32_t)(u % n_jobs);
    const uint32_t tk = __ldcg(la.keys + t);
    if (tk == kSlotEmpty || (tk >> kLazyKeyBits) != tag) continue;  // not claimed by this batch
    const uint32_t key = tk & ((1u << kLazyKeyBits) - 1u);
    const uint32_t a = key / n_cols, b = key % n_cols;
    const uint32_t w0 = chunk * 32;
    uint32_t word;
    if constexpr (sizeof(T) == 4) {
      word = pair_word_staged(mat + (uint64_t)a * la.ld, mat + (uint64_t)b * la.ld, n_rows, la.ld, w0,
                              pair_thr(la), lane, stage + (threadIdx.x >> 5) * kStageFloats);
    } else {
      word = pair_word_lane(mat + (uint64_t)a * la.ld, mat + (uint64_t)b * la.ld, n_rows, la.ld, w0 + lane,
                            pair_thr(la));
    }
    if (w0 + lane < wp) la.pool[(uint64_t)t * wp + w0 + lane] = word;
    __threadfence();
    __syncwarp();
    if (lane == 0 && atomicSub(la.left + t, 1u) == 1u) {  // the slot's last chunk: publish it
      __threadfence();
      la.keys[t] = kSlotEmpty;
      atomicExch(la.map + key, t);
    }
  }
}

// ---------------------------------------------------------------------------
// Cold batches of short vectors (float32 store): claim (lazy_claim_kernel),
// build every claimed slot here, publish (lazy_publish_kernel), then count
// with nothing left to build.  A pair vector built inside the count kernel
// reads both of its columns (2 x 80 KB at 20k rows) for 2.5 KB of output -- a
// C3 population's 48K first-visit vectors re-read the matrix ~100 times (11 GB
// of L2 traffic, 2.2 ms).  Here a CTA stages one 16-row slice of EVERY column
// (64 bytes per column) and builds that half-word of every slot in its part
// of the window from shared memory: a half-warp per slot -- lane i on row
// index_bit_row(i), so one ballot is two slots' half-words in index layout --
// the float32 bracket of the threshold, the double test only for the rare
// rows inside it.  Two CTAs per SM: one stages while the other builds.
//
// Units are (half-word h of the vectors, part of the slot window); the part
// count is chosen on the device so the units balance over the grid.


// THREADS = 512 (two CTAs per SM: one stages while the other builds) while
// two slices fit in shared memory (C <= ~1700), else 1024 (one CTA per SM).
__host__ __device__ constexpr uint32_t slab_build_smem(uint32_t n_cols, uint32_t threads) {
  return n_cols * 16 * 4 + (threads / 32) * 32 * 8;
}

template <uint32_t THREADS>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS)
lazy_slab_build_kernel(const LazyArgs la, uint32_t n_rows, uint32_t n_cols, uint32_t wp) {
  constexpr uint32_t kSlabBuildThreads = THREADS;
  const uint32_t start = la.start[la.seq % kLazyStartRing];
  const uint32_t end = lazy_window_end(la);
  if (end <= start) return;
  const uint32_t tag = lazy_tag(la.seq);
  constexpr int kWarps = kSlabBuildThreads / 32;
  const uint32_t n_halves = 2 * wp;
  // parts: >= 8 units per CTA, >= 2 slots per lane per part
  const uint32_t n_jobs = end - start;
  const uint32_t n_parts = max(1u, min((8u * gridDim.x + n_halves - 1) / n_halves, n_jobs / (2u * kSlabBuildThreads)));
  const uint32_t per_part = (n_jobs + n_parts - 1) / n_parts;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* mat = static_cast<const float*>(la.mat);
  const PairThr th = pair_thr(la);
  extern __shared__ float4 smem4[];
  float* sv = reinterpret_cast<float*>(smem4);                                   // [n_cols][16] values
  uint2* soff = reinterpret_cast<uint2*>(sv + (size_t)n_cols * 16) + warp * 32;  // the group's 32 (a, b) * 16
  const uint32_t row_off = 4u * index_bit_row((uint32_t)(lane & 15));  // this lane's row (0..15), bytes
  const uint32_t half_sel = (uint32_t)(lane & 16);                      // 0: slot j, 16: slot j + 16
  const unsigned char* sv_b = reinterpret_cast<const unsigned char*>(sv);
  auto lds_f32 = [&](uint32_t byte_off) { return *reinterpret_cast<const float*>(sv_b + byte_off); };
  uint16_t* pool16 = reinterpret_cast<uint16_t*>(la.pool);
  const uint64_t n_units = (uint64_t)n_halves * n_parts;
  for (uint64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const uint32_t hv = (uint32_t)(u / n_parts), part = (uint32_t)(u % n_parts);
    const uint32_t w = hv >> 1, hw = hv & 1;
    const uint32_t t_begin = start + part * per_part, t_end = min(end, t_begin + per_part);
    const uint32_t r0 = 32u * w + 16u * hw;
    // a half past the last row (the vector's padding words, wp rounded up) is
    // all zeros and is not staged: the store holds ld rows per column, and a
    // half with any valid row ends by 32 ceil(R / 32) <= ld
    const bool dead = r0 >= n_rows;
    __syncthreads();  // the previous slice is no longer read
    if (!dead) {
      constexpr int UNR = 4;  // loads in flight per thread
      const uint32_t total = n_cols * 4;
      for (uint32_t i0 = threadIdx.x; i0 < total; i0 += UNR * kSlabBuildThreads) {
        float4 x[UNR];
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t i = i0 + k * kSlabBuildThreads;
          if (i < total) x[k] = __ldg(reinterpret_cast<const float4*>(mat + (uint64_t)(i >> 2) * la.ld + r0) + (i & 3));
        }
#pragma unroll
        for (int k = 0; k < UNR; ++k) {
          const uint32_t i = i0 + k * kSlabBuildThreads;
          if (i < total) reinterpret_cast<float4*>(sv)[i] = x[k];
        }
      }
    }
    __syncthreads();
    const uint32_t valid = (index_valid_bits(n_rows, w) >> (16 * hw)) & 0xFFFFu;
    uint32_t tk_next = t_begin + 32u * warp + lane < t_end ? __ldcg(la.keys + t_begin + 32u * warp + lane) : kSlotEmpty;
    for (uint32_t t0 = t_begin + 32u * warp; t0 < t_end; t0 += 32u * kWarps) {
      const uint32_t t = t0 + lane;
      const uint32_t tk = tk_next;  // (loaded one group ahead)
      tk_next = t + 32u * kWarps < t_end ? __ldcg(la.keys + t + 32u * kWarps) : kSlotEmpty;
      const bool own = tk != kSlotEmpty && (tk >> kLazyKeyBits) == tag;
      const uint32_t key = tk & ((1u << kLazyKeyBits) - 1u);
      const uint32_t ka = own ? key / n_cols : 0u;
      // byte offsets of the slot's two column slices
      soff[lane] = make_uint2(ka * 64u, own ? (key - ka * n_cols) * 64u : 0u);
      const uint32_t own_m = __ballot_sync(kFull, own);
      __syncwarp();
      if (own_m && dead) {
        if (own) pool16[((uint64_t)t * wp + w) * 2 + hw] = 0;
      } else if (own_m) {
        bool unc = false;  // a row of this lane inside a bracket (rare): the double test below
        uint32_t hv = 0;   // ballot (lane & 15): this lane's slot's half-word in its low / high half
        // lanes 0..15: slot j, lanes 16..31: slot j + 16.  Software-pipelined:
        // the next two slots' offsets (one 16-byte load) and slot j + 1's
        // values are in flight while slot j is tested.
        const uint4* soff4 = reinterpret_cast<const uint4*>(soff + half_sel);
        uint4 o2 = soff4[0];
        float x_next = lds_f32(o2.x + row_off);
        float y_next = lds_f32(o2.y + row_off);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float x = x_next, y = y_next;
          if (j + 1 < 16) {
            if (j & 1) {
              o2 = soff4[(j + 1) >> 1];
              x_next = lds_f32(o2.x + row_off);
              y_next = lds_f32(o2.y + row_off);
            } else {
              x_next = lds_f32(o2.z + row_off);
              y_next = lds_f32(o2.w + row_off);
            }
          }
          const float ax = fabsf(x);
          const float tt = __fmaf_rn(-th.a_f, ax, x);
          const float d = bracket_halfwidth(ax, th.kscale);
          const bool above = y > __fadd_rn(tt, d);
          unc |= !above && y > __fsub_rn(tt, d);
          const uint32_t bal = __ballot_sync(kFull, above);
          hv = (lane & 15) == j ? bal : hv;
        }
        if (__any_sync(kFull, unc)) {
          // some row sits inside its bracket: redo the warp's ballots with the
          // reference's double test for those rows
          __syncwarp();
#pragma unroll 1
          for (int j = 0; j < 16; ++j) {
            const uint2 oj = soff[half_sel + j];
            const float x = lds_f32(oj.x + row_off), y = lds_f32(oj.y + row_off);
            const float ax = fabsf(x);
            const float tt = __fmaf_rn(-th.a_f, ax, x);
            const float d = bracket_halfwidth(ax, th.kscale);
            bool bit = y > __fadd_rn(tt, d);
            if (!bit && y > __fsub_rn(tt, d)) bit = (double)y > thr64((double)x, th.approx);
            const uint32_t bal = __ballot_sync(kFull, bit);
            hv = (lane & 15) == j ? bal : hv;
          }
        }
        // lane l: the half-word of slot t0 + l (ballot l & 15, low or high half)
        const uint32_t h = (hv >> half_sel) & 0xFFFFu;
        if (own) pool16[((uint64_t)t * wp + w) * 2 + hw] = (uint16_t)(h & valid);
      }
      __syncwarp();  // soff is refilled by the next group
    }
  }
}

// Publish the slots lazy_slab_build_kernel built for this batch (map[p] = t)
// and release their keys.  Runs after the build kernel on the same stream.
__global__ void __launch_bounds__(256) lazy_publish_kernel(const LazyArgs la) {
  const uint32_t start = la.start[la.seq % kLazyStartRing];
  const uint32_t end = lazy_window_end(la);
  const uint32_t tag = lazy_tag(la.seq);
  if (la.count_out && blockIdx.x == 0 && threadIdx.x == 0) {  // the fill after this batch's claims
    la.count_out[0] = *(volatile uint32_t*)la.count;
    __threadfence_system();
    la.count_out[1] = la.seq;
  }
  for (uint32_t t = start + blockIdx.x * blockDim.x + threadIdx.x; t < end; t += gridDim.x * blockDim.x) {
    const uint32_t tk = __ldcg(la.keys + t);
    if (tk == kSlotEmpty || (tk >> kLazyKeyBits) != tag) continue;
    la.keys[t] = kSlotEmpty;
    asm volatile("fence.proxy.async.global;" ::: "memory");  // (the count kernel reads the pool by TMA)
    atomicExch(la.map + (tk & ((1u << kLazyKeyBits) - 1u)), t);
  }
}

}  // namespace ebic
