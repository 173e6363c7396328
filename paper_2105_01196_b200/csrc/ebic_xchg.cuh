// ebic_xchg.cuh -- the row-sharded step's count reduction over peer memory.
//
// Row sharding: rank g evaluates the whole population on its
// row block; the global count of candidate i is the sum of the G partial
// counts.  Instead of an NCCL all_reduce, every rank owns an exchange WINDOW in
// its HBM, mapped into every peer (CUDA IPC over NVLink / NVSwitch):
//
//   window = [ header: 128 B (magic, world, max_cand, poison) |
//              flags: kMaxRanks x u64 (one 128-B line each) |
//              inbox[2][kMaxRanks][max_cand] u32 ]
//
// The header is written at create time and checked by every peer when it maps
// the window (ebic_xchg_open*): all ranks must agree on world and max_cand, or
// a push would land outside a smaller peer's inbox.
//
// xchg_sum_kernel, one launch per step after the count kernel (on the
// context's exchange stream, so step k's exchange overlaps step k+1's count):
//   1. push   -- CTA b stores its slice of this rank's partial counts into
//                slot [parity][rank] of EVERY rank's inbox (peer stores over
//                NVLink, a local store for itself).  A rank whose count
//                failed pushes zeros and poisons every window instead, so all
//                ranks stay on the same epoch and learn that the step failed;
//   2. signal -- system-scope fence, then one atomic add to flag[rank] of
//                every rank's window;
//   3. wait   -- until every rank's flag in this window has counted this
//                epoch's pushes from all its CTAs (bounded by a %globaltimer
//                deadline: a peer that never arrives raises the error flag
//                instead of hanging);
//   4. sum    -- the CTA's slice over the G slots (L1-bypassing loads) -> out.
//                On timeout or poison the slice is written as kXchgSentinel
//                (never a valid count: counts are < 2^31 rows) and *err is set
//                (4 = timeout, 5 = a peer failed), so stale counts are never
//                left in out.
// The inbox alternates between two parities by epoch: a rank can only push
// epoch e+2 into the buffer a peer read at epoch e after that peer has pushed
// epoch e+1, which it does only after finishing epoch e's sum (the exchange
// kernels of one rank are serialised on its exchange stream).  Exact: integer
// sums.
#pragma once
#include <cstdint>

namespace ebic {

constexpr int kMaxRanks = 16;
constexpr int kXchgCtas = 32;
constexpr uint64_t kXchgFlagStride = 16;  // u64 per flag (128 B: one line per writer)
constexpr uint64_t kXchgHeaderBytes = 128;
constexpr uint32_t kXchgMagic = 0xEB1C0C57u;
constexpr uint32_t kXchgSentinel = 0xFFFFFFFFu;

struct XchgHeader {  // first bytes of every window
  uint32_t magic, world, max_cand, poison;
};

struct XchgPeers {
  unsigned char* win[kMaxRanks];  // every rank's window (own included), device-accessible here
};

__host__ __device__ __forceinline__ uint64_t xchg_window_bytes(uint32_t max_cand) {
  return kXchgHeaderBytes + kMaxRanks * kXchgFlagStride * sizeof(uint64_t) +
         2ull * kMaxRanks * max_cand * sizeof(uint32_t);
}
__device__ __forceinline__ XchgHeader* xchg_header(unsigned char* win) { return reinterpret_cast<XchgHeader*>(win); }
__device__ __forceinline__ uint64_t* xchg_flags(unsigned char* win) {
  return reinterpret_cast<uint64_t*>(win + kXchgHeaderBytes);
}
__device__ __forceinline__ uint32_t* xchg_inbox(unsigned char* win, int parity, int slot, uint32_t max_cand) {
  return reinterpret_cast<uint32_t*>(win + kXchgHeaderBytes + kMaxRanks * kXchgFlagStride * sizeof(uint64_t)) +
         ((uint64_t)parity * kMaxRanks + slot) * max_cand;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// failed != 0: this rank's count did not run -- push zeros, poison every window.
__global__ void __launch_bounds__(256)
xchg_sum_kernel(const uint32_t* __restrict__ local, uint32_t n, XchgPeers peers, int world, int rank,
                uint64_t epoch, uint32_t max_cand, uint32_t* __restrict__ out, int* err, int failed,
                uint64_t timeout_ns) {
  const int parity = (int)(epoch & 1);
  const uint32_t i0 = (uint32_t)((uint64_t)blockIdx.x * n / gridDim.x);
  const uint32_t i1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * n / gridDim.x);
  // 1. push this rank's partial counts of the slice to every rank
  for (int g = 0; g < world; ++g) {
    uint32_t* dst = xchg_inbox(peers.win[g], parity, rank, max_cand);
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) dst[i] = failed ? 0u : local[i];
  }
  if (failed && blockIdx.x == 0 && threadIdx.x < (unsigned)world)
    atomicOr_system(&xchg_header(peers.win[threadIdx.x])->poison, 1u);
  // 2. make the pushes visible system-wide, then count this CTA in every rank's flag[rank]
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int g = 0; g < world; ++g)
      atomicAdd_system(reinterpret_cast<unsigned long long*>(xchg_flags(peers.win[g]) + rank * kXchgFlagStride),
                       1ull);
  // 3. wait for every rank's pushes of this epoch (all of its CTAs)
  __shared__ int s_status;
  if (threadIdx.x == 0) {
    const uint64_t want = epoch * gridDim.x;
    volatile uint64_t* flags = xchg_flags(peers.win[rank]);
    int status = 0;
    const uint64_t t0 = global_ns();
    for (int g = 0; g < world && !status; ++g) {
      while (flags[g * kXchgFlagStride] < want) {
        __nanosleep(256);
        if (global_ns() - t0 > timeout_ns) {  // a peer never arrived
          status = 4;
          break;
        }
      }
    }
    __threadfence_system();
    if (!status && *(volatile uint32_t*)&xchg_header(peers.win[rank])->poison) status = 5;
    if (status) atomicExch(err, status);
    s_status = status;
  }
  __syncthreads();
  if (s_status) {  // never leave stale counts behind
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) out[i] = kXchgSentinel;
    return;
  }
  // 4. sum the slice over the ranks' slots (bypassing L1: peers wrote them)
  for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    uint32_t s = 0;
    for (int g = 0; g < world; ++g) s += __ldcv(xchg_inbox(peers.win[rank], parity, g, max_cand) + i);
    out[i] = s;
  }
}

}  // namespace ebic
