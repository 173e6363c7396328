// ebic_xchg.cuh -- the row-sharded step's count reduction over peer memory.
//
// Row sharding: rank g evaluates the whole population on its
// row block; the global count of candidate i is the sum of the G partial
// counts.  Instead of an NCCL all_reduce, every rank owns an exchange WINDOW in
// its HBM, mapped into every peer (CUDA IPC over NVLink / NVSwitch):
//
//   window = [ flags: kMaxRanks x u64 (one 128-B line each) |
//              inbox[2][kMaxRanks][max_cand] u32 ]
//
// xchg_sum_kernel, one launch per step right after the count kernel:
//   1. push   -- CTA b stores its slice of this rank's partial counts into
//                slot [parity][rank] of EVERY rank's inbox (peer stores over
//                NVLink, a local store for itself);
//   2. signal -- system-scope fence, then one atomic add to flag[rank] of
//                every rank's window;
//   3. wait   -- until every rank's flag in this window has counted this
//                epoch's pushes from all its CTAs (bounded spin: a peer that
//                never arrives raises the error flag instead of hanging);
//   4. sum    -- the CTA's slice over the G slots (L1-bypassing loads) -> out.
// The inbox alternates between two parities by epoch: a rank can only push
// epoch e+2 into the buffer a peer read at epoch e after that peer has pushed
// epoch e+1, which it does only after finishing epoch e's sum (stream order).
// Exact: integer sums.
#pragma once
#include <cstdint>

namespace ebic {

constexpr int kMaxRanks = 16;
constexpr int kXchgCtas = 32;
constexpr uint64_t kXchgFlagStride = 16;  // u64 per flag (128 B: one line per writer)

struct XchgPeers {
  unsigned char* win[kMaxRanks];  // every rank's window (own included), device-accessible here
};

__device__ __forceinline__ uint64_t* xchg_flags(unsigned char* win) { return reinterpret_cast<uint64_t*>(win); }
__device__ __forceinline__ uint32_t* xchg_inbox(unsigned char* win, int parity, int slot, uint32_t max_cand) {
  return reinterpret_cast<uint32_t*>(win + kMaxRanks * kXchgFlagStride * sizeof(uint64_t)) +
         ((uint64_t)parity * kMaxRanks + slot) * max_cand;
}

__global__ void __launch_bounds__(256)
xchg_sum_kernel(const uint32_t* __restrict__ local, uint32_t n, XchgPeers peers, int world, int rank,
                uint64_t epoch, uint32_t max_cand, uint32_t* __restrict__ out, int* err) {
  const int parity = (int)(epoch & 1);
  const uint32_t i0 = (uint32_t)((uint64_t)blockIdx.x * n / gridDim.x);
  const uint32_t i1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * n / gridDim.x);
  // 1. push this rank's partial counts of the slice to every rank
  for (int g = 0; g < world; ++g) {
    uint32_t* dst = xchg_inbox(peers.win[g], parity, rank, max_cand);
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) dst[i] = local[i];
  }
  // 2. make the pushes visible system-wide, then count this CTA in every rank's flag[rank]
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    for (int g = 0; g < world; ++g)
      atomicAdd_system(reinterpret_cast<unsigned long long*>(xchg_flags(peers.win[g]) + rank * kXchgFlagStride),
                       1ull);
  // 3. wait for every rank's pushes of this epoch (all of its CTAs)
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const uint64_t want = epoch * gridDim.x;
    volatile uint64_t* flags = xchg_flags(peers.win[rank]);
    int ok = 1;
    for (int g = 0; g < world && ok; ++g) {
      uint32_t spins = 0;
      while (flags[g * kXchgFlagStride] < want) {
        __nanosleep(128);
        if (++spins > (1u << 24)) {  // ~2+ s: a peer never arrived
          ok = 0;
          atomicExch(err, 4);
          break;
        }
      }
    }
    __threadfence_system();
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  // 4. sum the slice over the ranks' slots (bypassing L1: peers wrote them)
  for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    uint32_t s = 0;
    for (int g = 0; g < world; ++g) s += __ldcv(xchg_inbox(peers.win[rank], parity, g, max_cand) + i);
    out[i] = s;
  }
}

}  // namespace ebic
