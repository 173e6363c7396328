// ebic_capi.cu -- host side of the C ABI declared in include/ebic.h.
//
// Replaces the reference's CPU evaluator (trend.cpp:48-72 on the WorkerPool of
// worker_pool.cpp:20-48) with: a device-resident column-major matrix store, the
// fitness_count / mask+scatter kernels of ebic_kernels.cuh, and a pinned-memory
// batch marshaller on one CUDA stream per context.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ebic.h"
#include "ebic_kernels.cuh"
#include "ebic_plane.cuh"
#include "ebic_simd.cuh"
#include "ebic_pair.cuh"
#include "ebic_table.cuh"
#include "ebic_xchg.cuh"

// NVTX ranges (header-only NVTX v3; no-ops unless a profiler is attached):
// every public entry point and every one-time build shows up by name on an
// nsys / ncu timeline ("ebic:<call>").
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define EBIC_CUDA(call)                                                                    \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(EBIC_ERR_CUDA, "%s:%d: %s: %s", __FILE__, __LINE__, #call,               \
                  cudaGetErrorString(e_));                                                 \
  } while (0)

#define EBIC_TRY(expr)            \
  do {                            \
    int s_ = (expr);              \
    if (s_ != EBIC_OK) return s_; \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
struct HostBuf {
  T* p = nullptr;
  size_t n = 0;
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
int ensure(DevBuf<T>& b, size_t n) {
  if (b.n >= n && b.p) return EBIC_OK;
  const size_t old = b.n;
  b.release();
  size_t cap = std::max<size_t>(std::max<size_t>(n, 1024), old + old / 2);
  EBIC_CUDA(cudaMalloc(&b.p, cap * sizeof(T)));
  b.n = cap;
  return EBIC_OK;
}

template <typename T>
int ensure(HostBuf<T>& b, size_t n) {
  if (b.n >= n && b.p) return EBIC_OK;
  const size_t old = b.n;
  b.release();
  size_t cap = std::max<size_t>(std::max<size_t>(n, 1024), old + old / 2);
  EBIC_CUDA(cudaMallocHost(&b.p, cap * sizeof(T)));
  b.n = cap;
  return EBIC_OK;
}

// ensure() for buffers whose contents must be zero when first used
template <typename T>
int ensure_zero(DevBuf<T>& b, size_t n, cudaStream_t s) {
  if (b.n >= n && b.p) return EBIC_OK;
  EBIC_TRY(ensure(b, n));
  EBIC_CUDA(cudaMemsetAsync(b.p, 0, b.n * sizeof(T), s));
  return EBIC_OK;
}

// Device alias of page-locked host memory (nullptr if the memory is not
// page-locked or not mapped into the device's address space).
void* dev_alias(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return static_cast<char*>(a.devicePointer) + 0;
}

struct Slot {
  HostBuf<uint32_t> h_cols, h_offs, h_counts;
  HostBuf<int> h_err;  // device-detected argument errors of this submission
  DevBuf<uint32_t> d_cols, d_offs, d_counts;
  cudaEvent_t done = nullptr;
  uint64_t ticket = 0;   // ticket currently occupying the slot (0 = free)
  uint32_t* user_counts = nullptr;
  uint64_t n_cand = 0;
};

}  // namespace

struct ebic_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;  // active stream (own or external)
  // matrix store
  void* d_mat = nullptr;
  int store = 0;  // EBIC_STORE_F32 / EBIC_STORE_F64 (0 = none)
  uint64_t n_rows = 0, n_cols = 0, ld = 0, row_base = 0;
  // scratch
  int* d_err = nullptr;
  int* d_flags = nullptr;
  int* d_out1 = nullptr;
  DevBuf<uint32_t> d_mask, d_rows, d_tmp_cols, d_tmp_offs, d_tmp_counts;
  DevBuf<uint64_t> d_row_offsets;
  HostBuf<uint32_t> h_tmp_counts;
  DevBuf<uint32_t> d_inter;  // ebic_support_overlap_batch: n x n intersections
  HostBuf<uint32_t> h_inter;
  // slab_pair_kernel: per-candidate partial-count accumulators and per-chunk
  // arrival counters, both zero between launches (the kernel re-zeroes them)
  DevBuf<uint32_t> d_acc, d_done;
  HostBuf<int> h_err1;  // page-locked, device-mapped: error flag of the zero-copy host path
  int* h_err1_dev = nullptr;  // its device alias
  // zero-copy host path, pipelined: input pieces DMA'd on copy_stream while the
  // previous piece is evaluated (piece_ev[k]: piece k has landed)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t piece_ev[5] = {};  // [kMaxPieces] arrivals + [kMaxPieces] "previous work done"
  // row-shard exchange window over peer memory (ebic_xchg.cuh)
  unsigned char* xchg_win = nullptr;               // this rank's window (device)
  unsigned char* xchg_peer[ebic::kMaxRanks] = {};  // every rank's window as mapped here
  bool xchg_ipc_opened[ebic::kMaxRanks] = {};      // peer windows opened through CUDA IPC
  int xchg_world = 0, xchg_rank = 0;
  uint64_t xchg_max = 0, xchg_epoch = 0;
  uint64_t xchg_timeout_ns = 10'000'000'000ull;    // EBIC_XCHG_TIMEOUT_MS (default 10 s)
  // Pipelining: step k counts into local[k % kXchgDepth] on the caller's
  // stream; its exchange runs on xchg_stream once the count has finished, so
  // step k+1's count overlaps step k's exchange.  cdone[s]: the count of the
  // step in ring slot s is done; xdone[s]: its exchange is done (the slot's
  // local buffer may be refilled).
  static constexpr int kXchgDepth = 2;
  cudaStream_t xchg_stream = nullptr;
  cudaEvent_t xchg_cdone[kXchgDepth] = {}, xchg_xdone[kXchgDepth] = {};
  bool xchg_xdone_armed[kXchgDepth] = {};
  DevBuf<uint32_t> d_xchg_local[kXchgDepth];       // this rank's partial counts, per ring slot
  // staged upload of pageable host matrices (staged_h2d): per worker thread a
  // stream and an event (the page-locked buffers are process-wide)
  struct Stager {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    bool armed = false;
  };
  std::vector<Stager> stagers;
  int pipeline_pieces = 1;       // EBIC_HOST_PIECES (1 = no pipelining; measured faster on B200 at 16K candidates)
  // EBIC_ZC_READ_MAX: page-locked inputs up to this many bytes are read in place
  // by the index kernel (measured: 29.1 -> 24.4 us at P = 392, 30.3 -> 28.4 us
  // at C2 (82 KB), 52.7 -> 58.7 us at C3 (327 KB): profiles/r2_e2e_small.txt)
  uint64_t zc_read_max = 128 * 1024;
  Slot slots[EBIC_MARSHAL_SLOTS];
  uint64_t next_ticket = 1;
  // tickets retired early (ring reuse / slot growth) whose device-side check failed
  std::vector<uint64_t> failed_tickets;
  uint64_t launches = 0;
  uint32_t slab_rows = 0;  // 0 = auto (value path)
  // rank plane (per matrix x approx)
  uint32_t* d_plane = nullptr;
  bool plane_valid = false;
  // pair-trend index (ebic_table.cuh), per matrix x approx; used when it fits
  // table_budget bytes.  Default budget: kDefaultBudgetFrac of the device
  // memory free at upload (counting a kept index allocation as free), so the
  // library never takes most of a shared GPU by itself; an explicit budget
  // (ebic_ctx_set_table_budget / EBIC_TABLE_BUDGET_MB) replaces the fraction
  // and is capped at the free memory minus a reserve of max(8 GiB, 10%).
  uint32_t* d_table = nullptr;
  bool table_valid = false, table_failed = false;
  double table_approx = 0.0;
  uint64_t table_budget = 0;
  uint64_t table_budget_user = 0;  // 0 = the default fraction
  bool full_requested = false;      // ebic_matrix_prepare asked for the full index
  // lazy pair-trend index (ebic_lazy.cuh), per matrix x approx: built pair by
  // pair inside the count kernel, kept in a pool that grows (stream-ordered
  // allocations) up to the budget and starts over when full
  uint32_t* d_lmap = nullptr;       // C x C slot per ordered pair
  uint32_t* d_lpool = nullptr;      // lcap x wp words
  uint32_t* d_lcount = nullptr;     // slots handed out (device)
  uint32_t* d_lkeys = nullptr;      // long vectors: per slot, the pair it was claimed for (lkcap slots)
  uint32_t* d_lleft = nullptr;      // long vectors: per slot, 32-word chunks still to build
  uint32_t* d_lstart = nullptr;     // long vectors: the count at the batch's start
  uint64_t lkcap = 0;
  // long vectors: per-batch scratch -- candidates the count kernel deferred
  // (lazy_deferred_kernel) and each candidate's first 31 pair slots
  // (lazy_claim_kernel) -- in a ring, so batches on different streams never
  // share one (a batch reusing a ring entry waits for its previous user)
  struct LazyScratch {
    DevBuf<uint32_t> defer, pslot;
    cudaEvent_t done = nullptr;
    bool armed = false;
  };
  static constexpr int kLazyScratch = 4;
  LazyScratch lscratch[kLazyScratch];
  uint64_t lcap = 0;                // pool capacity (slots)
  HostBuf<uint32_t> h_lmirror;      // page-locked, mapped: {count at a lazy kernel's start, its batch sequence}
  uint32_t* h_lmirror_dev = nullptr;
  bool lazy_valid = false;
  double lazy_approx = 0.0;
  uint32_t lazy_seq = 0, lazy_epoch_seq = 1;  // batch sequence; first batch of the current map epoch
  uint64_t lazy_built = 0;          // slots filled over all epochs of this (matrix, approx) (ski-rental rent)
  uint64_t lazy_epoch_seen = 0;     // slots of the current epoch already added to lazy_built
  uint64_t lazy_resets = 0;
  // fill samples (h_lmirror) -> is the pool still filling fast (ebic::LazyArgs::cold)?
  uint32_t lazy_sample_count = 0, lazy_sample_seq = 0;
  uint64_t lazy_recent_growth = 0;
  int lazy_build = EBIC_LAZY_BUILD_AUTO;  // EBIC_LAZY_BUILD / ebic_ctx_set_lazy_build
  bool lazy_shared_dirty = false;
  bool lazy_trace = false;  // EBIC_LAZY_TRACE: one line per lazy batch on stderr  // lazy state initialised on one stream, not yet synchronised
  int index_mode = 0;               // index used by the last counting launch (IndexMode)
  double plane_approx = 0.0;
  int path = EBIC_PATH_AUTO;
  int n_sms = 148;
  size_t smem_optin = 227 * 1024;
  int prefetch = -1;  // -1 auto, 0 off, 1 on (EBIC_PREFETCH)
  int plane_builder = 0;  // EBIC_PLANE_BUILDER: 0 auto, 1 per-row block builder, 2 row-tile builder
  uint64_t table_cap = 0;   // bytes allocated at d_table (kept across uploads for reuse)
  int table_build_a = 2;    // EBIC_TABLE_BUILD_A: a-columns per builder warp (1 or 2)
  int tma_slots = 0;       // EBIC_TMA_SLOTS: pair vectors in flight per warp in the TMA index kernel (2..4; 0 auto)
  int table_kernel = 0;    // EBIC_TABLE_KERNEL: 0 auto (lane groups up to 32 slices, TMA warps up to 256; beyond: warps if many candidates, else CTAs), 1 register-load warps, 2 CTAs, 3 TMA, 4 lane groups (A/B)
  int simd_force = 0;     // forced packed-pair layout P*16+SUB (ebic_ctx_set_pair_layout / EBIC_PAIR_LAYOUT="P,SUB"); 0 = auto
  bool pdl = true;         // programmatic dependent launch of the count kernels (EBIC_PDL=0 disables)
  // one-time build costs of the last (matrix, approx) preparation
  // (ebic_matrix_build_info): events around the plane and index kernels, host
  // clock around the index allocation (cudaMalloc is synchronous)
  cudaEvent_t ev_build[4] = {};  // plane start / plane end / index start / index end
  bool plane_timed = false, index_timed = false;
  double index_alloc_ms = 0.0;
};

namespace {

int set_device(ebic_ctx* ctx) {
  EBIC_CUDA(cudaSetDevice(ctx->device));
  return EBIC_OK;
}

ebic::TrendArgs make_args(double approx, int neg) {
  ebic::TrendArgs ta;
  ta.approx = approx;
  ta.a_f = (float)approx;
  // bracket half-width scale >= (1+|a|) * 2^-20; rounded up by a small factor
  ta.kscale = (float)((1.0 + std::fabs(approx)) * 0x1p-20 * 1.0001);
  ta.negative = neg ? 1 : 0;
  return ta;
}

int check_approx(double approx) {
  if (!std::isfinite(approx)) return fail(EBIC_ERR_INVALID_ARGUMENT, "approx must be finite");
  return EBIC_OK;
}

uint32_t pick_slab_rows(const ebic_ctx* ctx, uint64_t n_cand) {
  if (ctx->slab_rows) return ctx->slab_rows;
  // enough CTAs to fill 148 SMs several times, slabs small enough that the
  // concurrently resident working set (slab x all columns) stays in L2.
  const uint64_t groups = (n_cand + ebic::kWarps - 1) / ebic::kWarps;
  uint64_t slab = 2048;
  while (slab > ebic::kRowAlign && groups * ((ctx->n_rows + slab - 1) / slab) < 148 * 8) slab /= 2;
  return (uint32_t)std::max<uint64_t>(slab, ebic::kRowAlign);
}

template <typename T, int MODE, bool NEG, bool MASK>
void launch_count_t(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offs, uint64_t n_cand,
                    const ebic::TrendArgs& ta, uint32_t* d_counts, uint32_t* d_mask,
                    cudaStream_t s) {
  const uint32_t slab = pick_slab_rows(ctx, n_cand);
  dim3 grid((unsigned)((n_cand + ebic::kWarps - 1) / ebic::kWarps),
            (unsigned)((ctx->n_rows + slab - 1) / slab));
  ebic::fitness_count_kernel<T, MODE, NEG, MASK><<<grid, ebic::kThreads, 0, s>>>(
      static_cast<const T*>(ctx->d_mat), ctx->ld, (uint32_t)ctx->n_rows, (uint32_t)ctx->n_cols,
      d_cols, d_offs, (uint32_t)n_cand, slab, ta, d_counts, d_mask, ctx->d_err);
  ctx->launches++;
}

// ---- one-time build timing (ebic_matrix_build_info) --------------------------
int build_event(ebic_ctx* ctx, int k, cudaStream_t s) {
  if (!ctx->ev_build[k]) EBIC_CUDA(cudaEventCreate(&ctx->ev_build[k]));
  EBIC_CUDA(cudaEventRecord(ctx->ev_build[k], s));
  return EBIC_OK;
}

double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---- rank plane ------------------------------------------------------------
bool plane_fits(const ebic_ctx* ctx) { return ctx->n_cols >= 1 && ctx->n_cols <= ebic::kPlaneMaxCols; }

int ensure_plane(ebic_ctx* ctx, double approx, cudaStream_t s) {
  NvtxRange nvtx_("ebic:build_rank_plane");
  // bitwise comparison: -0.0 and 0.0 give identical thresholds, but keep it simple and exact
  if (ctx->plane_valid && std::memcmp(&ctx->plane_approx, &approx, sizeof(double)) == 0) return EBIC_OK;
  ctx->plane_valid = false;
  if (!ctx->d_plane) {
    EBIC_CUDA(cudaMalloc(&ctx->d_plane, ctx->ld * ctx->n_cols * sizeof(uint32_t)));
  }
  EBIC_TRY(build_event(ctx, 0, s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_plane, 0, ctx->ld * ctx->n_cols * sizeof(uint32_t), s));
  uint32_t pow2 = 1;
  while (pow2 < ctx->n_cols) pow2 <<= 1;
  const size_t esz = ctx->store == EBIC_STORE_F32 ? sizeof(float) : sizeof(double);
  const size_t smem = pow2 * esz;
  const unsigned grid = (unsigned)std::min<uint64_t>(ctx->n_rows, (uint64_t)ctx->n_sms * 8);
  // Row-tile builder (RG rows per CTA, register sort) for f32 rows of <= 1024
  // columns; otherwise the per-row block builder -- measured faster than the
  // warp-level shared-memory sort for wide or f64 rows (C4: 22.7 vs 26.8 ms).
  uint32_t rg = 8;
  while (rg > 1 && (size_t)rg * ((ctx->n_cols + 1) + pow2) * esz > 96 * 1024) rg >>= 1;
  const size_t tile_smem = (size_t)rg * ((ctx->n_cols + 1) + pow2) * esz;
  const bool tile = ctx->plane_builder == 2 || (ctx->plane_builder == 0 && ctx->store == EBIC_STORE_F32 &&
                                                ctx->n_cols <= 1024);
  if (tile && tile_smem <= 200 * 1024) {
    const unsigned g = (unsigned)std::min<uint64_t>((ctx->n_rows + rg - 1) / rg, (uint64_t)ctx->n_sms * 16);
    const uint32_t R = (uint32_t)ctx->n_rows, C = (uint32_t)ctx->n_cols;
    auto go = [&](auto kern, const auto* st) -> int {
      EBIC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem));
      kern<<<g, 256, tile_smem, s>>>(st, ctx->ld, R, C, pow2, rg, approx, ctx->d_plane);
      return EBIC_OK;
    };
    const float* sf = (const float*)ctx->d_mat;
    if (ctx->store != EBIC_STORE_F32) EBIC_TRY(go(ebic::build_plane_tile_kernel<double, 0>, (const double*)ctx->d_mat));
    else if (C <= 64) EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 2>, sf));
    else if (C <= 128) EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 4>, sf));
    else if (C <= 256) EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 8>, sf));
    else if (C <= 512) EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 16>, sf));
    else if (C <= 1024) EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 32>, sf));
    else EBIC_TRY(go(ebic::build_plane_tile_kernel<float, 0>, sf));
  } else if (ctx->store == EBIC_STORE_F32) {
    EBIC_CUDA(cudaFuncSetAttribute(ebic::build_plane_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ebic::build_plane_kernel<float><<<grid, 256, smem, s>>>((const float*)ctx->d_mat, ctx->ld, (uint32_t)ctx->n_rows,
                                                           (uint32_t)ctx->n_cols, pow2, approx, ctx->d_plane);
  } else {
    EBIC_CUDA(cudaFuncSetAttribute(ebic::build_plane_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ebic::build_plane_kernel<double><<<grid, 256, smem, s>>>((const double*)ctx->d_mat, ctx->ld, (uint32_t)ctx->n_rows,
                                                            (uint32_t)ctx->n_cols, pow2, approx, ctx->d_plane);
  }
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  EBIC_TRY(build_event(ctx, 1, s));
  ctx->plane_timed = true;
  ctx->plane_valid = true;
  ctx->plane_approx = approx;
  return EBIC_OK;
}

// Launch with the programmatic-stream-serialization attribute (PDL) when `pdl`.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Raise a kernel's dynamic shared-memory limit to the opt-in maximum, once per
// (kernel, device): the attribute call is a driver round trip, so it stays off
// the per-launch path.  Keyed by the kernel's address (the instantiations of
// one template share a function TYPE, so a per-type static would not do).
int allow_max_smem(const void* kern, const ebic_ctx* ctx) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == kern && d.second == ctx->device) return EBIC_OK;
  EBIC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ctx->smem_optin - 1024)));
  done.emplace_back(kern, ctx->device);
  return EBIC_OK;
}

// Resident CTAs per SM of a kernel at a block size / dynamic shared memory
// (cached: the occupancy query is a driver call).
int resident_ctas(const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, size_t>, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& c : cache)
    if (c.first.first == kern && c.first.second == smem) return c.second;
  int n = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  cache.push_back({{kern, smem}, std::max(1, n)});
  return std::max(1, n);
}

// ---- pair-trend index ------------------------------------------------------
// Device memory the index may take out of `free_bytes`: all but a reserve of
// max(8 GiB, 10%) for the caller's own buffers (a B200 has 180 GB of HBM: a
// 100-GB index for a 200k x 2000 matrix fits next to everything else).
uint64_t index_headroom(uint64_t free_bytes) {
  const uint64_t reserve = std::max<uint64_t>(8ull << 30, free_bytes / 10);
  return free_bytes > reserve ? free_bytes - reserve : 0;
}

// The index budget for `avail` bytes of device memory (free memory plus a kept
// index allocation): the explicit budget if one was set, else
// kDefaultBudgetFrac of avail; never more than the headroom.
constexpr double kDefaultBudgetFrac = 0.4;
uint64_t index_budget(const ebic_ctx* ctx, uint64_t avail) {
  const uint64_t head = index_headroom(avail);
  if (ctx->table_budget_user) return std::min<uint64_t>(ctx->table_budget_user, head);
  return std::min<uint64_t>(head, (uint64_t)((double)avail * kDefaultBudgetFrac));
}

constexpr int kTableNoMemory = -1;  // internal status: the index does not fit (fall back)

// Words per pair vector: whole uint4 slices, and whole 32-slice groups (128
// words, 512 B) above 128 words -- the register-load kernels read those with
// unpredicated loads, and the TMA kernel measured faster on 512-B-aligned
// vectors than on tight ones (C3: 27.4 us with 640 words vs 28.5 us with 628,
// 200-step A/B on one box, profiles/r1f_index_padding.txt).
uint64_t table_wp(const ebic_ctx* ctx) {
  const uint64_t words = (ctx->n_rows + 31) / 32;
  return words > 128 ? (words + 127) / 128 * 128 : (words + 3) / 4 * 4;
}
uint64_t table_bytes(const ebic_ctx* ctx) { return ctx->n_cols * ctx->n_cols * table_wp(ctx) * sizeof(uint32_t); }

bool table_allowed(const ebic_ctx* ctx) {
  if (!(ctx->path == EBIC_PATH_AUTO || ctx->path == EBIC_PATH_TABLE) || !plane_fits(ctx) || ctx->table_failed)
    return false;
  return ctx->path == EBIC_PATH_TABLE || table_bytes(ctx) <= ctx->table_budget;
}

// Build (or reuse) the index for `approx`.  kTableNoMemory if it cannot be
// allocated (the caller falls back to the slab kernels; not retried for this
// matrix).
int ensure_table(ebic_ctx* ctx, double approx, cudaStream_t s) {
  NvtxRange nvtx_("ebic:build_pair_trend_index");
  if (ctx->table_valid && std::memcmp(&ctx->table_approx, &approx, sizeof(double)) == 0) return EBIC_OK;
  EBIC_TRY(ensure_plane(ctx, approx, s));
  ctx->table_valid = false;
  if (ctx->d_table && ctx->table_cap < table_bytes(ctx)) {  // a kept allocation too small for this matrix
    cudaFree(ctx->d_table);
    ctx->d_table = nullptr;
    ctx->table_cap = 0;
  }
  ctx->index_alloc_ms = 0.0;
  if (!ctx->d_table) {
    const double t0 = host_ms();
    if (cudaMalloc(&ctx->d_table, table_bytes(ctx)) != cudaSuccess) {
      cudaGetLastError();
      ctx->d_table = nullptr;
      ctx->table_failed = true;
      return kTableNoMemory;
    }
    ctx->index_alloc_ms = host_ms() - t0;
    ctx->table_cap = table_bytes(ctx);
  }
  EBIC_TRY(build_event(ctx, 2, s));
  const uint32_t wp = (uint32_t)table_wp(ctx);
  // (row block, a tile) CTAs, times z slices of the b columns chosen so the
  // last wave is as full as possible (C3: 640 tiles = 2.2 waves of 2 CTAs per
  // SM unsliced; 3 slices = 6.5 waves)
  const uint64_t tiles = (uint64_t)((wp + 31) / 32) *
                         ((ctx->n_cols + ebic::kTableBuildWarps - 1) / ebic::kTableBuildWarps);
  const double slots = 2.0 * ctx->n_sms;  // resident builder CTAs (2 x 512 threads per SM)
  uint32_t z = 1;
  double best = 1e30;
  for (uint32_t zz = 1; zz <= 8 && (zz == 1 || ctx->n_cols / zz >= 64); ++zz) {
    const double waves = tiles * zz / slots;
    const double waste = std::ceil(waves) / waves;
    if (waste < best - 1e-9) {
      best = waste;
      z = zz;
    }
  }
  const uint32_t b_per_z = (uint32_t)(((ctx->n_cols + z - 1) / z + 1) / 2 * 2);
  z = (uint32_t)((ctx->n_cols + b_per_z - 1) / b_per_z);
  const dim3 grid((wp + 31) / 32, (unsigned)((ctx->n_cols + ebic::kTableBuildWarps - 1) / ebic::kTableBuildWarps), z);
  if (ctx->table_build_a == 2)
    ebic::build_pair_table_kernel<2><<<grid, ebic::kTableBuildWarps / 2 * 32, 0, s>>>(
        ctx->d_plane, ctx->ld, (uint32_t)ctx->n_rows, (uint32_t)ctx->n_cols, wp, ctx->d_table, b_per_z);
  else
    ebic::build_pair_table_kernel<1><<<grid, ebic::kTableBuildWarps * 32, 0, s>>>(
        ctx->d_plane, ctx->ld, (uint32_t)ctx->n_rows, (uint32_t)ctx->n_cols, wp, ctx->d_table, b_per_z);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  EBIC_TRY(build_event(ctx, 3, s));
  ctx->index_timed = true;
  ctx->table_valid = true;
  ctx->table_approx = approx;
  return EBIC_OK;
}

// ---- index policy: full pair-trend index, lazy index, or none ---------------
enum IndexMode { kIndexNone = 0, kIndexFull = 1, kIndexLazy = 2 };
constexpr uint64_t kLazyMaxCols = 8192;              // map of C^2 slots <= 256 MB
constexpr uint64_t kSmallFullIndex = 1ull << 30;     // a full index this small is built outright (ms)
constexpr double kLazyRentFrac = 0.5;                // ski rental: buy the full index once this share of
                                                     // the C^2 pairs has been built lazily
constexpr uint64_t kLazyColdGrowth = 1024;           // slots claimed between two fill samples that keep
                                                     // batches on the build-first (cold) route
constexpr uint64_t kLazyColdMinCand = 256;           // smaller batches always build inside the count kernel

// The lazy index runs in the TMA kernel (vectors of <= 256 uint4 slices, i.e.
// <= 32K rows per shard).
bool lazy_allowed(const ebic_ctx* ctx) {
  if (!(ctx->path == EBIC_PATH_AUTO || ctx->path == EBIC_PATH_LAZY)) return false;
  const uint64_t C = ctx->n_cols;
  return C >= 1 && C <= kLazyMaxCols;  // (the lazy index runs its own kernels whatever EBIC_TABLE_KERNEL says)
}

uint64_t lazy_map_bytes(const ebic_ctx* ctx) { return ctx->n_cols * ctx->n_cols * sizeof(uint32_t); }

void lazy_release(ebic_ctx* ctx, cudaStream_t s) {
  (void)s;  // (cudaFree waits for the device's work in flight)
  if (ctx->d_lpool) cudaFree(ctx->d_lpool);
  if (ctx->d_lkeys) cudaFree(ctx->d_lkeys);
  if (ctx->d_lleft) cudaFree(ctx->d_lleft);
  ctx->d_lpool = ctx->d_lkeys = ctx->d_lleft = nullptr;
  ctx->lcap = ctx->lkcap = 0;
  ctx->lazy_valid = false;
}

// Start a new map epoch (first use, new approx, or a full pool): every pair
// is unbuilt again.  Stream-ordered, so in-flight batches keep their vectors.
int lazy_new_epoch(ebic_ctx* ctx, cudaStream_t s) {
  EBIC_CUDA(cudaMemsetAsync(ctx->d_lmap, 0xFF, lazy_map_bytes(ctx), s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_lcount, 0, sizeof(uint32_t), s));
  ctx->lazy_shared_dirty = true;
  ctx->lazy_epoch_seq = ctx->lazy_seq + 1;
  ctx->lazy_epoch_seen = 0;
  ctx->lazy_sample_count = ctx->lazy_sample_seq = 0;
  ctx->lazy_recent_growth = 0;
  return EBIC_OK;
}

// Make room for a batch that may need `worst` new vectors, without a host
// sync: the mirror tells how full the pool was when some earlier batch
// started.  Grows the pool (cudaMalloc + copy on the stream + cudaFree of the
// old one) up to the budget, or starts a new epoch when it cannot grow.  An
// underestimate is still exact: a pair that finds no free slot is built
// privately (short vectors) or computed by the count kernel (long ones).
int lazy_reserve(ebic_ctx* ctx, double approx, uint64_t worst, cudaStream_t s, ebic::LazyArgs* la) {
  NvtxRange nvtx_("ebic:lazy_reserve");
  const double t_enter = ctx->lazy_trace ? host_ms() : 0.0;
  const uint64_t vec_bytes = table_wp(ctx) * sizeof(uint32_t);
  if (!ctx->d_lmap) {
    EBIC_CUDA(cudaMalloc(&ctx->d_lmap, lazy_map_bytes(ctx)));
    ctx->lazy_valid = false;
  }
  if (!ctx->d_lcount) EBIC_CUDA(cudaMalloc(&ctx->d_lcount, sizeof(uint32_t)));
  if (!ctx->h_lmirror.p) {
    EBIC_TRY(ensure(ctx->h_lmirror, 2));
    ctx->h_lmirror.p[0] = ctx->h_lmirror.p[1] = 0;
    ctx->h_lmirror_dev = static_cast<uint32_t*>(dev_alias(ctx->h_lmirror.p));
  }
  if (!ctx->lazy_valid || std::memcmp(&ctx->lazy_approx, &approx, sizeof(double)) != 0) {
    if (ctx->lazy_valid) EBIC_CUDA(cudaDeviceSynchronize());  // (another approx's batches may be in flight)
    EBIC_TRY(lazy_new_epoch(ctx, s));
    ctx->lazy_valid = true;
    ctx->lazy_approx = approx;
    ctx->lazy_built = 0;
  }
  // lagged fill of the pool
  const uint32_t m_count = *(volatile uint32_t*)&ctx->h_lmirror.p[0];
  const uint32_t m_seq = *(volatile uint32_t*)&ctx->h_lmirror.p[1];
  uint64_t used = 0;
  const bool observed = m_seq >= ctx->lazy_epoch_seq && m_seq <= ctx->lazy_seq;
  if (observed) {
    used = std::min<uint64_t>(m_count, ctx->lcap);
    if (used > ctx->lazy_epoch_seen) {
      ctx->lazy_built += used - ctx->lazy_epoch_seen;
      ctx->lazy_epoch_seen = used;
    }
    // growth between the two latest distinct samples (a sample is taken at
    // the start of a lazy kernel and after a cold batch's claims)
    if (m_seq != ctx->lazy_sample_seq || m_count != ctx->lazy_sample_count) {
      ctx->lazy_recent_growth = m_count > ctx->lazy_sample_count ? m_count - ctx->lazy_sample_count : 0;
      ctx->lazy_sample_count = m_count;
      ctx->lazy_sample_seq = m_seq;
    }
  }
  // cold: nothing observed yet in this epoch, or the pool grew by many slots
  // recently -- the batch probably brings many new pairs (first calls, a new
  // population), which a separate build pass makes ~5x cheaper
  la->cold = ctx->lazy_build == EBIC_LAZY_BUILD_FIRST ||
             (ctx->lazy_build == EBIC_LAZY_BUILD_AUTO && (!observed || ctx->lazy_recent_growth >= kLazyColdGrowth));
  // Room for this batch at its worst case.  Batches issued since the
  // mirror's sample are not counted at theirs: a GA's populations (and a
  // cycled benchmark pool) reuse most pairs, so a sum of worst cases grows
  // the pool -- or restarts it -- for pairs that never come.  An
  // underestimate stays exact: a claim past the capacity is computed by the
  // count kernel itself.  A new pool holds three worst-case batches.
  const uint64_t c2 = ctx->n_cols * ctx->n_cols;
  const uint64_t budget = ctx->table_budget > lazy_map_bytes(ctx) ? ctx->table_budget - lazy_map_bytes(ctx) : 0;
  const uint64_t max_slots = std::max<uint64_t>(1, std::min<uint64_t>({c2, budget / vec_bytes, 0x7fffffffull}));
  const uint64_t need_raw = used + worst;
  const uint64_t need = std::min<uint64_t>(need_raw, max_slots);
  if (need_raw > ctx->lcap) {
    if (ctx->lcap < max_slots) {
      // room for ~3 batches of this size: the mirror lags by a batch or two,
      // so a pool sized for one batch would grow again on the next call
      const uint64_t cap = std::min<uint64_t>(max_slots, std::max<uint64_t>({need + 2 * worst, 2 * ctx->lcap, 4096}));
      // cudaMalloc, not the stream-ordered allocator: measured on B200, making
      // 4 GB usable takes 4 ms with cudaMalloc and 120 ms with cudaMallocAsync
      // from the default pool (profiles/r2_alloc_cost.txt).  Freeing the old
      // pool waits for the copy (cudaFree synchronises): growth is rare.
      uint32_t* np = nullptr;
      if (cudaMalloc(reinterpret_cast<void**>(&np), cap * vec_bytes) != cudaSuccess) {
        cudaGetLastError();  // cannot grow: stay at this capacity (warps build private copies)
      } else {
        if (ctx->d_lpool) {
          // batches on other streams may still be writing the old pool (their
          // builds): let them finish before it is copied (growth is rare)
          EBIC_CUDA(cudaDeviceSynchronize());
          EBIC_CUDA(cudaMemcpyAsync(np, ctx->d_lpool, ctx->lcap * vec_bytes, cudaMemcpyDeviceToDevice, s));
          ctx->lazy_shared_dirty = true;
          EBIC_CUDA(cudaFree(ctx->d_lpool));
        }
        ctx->d_lpool = np;
        ctx->lcap = cap;
      }
    } else if (ctx->lcap < c2) {
      // the pool cannot grow and this batch may not fit: start over (a pool
      // of all C^2 pairs never fills)
      ++ctx->lazy_resets;
      // (slots are handed out again from 0: batches on other streams must not
      // be building the old epoch's slots any more)
      EBIC_CUDA(cudaDeviceSynchronize());
      EBIC_TRY(lazy_new_epoch(ctx, s));
    }
  }
  if (ctx->lkcap < ctx->lcap) {
    // per-slot claim bookkeeping of the claim / build kernels (long vectors,
    // cold batches of short ones; only read within one batch: no copy)
    uint32_t *nk = nullptr, *nl = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&nk), ctx->lcap * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&nl), ctx->lcap * sizeof(uint32_t)) != cudaSuccess) {
      cudaGetLastError();
      if (nk) cudaFree(nk);
      return fail(EBIC_ERR_CUDA, "lazy index: cannot allocate %llu slots of bookkeeping",
                  (unsigned long long)ctx->lcap);
    }
    EBIC_CUDA(cudaMemsetAsync(nk, 0xFF, ctx->lcap * sizeof(uint32_t), s));  // kSlotEmpty: nothing claimed
    ctx->lazy_shared_dirty = true;
    if (ctx->d_lkeys) cudaFree(ctx->d_lkeys);
    if (ctx->d_lleft) cudaFree(ctx->d_lleft);
    ctx->d_lkeys = nk;
    ctx->d_lleft = nl;
    ctx->lkcap = ctx->lcap;
  }
  if (!ctx->d_lstart) EBIC_CUDA(cudaMalloc(&ctx->d_lstart, 2 * ebic::kLazyStartRing * sizeof(uint32_t)));
  if (ctx->lazy_shared_dirty) {
    // the map / count / keys were (re)initialised or the pool copied on this
    // stream: batches the caller issues next on OTHER streams must not see
    // them half done (fresh cudaMalloc memory can hold a previous map's slot
    // numbers).  First use, growth and resets only.
    EBIC_CUDA(cudaStreamSynchronize(s));
    ctx->lazy_shared_dirty = false;
  }
  const uint32_t seq = ++ctx->lazy_seq;
  if (ctx->lazy_trace)
    std::fprintf(stderr,
                 "lazy: seq %u stream %p cold %d used %llu (sample %u/%u growth %llu) cap %llu worst %llu "
                 "reserve %.3f ms\n",
                 seq, (void*)s, la->cold, (unsigned long long)used, m_count, m_seq,
                 (unsigned long long)ctx->lazy_recent_growth, (unsigned long long)ctx->lcap,
                 (unsigned long long)worst, host_ms() - t_enter);
  la->map = ctx->d_lmap;
  la->pool = ctx->d_lpool;
  la->count = ctx->d_lcount;
  la->count_out = ctx->h_lmirror_dev;
  la->cap = (uint32_t)ctx->lcap;
  la->seq = seq;
  la->mat = ctx->d_mat;
  la->ld = ctx->ld;
  la->f64 = ctx->store == EBIC_STORE_F64 ? 1 : 0;
  la->approx = approx;
  {
    const ebic::TrendArgs ta = make_args(approx, 0);
    la->a_f = ta.a_f;
    la->kscale = ta.kscale;
  }
  la->keys = ctx->d_lkeys;
  la->left = ctx->d_lleft;
  la->start = ctx->d_lstart;
  return EBIC_OK;
}

// Which index serves this evaluation (IndexMode in *mode; kIndexNone: the
// slab / value kernels).  The full index is built on first use when the path
// forces it, when it is small (<= 1 GiB: milliseconds), when
// ebic_matrix_prepare asked for it, when the lazy index cannot serve the
// matrix, or -- ski rental -- once the lazy index has built kLazyRentFrac of
// all C^2 pairs (the work already spent is then about what the full build
// costs, and every later batch saves the lazy lookups); always within the
// budget.  Otherwise the lazy index (ebic_lazy.cuh) builds just the pairs the
// batches use.  `worst` bounds the new pairs this batch can need.
int use_index(ebic_ctx* ctx, double approx, uint64_t worst, cudaStream_t s, int* mode, ebic::LazyArgs* la) {
  *mode = kIndexNone;
  if (ctx->path == EBIC_PATH_TABLE && !table_allowed(ctx))
    return fail(EBIC_ERR_INVALID_ARGUMENT, "pair-trend index unavailable for this matrix (%llu columns)",
                (unsigned long long)ctx->n_cols);
  const bool lazy_ok = lazy_allowed(ctx);
  if (table_allowed(ctx)) {
    const bool have = ctx->table_valid && std::memcmp(&ctx->table_approx, &approx, sizeof(double)) == 0;
    const bool rent_paid = ctx->lazy_valid && std::memcmp(&ctx->lazy_approx, &approx, sizeof(double)) == 0 &&
                           (double)ctx->lazy_built >= kLazyRentFrac * (double)(ctx->n_cols * ctx->n_cols);
    if (have || ctx->path == EBIC_PATH_TABLE || !lazy_ok || table_bytes(ctx) <= kSmallFullIndex ||
        ctx->full_requested || rent_paid) {
      const int st = ensure_table(ctx, approx, s);
      if (st == EBIC_OK) {
        if (ctx->d_lpool) lazy_release(ctx, s);  // the full index replaces the pool
        *mode = kIndexFull;
        ctx->index_mode = kIndexFull;
        return EBIC_OK;
      }
      if (st != kTableNoMemory) return st;
      if (ctx->path == EBIC_PATH_TABLE)
        return fail(EBIC_ERR_CUDA, "pair-trend index (%llu bytes) does not fit in device memory",
                    (unsigned long long)table_bytes(ctx));
    }
  }
  if (lazy_ok && !(ctx->d_mat && ctx->n_rows == 0)) {
    EBIC_TRY(lazy_reserve(ctx, approx, worst, s, la));
    *mode = kIndexLazy;
    ctx->index_mode = kIndexLazy;
    return EBIC_OK;
  }
  if (ctx->path == EBIC_PATH_LAZY)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "lazy pair-trend index unavailable for this matrix (%llu x %llu)",
                (unsigned long long)ctx->n_rows, (unsigned long long)ctx->n_cols);
  ctx->index_mode = kIndexNone;
  return EBIC_OK;
}

// True when launch_table takes the TMA kernel (short pair vectors).
bool tma_table_kernel(const ebic_ctx* ctx) {
  return table_wp(ctx) / 4 <= 256 && (ctx->table_kernel == 0 || ctx->table_kernel == 3);
}

// The index one counting launch uses (use_index), decided once per launch.
struct IndexPlan {
  int mode = kIndexNone;
  ebic::LazyArgs la{};
};

// Worst-case new pair vectors of a batch (n_idx unknown on the device API:
// an estimate; an underestimate only costs private builds, never exactness).
uint64_t worst_pairs(uint64_t n_cand, uint64_t n_idx, int neg) {
  const uint64_t pairs = n_idx != 0xffffffffull && n_idx >= n_cand ? n_idx - n_cand : 4 * n_cand;
  return pairs * (neg ? 2 : 1);
}

// lazy_slab_build_kernel: 512 threads x 2 CTAs per SM while two slices fit
// in shared memory, else 1024 threads x 1 (C up to ~3400 at 227 KB).
bool slab_build_fits(const ebic_ctx* ctx) {
  return ctx->store == EBIC_STORE_F32 && ebic::slab_build_smem((uint32_t)ctx->n_cols, 1024) <= ctx->smem_optin;
}
int launch_slab_build(ebic_ctx* ctx, const ebic::LazyArgs& la, uint32_t wp, cudaStream_t s) {
  const uint32_t C = (uint32_t)ctx->n_cols;
  auto go = [&](auto kern, uint32_t threads) -> int {
    const size_t smem = ebic::slab_build_smem(C, threads);
    EBIC_TRY(allow_max_smem(reinterpret_cast<const void*>(kern), ctx));
    const unsigned grid = (unsigned)ctx->n_sms *
        (unsigned)std::max(1, resident_ctas(reinterpret_cast<const void*>(kern), (int)threads, smem));
    kern<<<grid, threads, smem, s>>>(la, (uint32_t)ctx->n_rows, C, wp);
    EBIC_CUDA(cudaGetLastError());
    return EBIC_OK;
  };
  if (2 * (ebic::slab_build_smem(C, 512) + 1024) <= ctx->smem_optin + 1024)
    return go(ebic::lazy_slab_build_kernel<512>, 512);
  return go(ebic::lazy_slab_build_kernel<1024>, 1024);
}

// Counts WRITTEN to out (any device-accessible pointer), optional row masks.
// n_idx bounds the offsets (checked on device).
template <bool MASK>
int launch_table(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offs, uint64_t n_cand, uint64_t n_idx,
                 int neg, uint32_t* out, int* err_out, uint32_t* d_mask, cudaStream_t s, const IndexPlan& plan) {
  const uint32_t nv = (uint32_t)(table_wp(ctx) / 4);
  const bool lazy = plan.mode == kIndexLazy;
  // enough warps per SM for the (pipelined) multi-pass kernel (measured
  // better than a CTA per candidate down to ~1000 candidates: C5's 1024 of
  // 1M rows 0.29 -> 0.21 ms); below that a CTA per candidate streams better
  const bool many = n_cand >= (uint64_t)ctx->n_sms * 6;
  if (!lazy && nv <= 32 && (ctx->table_kernel == 0 || ctx->table_kernel == 4) && !MASK) {
    // tiny vectors (R <= 4096 rows): a group of next_pow2(nv) lanes per
    // candidate, register loads (table_count_group_kernel)
    // lanes per candidate GL <= 8 (at least 4 candidates per warp), J = nv / GL
    // slices per lane: nv 1, 2, 4 -> GL = nv; up to 8 -> 8 x 1; beyond: 8 x
    // ceil(nv / 8) (20 slices: 8 x 3, not 8 x 4)
    const int GL = nv <= 1 ? 1 : nv <= 2 ? 2 : nv <= 4 ? 4 : 8;
    const int J = (int)((nv + 7) / 8);
    const uint64_t per_cta = 8ull * (32 / GL);
    const unsigned grid = (unsigned)std::min<uint64_t>((n_cand + per_cta - 1) / per_cta, (uint64_t)ctx->n_sms * 8);
    auto go = [&](auto kern) -> cudaError_t {
      // programmatic dependent launch, as the TMA kernel: back-to-back batches
      // overlap one kernel's tail with the next one's start
      return launch_pdl(kern, dim3(grid), dim3(256), 0, s, ctx->pdl, (const uint32_t*)ctx->d_table,
                        (uint32_t)ctx->n_cols, (uint32_t)table_wp(ctx), (uint32_t)ctx->n_rows, d_cols, d_offs,
                        (uint32_t)n_cand, (uint32_t)n_idx, out, err_out ? err_out : ctx->d_err);
    };
    auto pick = [&](auto negc) -> cudaError_t {
      constexpr bool N = decltype(negc)::value;
      if (GL == 1) return go(ebic::table_count_group_kernel<1, 1, 4, N>);
      if (GL == 2) return go(ebic::table_count_group_kernel<2, 1, 4, N>);
      if (GL == 4) return go(ebic::table_count_group_kernel<4, 1, 4, N>);
      if (J == 1) return go(ebic::table_count_group_kernel<8, 1, 4, N>);
      if (J == 2) return go(ebic::table_count_group_kernel<8, 2, 4, N>);
      if (J == 3) return go(ebic::table_count_group_kernel<8, 3, 2, N>);
      return go(ebic::table_count_group_kernel<8, 4, 2, N>);
    };
    EBIC_CUDA(neg ? pick(std::true_type{}) : pick(std::false_type{}));
    ctx->launches++;
    return EBIC_OK;
  }
  if (lazy && nv > 256) {
    // long vectors from the lazy index: claim the batch's missing pairs, build
    // them (ebic_lazy.cuh), then count through the pool
    const uint32_t wp = (uint32_t)table_wp(ctx);
    auto& sc = ctx->lscratch[plan.la.seq % ebic_ctx::kLazyScratch];
    if (!sc.done) EBIC_CUDA(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming));
    if (sc.armed) EBIC_CUDA(cudaStreamWaitEvent(s, sc.done, 0));
    EBIC_TRY(ensure(sc.defer, n_cand + 1));  // (a reallocation's cudaFree waits for the device)
    EBIC_TRY(ensure(sc.pslot, n_cand * 64));
    ebic::LazyArgs la = plan.la;
    la.defer = sc.defer.p;
    la.pslot = sc.pslot.p;
    EBIC_CUDA(cudaMemcpyAsync(ctx->d_lstart + la.seq % ebic::kLazyStartRing, ctx->d_lcount, sizeof(uint32_t),
                              cudaMemcpyDeviceToDevice, s));
    const unsigned cgrid = (unsigned)std::min<uint64_t>((n_cand + 7) / 8, (uint64_t)ctx->n_sms * 16);
    ebic::lazy_claim_kernel<<<cgrid, 256, 0, s>>>(la, d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx,
                                                  (uint32_t)ctx->n_cols, (wp + 31) / 32, neg);
    EBIC_CUDA(cudaMemcpyAsync(ctx->d_lstart + ebic::kLazyStartRing + la.seq % ebic::kLazyStartRing, ctx->d_lcount,
                              sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));  // the window end (lazy_window_end)
    const unsigned bgrid = (unsigned)ctx->n_sms * 8;
    if (slab_build_fits(ctx) && ctx->lazy_build != EBIC_LAZY_BUILD_INLINE) {
      // 16-row slices of every column staged once per unit (the cold-batch
      // builder of the short path), then publish: the claimed slots are then
      // all ready for the count kernel
      EBIC_TRY(launch_slab_build(ctx, la, wp, s));
      ebic::lazy_publish_kernel<<<(unsigned)ctx->n_sms * 2, 256, 0, s>>>(la);
      ctx->launches++;
    } else if (ctx->store == EBIC_STORE_F64)
      ebic::lazy_build_kernel<double><<<bgrid, 256, 0, s>>>(la, (uint32_t)ctx->n_rows, (uint32_t)ctx->n_cols, wp);
    else {
      const size_t smem = 8 * ebic::kStageFloats * sizeof(float);
      EBIC_TRY(allow_max_smem(reinterpret_cast<const void*>(ebic::lazy_build_kernel<float>), ctx));
      const unsigned fgrid = (unsigned)ctx->n_sms *
          (unsigned)std::max(1, resident_ctas(reinterpret_cast<const void*>(ebic::lazy_build_kernel<float>), 256, smem));
      ebic::lazy_build_kernel<float><<<fgrid, 256, smem, s>>>(la, (uint32_t)ctx->n_rows, (uint32_t)ctx->n_cols, wp);
    }
    auto go = [&](auto kern) -> cudaError_t {
      // a warp per candidate for the whole population (the block scheduler
      // balances the tail better than a grid-stride loop over fewer warps);
      // a plain launch: it reads the pool the build kernel just wrote, so it
      // must not overlap it (no PDL attribute: the kernel's pdl_* are no-ops)
      const unsigned grid = (unsigned)std::min<uint64_t>((n_cand + 7) / 8, 1u << 30);
      return launch_pdl(kern, dim3(grid), dim3(256), 0, s, false, (const uint32_t*)nullptr, (uint32_t)ctx->n_cols,
                        wp, (uint32_t)ctx->n_rows, d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx, out,
                        err_out ? err_out : ctx->d_err, d_mask, (uint64_t)(ctx->ld / 32), la);
    };
    EBIC_CUDA(neg ? go(ebic::table_count_warp_multi_kernel<8, true, MASK, true, true>)
                  : go(ebic::table_count_warp_multi_kernel<8, false, MASK, true, true>));
    // candidates with a pair not in the pool (rare): computed from the store
    const unsigned dgrid = (unsigned)ctx->n_sms * 2;
    auto god = [&](auto kern) {
      kern<<<dgrid, 256, 0, s>>>(la, (uint32_t)ctx->n_cols, wp, (uint32_t)ctx->n_rows, d_cols, d_offs, out, d_mask,
                                 ctx->ld / 32);
    };
    if (neg) god(ebic::lazy_deferred_kernel<true, MASK>);
    else god(ebic::lazy_deferred_kernel<false, MASK>);
    EBIC_CUDA(cudaEventRecord(sc.done, s));
    sc.armed = true;
    ctx->launches += 4;
    EBIC_CUDA(cudaGetLastError());
    return EBIC_OK;
  }
  if (!lazy && nv > 256 && (ctx->table_kernel == 1 || (ctx->table_kernel == 0 && many))) {
    // long vectors, many candidates: a warp per candidate sweeping its vectors
    // in passes of 256 slices (no block barriers; measured 0.44 vs 0.67 ms for
    // the CTA kernel at 200k x 2000, P = 32768, before the pipelining that
    // took it to 0.41).  Very few candidates keep the CTA kernel, which puts
    // a whole CTA on each.
    auto go = [&](auto kern) -> cudaError_t {
      // a warp per candidate for the whole population (the block scheduler
      // balances the tail better than a grid-stride loop over fewer warps);
      // programmatic dependent launch like the short-vector kernels
      const unsigned grid = (unsigned)std::min<uint64_t>((n_cand + 7) / 8, 1u << 30);
      return launch_pdl(kern, dim3(grid), dim3(256), 0, s, ctx->pdl, (const uint32_t*)ctx->d_table,
                        (uint32_t)ctx->n_cols, (uint32_t)table_wp(ctx), (uint32_t)ctx->n_rows, d_cols, d_offs,
                        (uint32_t)n_cand, (uint32_t)n_idx, out, err_out ? err_out : ctx->d_err, d_mask,
                        (uint64_t)(ctx->ld / 32), ebic::LazyArgs{});
    };
    EBIC_CUDA(neg ? go(ebic::table_count_warp_multi_kernel<8, true, MASK>)
                  : go(ebic::table_count_warp_multi_kernel<8, false, MASK>));
    ctx->launches++;
    return EBIC_OK;
  }
  if (lazy || tma_table_kernel(ctx)) {
    // short vectors (the default): through the TMA engine -- bulk copies of
    // whole pair vectors into per-warp shared-memory slots, mbarrier
    // completion (27.5 vs 31 us for the register-load warp kernel at C3, ncu).
    // The lazy index always runs here (S = 2).
    const uint32_t J = (nv + 31) / 32;
    // slots per warp: 2 (more CTAs per SM) when warps loop over several
    // candidates; 4 -- every pair of a candidate of up to 5 columns in one
    // round of copies -- when there is about one candidate per warp and the
    // launch is one latency-bound chain (measured: P = 392 +23%, C2 +6%)
    auto slots_smem = [&](int k) { return (size_t)ebic::kTmaWarps * k * (neg ? 2 : 1) * table_wp(ctx) * 4 + 512; };
    int S = lazy ? 2 : ctx->tma_slots ? ctx->tma_slots : n_cand <= (uint64_t)ctx->n_sms * 32 ? 4 : 2;
    while (S > 2 && slots_smem(S) > ctx->smem_optin) --S;
    const size_t smem = slots_smem(S);
    bool pdl = ctx->pdl;
    if (lazy && plan.la.cold && slab_build_fits(ctx) &&
        (n_cand >= kLazyColdMinCand || ctx->lazy_build == EBIC_LAZY_BUILD_FIRST)) {
      // a cold batch (the pool still filling fast): claim its missing pairs,
      // build them from 32-row slices of the whole matrix staged once per CTA
      // (lazy_slab_build_kernel), publish, then count -- nothing left to build
      // inside the count kernel (which runs without PDL: it reads what the
      // publish kernel wrote)
      const uint32_t wp = (uint32_t)table_wp(ctx);
      ebic::LazyArgs la = plan.la;
      la.defer = nullptr;
      la.pslot = nullptr;
      EBIC_CUDA(cudaMemcpyAsync(ctx->d_lstart + la.seq % ebic::kLazyStartRing, ctx->d_lcount, sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
      const unsigned cgrid = (unsigned)std::min<uint64_t>((n_cand + 7) / 8, (uint64_t)ctx->n_sms * 16);
      ebic::lazy_claim_kernel<<<cgrid, 256, 0, s>>>(la, d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx,
                                                    (uint32_t)ctx->n_cols, 1, neg);
      EBIC_CUDA(cudaMemcpyAsync(ctx->d_lstart + ebic::kLazyStartRing + la.seq % ebic::kLazyStartRing, ctx->d_lcount,
                                sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));  // the window end
      EBIC_TRY(launch_slab_build(ctx, la, wp, s));
      ebic::lazy_publish_kernel<<<(unsigned)ctx->n_sms * 2, 256, 0, s>>>(la);
      ctx->launches += 3;
      pdl = false;
    }
    auto go = [&](auto kern) -> int {
      EBIC_TRY(allow_max_smem(reinterpret_cast<const void*>(kern), ctx));
      // persistent warps: as many CTAs as are resident at once (the kernel
      // pipelines each warp's candidates), never more than the candidates need
      const uint64_t per_sm = (uint64_t)resident_ctas(reinterpret_cast<const void*>(kern), ebic::kTmaWarps * 32, smem);
      const unsigned grid = (unsigned)std::min<uint64_t>((n_cand + ebic::kTmaWarps - 1) / ebic::kTmaWarps,
                                                         std::max<uint64_t>(1, per_sm) * ctx->n_sms);
      // programmatic dependent launch (ebic_table.cuh pdl_trigger / pdl_wait):
      // back-to-back batches overlap one kernel's tail with the next one's start
      EBIC_CUDA(launch_pdl(kern, dim3(grid), dim3(ebic::kTmaWarps * 32), smem, s, pdl,
                           (const uint32_t*)ctx->d_table, (uint32_t)ctx->n_cols, (uint32_t)table_wp(ctx),
                           (uint32_t)ctx->n_rows, d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx, out,
                           err_out ? err_out : ctx->d_err, d_mask, (uint64_t)(ctx->ld / 32), plan.la));
      return EBIC_OK;
    };
    auto pickj = [&](auto negc, auto sc) -> int {
      constexpr bool N = decltype(negc)::value;
      constexpr int SS = decltype(sc)::value;
      switch (J) {
        case 1: return go(ebic::table_count_tma_kernel<1, SS, N, MASK>);
        case 2: return go(ebic::table_count_tma_kernel<2, SS, N, MASK>);
        case 3: return go(ebic::table_count_tma_kernel<3, SS, N, MASK>);
        case 4: return go(ebic::table_count_tma_kernel<4, SS, N, MASK>);
        case 5: return go(ebic::table_count_tma_kernel<5, SS, N, MASK>);
        case 6: return go(ebic::table_count_tma_kernel<6, SS, N, MASK>);
        case 7: return go(ebic::table_count_tma_kernel<7, SS, N, MASK>);
        default: return go(ebic::table_count_tma_kernel<8, SS, N, MASK>);
      }
    };
    auto pickj_lazy = [&](auto negc) -> int {
      constexpr bool N = decltype(negc)::value;
      switch (J) {
        case 1: return go(ebic::table_count_tma_kernel<1, 2, N, MASK, true>);
        case 2: return go(ebic::table_count_tma_kernel<2, 2, N, MASK, true>);
        case 3: return go(ebic::table_count_tma_kernel<3, 2, N, MASK, true>);
        case 4: return go(ebic::table_count_tma_kernel<4, 2, N, MASK, true>);
        case 5: return go(ebic::table_count_tma_kernel<5, 2, N, MASK, true>);
        case 6: return go(ebic::table_count_tma_kernel<6, 2, N, MASK, true>);
        case 7: return go(ebic::table_count_tma_kernel<7, 2, N, MASK, true>);
        default: return go(ebic::table_count_tma_kernel<8, 2, N, MASK, true>);
      }
    };
    int st;
    if (lazy) st = neg ? pickj_lazy(std::true_type{}) : pickj_lazy(std::false_type{});
    else if (S >= 4) st = neg ? pickj(std::true_type{}, std::integral_constant<int, 4>{})
                         : pickj(std::false_type{}, std::integral_constant<int, 4>{});
    else if (S == 3) st = neg ? pickj(std::true_type{}, std::integral_constant<int, 3>{})
                              : pickj(std::false_type{}, std::integral_constant<int, 3>{});
    else st = neg ? pickj(std::true_type{}, std::integral_constant<int, 2>{})
                  : pickj(std::false_type{}, std::integral_constant<int, 2>{});
    EBIC_TRY(st);
    ctx->launches++;
    EBIC_CUDA(cudaGetLastError());
    return EBIC_OK;
  }
  if (nv <= 256 && ctx->table_kernel != 2) {
    // short vectors: a warp per candidate, J = ceil(nv / 32) slices per lane
    const uint32_t J = (nv + 31) / 32;
    // a warp per candidate for the whole population (the block scheduler
    // balances the tail better than a grid-stride loop over fewer warps)
    const unsigned grid = (unsigned)std::min<uint64_t>((n_cand + 7) / 8, 1u << 30);
    auto go = [&](auto kern) {
      kern<<<grid, 256, 0, s>>>(ctx->d_table, (uint32_t)ctx->n_cols, (uint32_t)table_wp(ctx), (uint32_t)ctx->n_rows,
                                d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx, out, err_out ? err_out : ctx->d_err,
                                d_mask, ctx->ld / 32);
    };
    auto pickj = [&](auto negc) {
      constexpr bool N = decltype(negc)::value;
      switch (J) {
        case 1: go(ebic::table_count_warp_kernel<1, N, MASK>); break;
        case 2: go(ebic::table_count_warp_kernel<2, N, MASK>); break;
        case 3: go(ebic::table_count_warp_kernel<3, N, MASK>); break;
        case 4: go(ebic::table_count_warp_kernel<4, N, MASK>); break;
        case 5: go(ebic::table_count_warp_kernel<5, N, MASK>); break;
        case 6: go(ebic::table_count_warp_kernel<6, N, MASK>); break;
        case 7: go(ebic::table_count_warp_kernel<7, N, MASK>); break;
        default: go(ebic::table_count_warp_kernel<8, N, MASK>); break;
      }
    };
    if (neg) pickj(std::true_type{});
    else pickj(std::false_type{});
    ctx->launches++;
    EBIC_CUDA(cudaGetLastError());
    return EBIC_OK;
  }
  // long vectors: a CTA per candidate, T threads (one uint4 slice of every
  // pair vector each, J slices when the vector exceeds 1024 slices)
  const uint32_t T = std::min<uint32_t>(1024, (nv + 31) / 32 * 32);
  const uint32_t J = (nv + T - 1) / T;
  const uint64_t resident = (uint64_t)ctx->n_sms * std::max<uint32_t>(1, 2048 / T);
  const unsigned grid = (unsigned)std::min<uint64_t>(n_cand, resident);
  auto go = [&](auto kern) {
    kern<<<grid, T, 0, s>>>(ctx->d_table, (uint32_t)ctx->n_cols, (uint32_t)table_wp(ctx), (uint32_t)ctx->n_rows,
                            d_cols, d_offs, (uint32_t)n_cand, (uint32_t)n_idx, out, err_out ? err_out : ctx->d_err,
                            d_mask, ctx->ld / 32);
  };
  auto pick = [&](auto negc) {
    constexpr bool N = decltype(negc)::value;
    if (J <= 1) go(ebic::table_count_kernel<1, N, MASK>);
    else if (J <= 2) go(ebic::table_count_kernel<2, N, MASK>);
    else if (J <= 4) go(ebic::table_count_kernel<4, N, MASK>);
    else go(ebic::table_count_kernel<8, N, MASK>);
  };
  if (neg) pick(std::true_type{});
  else pick(std::false_type{});
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  return EBIC_OK;
}

struct SlabCfg {
  bool simd = false;  // packed 16-bit rank pairs (slab_pair_kernel); p = pair-words per lane
  bool v2 = false;    // (always with simd: the pair kernel publishes final counts itself)
  int p = 1;
  int rpl = 1, sub = 1;
  uint32_t rt = 32;
  uint32_t chunk = 0;
  size_t smem = 0;
  bool ok = false;
};

SlabCfg choose_slab(const ebic_ctx* ctx, uint64_t n_cand, bool mask) {
  // Shared memory: the slab (RT rows x all C columns of plane words) plus 20 B per
  // candidate of the chunk (16 B record + 4 B count).  Prefer more rows per lane
  // (fewer per-candidate overheads per row) while the slab stays <= 128 KB.
  SlabCfg c;
  const size_t budget = std::min<size_t>(ctx->smem_optin, 227 * 1024) - 1024;
  const size_t C = ctx->n_cols;
  const size_t kSlabCap = 128 * 1024;
  bool found = false;
  if (!mask && ctx->path != EBIC_PATH_PLANE_U32) {
    // packed pairs: the first layout (in measured order of speed on B200, see
    // profiles/r1b_layout_ab.txt) whose slab fits in 128 KB.  The other
    // layouts are reachable through ebic_ctx_set_pair_layout.
    // (P = 4 would need > 64 registers per thread at 1024 threads: spills)
    struct Opt { int p, sub; uint32_t rt; };
    const Opt opts[6] = {{2, 1, 128}, {1, 2, 32}, {1, 4, 16}, {2, 4, 32}, {2, 2, 64}, {1, 1, 64}};
    for (int k = 0; k < 6; ++k) {
      const Opt& o = opts[k];
      if (ctx->simd_force ? ctx->simd_force != o.p * 16 + o.sub : k >= 3) continue;
      if (C * o.rt * 4 <= kSlabCap) {
        c.simd = true;
        c.p = o.p;
        c.sub = o.sub;
        c.rt = o.rt;
        found = true;
        break;
      }
    }
  }
  if (found) {
    // slab_pair_kernel: per position a record (<= 16 B), a count and a slot; the
    // (kClasses - 1) swept classes are each padded to the sweep stride
    const size_t slab = C * c.rt * 4;
    const size_t stride = (size_t)ebic::kSlabWarps * c.sub;
    const size_t fixed = slab + (size_t)(ebic::kClasses - 1) * stride * ebic::kPairPosBytes + 16;
    const uint64_t cmax = std::min<uint64_t>((budget - fixed) / ebic::kPairPosBytes, 16384);
    const uint64_t n_chunks = (n_cand + cmax - 1) / cmax;
    c.chunk = (uint32_t)((n_cand + n_chunks - 1) / n_chunks);
    c.smem = fixed + (size_t)c.chunk * ebic::kPairPosBytes;
    c.v2 = true;
    c.ok = true;
    return c;
  }
  const int rpls[3] = {4, 2, 1};
  for (int rpl : rpls) {
    if (mask && rpl != 1) continue;
    if (C * 32 * rpl * 4 <= kSlabCap) {
      c.rpl = rpl;
      c.sub = 1;
      found = true;
      break;
    }
  }
  if (!found) {
    if (mask) return c;
    if (C * 16 * 4 <= 160 * 1024) { c.rpl = 1; c.sub = 2; }
    else if (C * 8 * 4 <= 160 * 1024) { c.rpl = 1; c.sub = 4; }
    else return c;
  }
  c.rt = (32 / c.sub) * c.rpl;
  const size_t slab = C * c.rt * 4;
  // records: chunk + class padding (ebic::kClasses x sweep stride), 16 B each; counts: chunk + 1
  const size_t fixed = slab + (size_t)ebic::kClasses * ebic::kSlabWarps * c.sub * 16 + 16;
  if (fixed + 20 * 64 > budget) return c;
  const uint64_t cmax = std::min<uint64_t>((budget - fixed) / 20, 16384);
  const uint64_t n_chunks = (n_cand + cmax - 1) / cmax;
  c.chunk = (uint32_t)((n_cand + n_chunks - 1) / n_chunks);
  c.smem = fixed + (size_t)c.chunk * 20;
  c.ok = true;
  return c;
}

ebic::SlabArgs make_slab_args(const ebic_ctx* ctx, const SlabCfg& cfg, const uint32_t* d_cols,
                              const uint32_t* d_offs, uint64_t n_cand, uint32_t* d_counts, uint32_t* d_mask) {
  ebic::SlabArgs a;
  a.plane = ctx->d_plane;
  a.ld = ctx->ld;
  a.n_rows = (uint32_t)ctx->n_rows;
  a.n_cols = (uint32_t)ctx->n_cols;
  a.cols = d_cols;
  a.offs = d_offs;
  a.n_cand = (uint32_t)n_cand;
  a.chunk = cfg.chunk;
  a.n_chunks = (uint32_t)((n_cand + cfg.chunk - 1) / cfg.chunk);
  a.n_slabs = (uint32_t)((ctx->n_rows + cfg.rt - 1) / cfg.rt);
  a.counts = d_counts;
  a.mask = d_mask;
  a.mask_wpc = ctx->ld / 32;
  a.err = ctx->d_err;
  // L2 prefetch of the next slab (EBIC_PREFETCH=0/1 forces it).  Measured on
  // B200 (profiles/archive/r1_ab_prefetch.txt): +4% when the plane is L2-resident
  // (20k x 1000, 80 MB), -5% when it streams from HBM (200k x 2000, 1.6 GB,
  // where the extra requests compete with other chunks' reuse of the same
  // slabs).  Default: on iff the plane fits comfortably in the 126 MB L2.
  const uint64_t plane_bytes = ctx->ld * ctx->n_cols * 4;
  a.prefetch = ctx->prefetch >= 0 ? ctx->prefetch : (plane_bytes <= (96ull << 20) ? 1 : 0);
  a.group = 0;
  return a;
}

template <int RPL, int SUB, bool NEG, bool MASK>
int launch_slab_t(ebic_ctx* ctx, const SlabCfg& cfg, const uint32_t* d_cols, const uint32_t* d_offs,
                  uint64_t n_cand, uint32_t* d_counts, uint32_t* d_mask, cudaStream_t s) {
  auto kern = ebic::slab_count_kernel<RPL, SUB, NEG, MASK>;
  // raise the dynamic shared-memory limit once per (kernel, device), to the opt-in maximum
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (!(attr_done.load(std::memory_order_relaxed) & bit)) {
    EBIC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ctx->smem_optin - 1024)));
    attr_done.fetch_or(bit);
  }
  ebic::SlabArgs a = make_slab_args(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask);
  const uint64_t units = (uint64_t)a.n_chunks * a.n_slabs;
  const unsigned grid = (unsigned)std::min<uint64_t>(units, (uint64_t)ctx->n_sms);
  kern<<<grid, ebic::kSlabThreads, cfg.smem, s>>>(a);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  return EBIC_OK;
}

struct PairOut {       // where slab_pair_kernel publishes its results
  uint32_t* out;       // final counts (device-accessible)
  int* err_out;        // device error flag forwarded here (nullptr: kept in ctx->d_err)
};

template <int P, int SUB, bool NEG>
int launch_simd_t(ebic_ctx* ctx, const SlabCfg& cfg, const uint32_t* d_cols, const uint32_t* d_offs,
                  uint64_t n_cand, uint32_t* d_counts, const PairOut* po, cudaStream_t s) {
  auto kern = ebic::slab_pair_kernel<P, SUB, NEG>;
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (!(attr_done.load(std::memory_order_relaxed) & bit)) {
    EBIC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ctx->smem_optin - 1024)));
    attr_done.fetch_or(bit);
  }
  ebic::SlabArgs a = make_slab_args(ctx, cfg, d_cols, d_offs, n_cand, d_counts, nullptr);
  unsigned grid = 0;
  {
    if (!po || !po->out) return fail(EBIC_ERR_INVALID_ARGUMENT, "internal: pair kernel without an output");
    // chunk groups of `group` CTAs (a CTA per SM; up to n_sms % n_chunks SMs idle):
    // the groups walk the plane in step, and every CTA packs its chunk once
    const uint32_t n_sms = (uint32_t)ctx->n_sms;
    a.group = std::max<uint32_t>(1, std::min<uint32_t>(n_sms / std::min<uint32_t>(a.n_chunks, n_sms), a.n_slabs));
    const uint32_t n_groups = std::min<uint32_t>(a.n_chunks, n_sms / a.group);
    grid = a.group * n_groups;
    EBIC_TRY(ensure_zero(ctx->d_acc, n_cand, s));
    EBIC_TRY(ensure_zero(ctx->d_done, (size_t)a.n_chunks + 1, s));
    a.counts = ctx->d_acc.p;
    a.out = po->out;
    a.done = ctx->d_done.p;
    a.err_out = po->err_out ? po->err_out : ctx->d_err;
  }
  kern<<<grid, ebic::kSlabThreads, cfg.smem, s>>>(a);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  return EBIC_OK;
}

template <bool NEG, bool MASK>
int launch_slab(ebic_ctx* ctx, const SlabCfg& cfg, const uint32_t* d_cols, const uint32_t* d_offs,
                uint64_t n_cand, uint32_t* d_counts, uint32_t* d_mask, const PairOut* po, cudaStream_t s) {
  if constexpr (!MASK) {
    if (cfg.simd) {
      if (cfg.p == 2) {
        if (cfg.sub == 1) return launch_simd_t<2, 1, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
        if (cfg.sub == 2) return launch_simd_t<2, 2, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
        return launch_simd_t<2, 4, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
      }
      if (cfg.sub == 1) return launch_simd_t<1, 1, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
      if (cfg.sub == 2) return launch_simd_t<1, 2, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
      return launch_simd_t<1, 4, NEG>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, po, s);
    }
  }
  if constexpr (MASK) {
    return launch_slab_t<1, 1, NEG, true>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
  } else {
    if (cfg.sub == 1) {
      if (cfg.rpl == 4) return launch_slab_t<4, 1, NEG, false>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
      if (cfg.rpl == 2) return launch_slab_t<2, 1, NEG, false>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
      return launch_slab_t<1, 1, NEG, false>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
    }
    if (cfg.sub == 2) return launch_slab_t<1, 2, NEG, false>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
    return launch_slab_t<1, 4, NEG, false>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, s);
  }
}

// Counting launch.  d_counts must be zero: the kernels ADD into it -- except
// slab_pair_kernel, which writes final counts to po->out (see count_into).
// `plan_in`: the index decision already taken for this launch (nullptr:
// decide here).
template <bool MASK>
int launch_count(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offs, uint64_t n_cand,
                 double approx, int neg, uint32_t* d_counts, uint32_t* d_mask, cudaStream_t s,
                 const PairOut* po = nullptr, uint64_t n_idx = 0xffffffffull, const IndexPlan* plan_in = nullptr) {
  if (n_cand == 0) return EBIC_OK;
  if (n_cand > 0xffffffffull / 2) return fail(EBIC_ERR_INVALID_ARGUMENT, "too many candidates");
  IndexPlan local;
  if (!plan_in) EBIC_TRY(use_index(ctx, approx, worst_pairs(n_cand, n_idx, neg), s, &local.mode, &local.la));
  const IndexPlan& plan = plan_in ? *plan_in : local;
  if (plan.mode != kIndexNone)
    return launch_table<MASK>(ctx, d_cols, d_offs, n_cand, n_idx, neg, po ? po->out : d_counts,
                              po ? po->err_out : nullptr, d_mask, s, plan);
  if (ctx->path != EBIC_PATH_VALUE && ctx->path != EBIC_PATH_TABLE && plane_fits(ctx)) {
    const SlabCfg cfg = choose_slab(ctx, n_cand, MASK);
    if (cfg.ok) {
      EBIC_TRY(ensure_plane(ctx, approx, s));
      if (neg) return launch_slab<true, MASK>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, po, s);
      return launch_slab<false, MASK>(ctx, cfg, d_cols, d_offs, n_cand, d_counts, d_mask, po, s);
    }
  }
  // (row masks for supporting_rows may always fall back to the value kernel:
  // the path knob is about the counting kernels)
  if (!MASK && (ctx->path == EBIC_PATH_PLANE || ctx->path == EBIC_PATH_PLANE_U32))
    return fail(EBIC_ERR_INVALID_ARGUMENT, "rank-plane path unavailable for a %llu-column matrix",
                (unsigned long long)ctx->n_cols);
  const ebic::TrendArgs ta = make_args(approx, neg);
  const bool a0 = (approx == 0.0);
  if (ctx->store == EBIC_STORE_F32) {
    if (a0) {
      if (neg) launch_count_t<float, ebic::kModeNative, true, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
      else     launch_count_t<float, ebic::kModeNative, false, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
    } else {
      if (neg) launch_count_t<float, ebic::kModeFilter, true, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
      else     launch_count_t<float, ebic::kModeFilter, false, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
    }
  } else {
    if (a0) {
      if (neg) launch_count_t<double, ebic::kModeNative, true, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
      else     launch_count_t<double, ebic::kModeNative, false, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
    } else {
      if (neg) launch_count_t<double, ebic::kModeF64, true, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
      else     launch_count_t<double, ebic::kModeF64, false, MASK>(ctx, d_cols, d_offs, n_cand, ta, d_counts, d_mask, s);
    }
  }
  EBIC_CUDA(cudaGetLastError());
  return EBIC_OK;
}

// Does a counting launch of n_cand candidates run slab_pair_kernel?  That
// kernel writes final counts to any device-accessible pointer -- including
// the device alias of page-locked host memory -- with no memset before and no
// copy after; the other kernels add into zeroed device memory.
bool pair_path(const ebic_ctx* ctx, uint64_t n_cand) {
  if (n_cand == 0 || ctx->path == EBIC_PATH_VALUE || !plane_fits(ctx)) return false;
  const SlabCfg cfg = choose_slab(ctx, n_cand, false);
  return cfg.ok && cfg.simd && cfg.v2;
}

// The decisions of one counting launch: which index (built or reserved now),
// and whether the kernel writes its results directly (an index kernel or
// slab_pair_kernel) -- then `out` may be the device alias of host memory.
struct LaunchPlan {
  IndexPlan index;
  bool direct = false;
};

int plan_launch(ebic_ctx* ctx, uint64_t n_cand, uint64_t n_idx, double approx, int neg, cudaStream_t s,
                LaunchPlan* lp) {
  EBIC_TRY(use_index(ctx, approx, worst_pairs(n_cand, n_idx, neg), s, &lp->index.mode, &lp->index.la));
  lp->direct = lp->index.mode != kIndexNone || pair_path(ctx, n_cand);
  return EBIC_OK;
}

// Evaluate and leave the FINAL counts in `out` and the device error flag in
// `err_out` (nullptr: ctx->d_err, read by ebic_ctx_sync).  `out` may be host
// memory (device alias) only when the plan is direct; `err_out` may be host
// memory (device alias) always.  `lp_in`: a plan already made for this launch.
int count_into(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offs, uint64_t n_cand, double approx,
               int neg, uint32_t* out, int* err_out, cudaStream_t s, uint64_t n_idx = 0xffffffffull,
               const LaunchPlan* lp_in = nullptr) {
  if (n_cand == 0) return EBIC_OK;
  LaunchPlan local;
  if (!lp_in) EBIC_TRY(plan_launch(ctx, n_cand, n_idx, approx, neg, s, &local));
  const LaunchPlan& lp = lp_in ? *lp_in : local;
  if (lp.direct) {
    const PairOut po{out, err_out};
    return launch_count<false>(ctx, d_cols, d_offs, n_cand, approx, neg, nullptr, nullptr, s, &po, n_idx, &lp.index);
  }
  EBIC_CUDA(cudaMemsetAsync(out, 0, n_cand * sizeof(uint32_t), s));
  EBIC_TRY(launch_count<false>(ctx, d_cols, d_offs, n_cand, approx, neg, out, nullptr, s, nullptr, n_idx, &lp.index));
  if (err_out && err_out != ctx->d_err) {
    EBIC_CUDA(cudaMemcpyAsync(err_out, ctx->d_err, sizeof(int), cudaMemcpyDefault, s));
    EBIC_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), s));
  }
  return EBIC_OK;
}

// Host-side validation of a CSR population (trend.hpp callers pass valid
// chromosomes; bicluster.cpp:8-15 is the reference's validity rule, but
// evaluate_population itself accepts duplicates and any length >= 1).
int validate_population(const ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                        uint64_t n_cand, bool check_cols = true) {
  if (n_cand && (!cols || !offsets)) return fail(EBIC_ERR_INVALID_ARGUMENT, "null population pointer");
  if (n_cand && offsets[0] != 0) return fail(EBIC_ERR_INVALID_ARGUMENT, "offsets[0] must be 0");
  if (!check_cols) {
    // branch-free (vectorisable) scan first; the detailed loop below only runs
    // to name the first bad candidate
    uint32_t bad = 0;
    for (uint64_t i = 0; i < n_cand; ++i) bad |= offsets[i + 1] <= offsets[i] ? 1u : 0u;
    if (!bad) return EBIC_OK;
  }
  for (uint64_t i = 0; i < n_cand; ++i) {
    if (offsets[i + 1] <= offsets[i])
      return fail(EBIC_ERR_INVALID_ARGUMENT, "candidate %llu is empty or offsets decrease",
                  (unsigned long long)i);
    if (check_cols)
      for (uint32_t k = offsets[i]; k < offsets[i + 1]; ++k)
        if (cols[k] >= ctx->n_cols)
          return fail(EBIC_ERR_INVALID_ARGUMENT, "candidate %llu: column %u out of range (cols=%llu)",
                      (unsigned long long)i, cols[k], (unsigned long long)ctx->n_cols);
  }
  return EBIC_OK;
}

int need_matrix(const ebic_ctx* ctx) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (!ctx->d_mat) return fail(EBIC_ERR_NO_MATRIX, "no matrix uploaded in this context");
  return EBIC_OK;
}

// Drop the resident matrix and what derives from it.  `keep_index_alloc`
// (a new upload follows): the pair-trend index allocation is kept for reuse --
// allocating gigabytes costs tens to hundreds of milliseconds per upload.
void drop_matrix(ebic_ctx* ctx, bool keep_index_alloc) {
  if (ctx->d_mat) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_mat);
  }
  if (ctx->d_plane) cudaFree(ctx->d_plane);
  ctx->d_plane = nullptr;
  ctx->plane_valid = false;
  if (ctx->d_table && !keep_index_alloc) {
    cudaFree(ctx->d_table);
    ctx->d_table = nullptr;
    ctx->table_cap = 0;
  }
  ctx->table_valid = ctx->table_failed = false;
  ctx->plane_timed = ctx->index_timed = false;
  ctx->full_requested = false;
  if (ctx->d_lpool) lazy_release(ctx, ctx->stream);
  if (ctx->d_lmap) cudaFree(ctx->d_lmap);
  ctx->d_lmap = nullptr;
  ctx->lazy_valid = false;
  ctx->lazy_built = ctx->lazy_epoch_seen = ctx->lazy_resets = 0;
  ctx->index_mode = kIndexNone;
  ctx->d_mat = nullptr;
  ctx->store = 0;
  ctx->n_rows = ctx->n_cols = ctx->ld = ctx->row_base = 0;
}

// Host -> device copy of a PAGEABLE buffer through page-locked staging: T
// worker threads each own a staging buffer, a stream and an event, and take
// chunks t, t + T, ...: copy the chunk into the buffer (once the buffer's
// previous DMA is done), then DMA it on their own stream -- the host copies
// and the DMAs of different chunks overlap.  Measured on B200's host (16
// cores), 1.6 GB: 362 ms for cudaMemcpy from pageable memory, 22 ms for a
// 16-thread copy into page-locked memory, 29 ms for a page-locked DMA
// (profiles/r2_host_copy.txt).  `s` waits for every chunk's DMA.
constexpr size_t kStageChunk = 8u << 20;
constexpr int kStageThreads = 8;
// The page-locked staging buffers are shared by every context of the process
// (cudaHostAllocPortable): a page-locked allocation costs ~0.45 ms per MB on
// the B200 host, so each context paying for its own made a context's first
// upload 56 ms slower.  Uploads through them are serialised by `mu`.
struct StagePool {
  std::mutex mu;
  std::vector<unsigned char*> bufs;
};
StagePool& stage_pool() {
  static StagePool* p = new StagePool;  // (never freed: lives as long as the process)
  return *p;
}

int staged_h2d(ebic_ctx* ctx, void* d_dst, const void* h_src, size_t bytes, cudaStream_t s) {
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::max<size_t>(1, std::min<size_t>({(size_t)std::min(hw, kStageThreads), bytes / (4 * kStageChunk)}));
  StagePool& sp = stage_pool();
  std::lock_guard<std::mutex> lock(sp.mu);
  const double ta = host_ms();
  while ((int)sp.bufs.size() < T) {
    unsigned char* b = nullptr;
    EBIC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b), kStageChunk, cudaHostAllocPortable));
    sp.bufs.push_back(b);
  }
  if ((int)ctx->stagers.size() < T) ctx->stagers.resize(T);
  for (int t = 0; t < T; ++t) {
    auto& st = ctx->stagers[t];
    if (!st.stream) EBIC_CUDA(cudaStreamCreateWithFlags(&st.stream, cudaStreamNonBlocking));
    if (!st.done) EBIC_CUDA(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
    // (the destination may still be in use by work queued on s)
    EBIC_CUDA(cudaEventRecord(st.done, s));
    EBIC_CUDA(cudaStreamWaitEvent(st.stream, st.done, 0));
    st.armed = false;
  }
  if (std::getenv("EBIC_UPLOAD_TRACE")) std::fprintf(stderr, "upload: staging setup %.1f ms (%d threads)\n", host_ms() - ta, T);
  const size_t n_chunks = (bytes + kStageChunk - 1) / kStageChunk;
  std::vector<cudaError_t> errs(T, cudaSuccess);
  auto work = [&](int t) {
    auto& st = ctx->stagers[t];
    unsigned char* buf = sp.bufs[t];
    cudaSetDevice(ctx->device);
    for (size_t k = t; k < n_chunks && errs[t] == cudaSuccess; k += T) {
      const size_t off = k * kStageChunk, len = std::min(kStageChunk, bytes - off);
      if (st.armed && (errs[t] = cudaEventSynchronize(st.done)) != cudaSuccess) break;
      std::memcpy(buf, static_cast<const unsigned char*>(h_src) + off, len);
      errs[t] = cudaMemcpyAsync(static_cast<unsigned char*>(d_dst) + off, buf, len, cudaMemcpyHostToDevice, st.stream);
      if (errs[t] == cudaSuccess) errs[t] = cudaEventRecord(st.done, st.stream);
      st.armed = true;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int t = 0; t < T; ++t) {
    if (errs[t] != cudaSuccess) return fail(EBIC_ERR_CUDA, "staged upload: %s", cudaGetErrorString(errs[t]));
    EBIC_CUDA(cudaEventRecord(ctx->stagers[t].done, ctx->stagers[t].stream));
    EBIC_CUDA(cudaStreamWaitEvent(s, ctx->stagers[t].done, 0));
  }
  // the shared buffers may be refilled by the next upload: wait for the DMAs
  for (int t = 0; t < T; ++t) EBIC_CUDA(cudaEventSynchronize(ctx->stagers[t].done));
  return EBIC_OK;
}

// Pageable host memory (not page-locked / registered / managed)?
bool pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// `src` is host memory, or (src_on_device) a buffer on this context's GPU that
// is read in place (checked and transposed from it; the caller keeps it).
template <typename TI>
int upload_impl(ebic_ctx* ctx, const TI* host, uint64_t n_rows, uint64_t n_cols, uint64_t row_base,
                int store, int* store_out, bool src_on_device = false) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (!host && n_rows * n_cols) return fail(EBIC_ERR_INVALID_ARGUMENT, "null matrix pointer");
  if (n_rows == 0 || n_cols == 0) return fail(EBIC_ERR_INVALID_ARGUMENT, "matrix must be non-empty");
  if (n_rows >= (1ull << 31) || n_cols >= (1ull << 31) || row_base + n_rows >= (1ull << 32))
    return fail(EBIC_ERR_INVALID_ARGUMENT, "matrix too large for 32-bit row/column indices");
  if (store < EBIC_STORE_AUTO || store > EBIC_STORE_F64)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "bad store mode %d", store);
  EBIC_TRY(set_device(ctx));
  const bool trace = std::getenv("EBIC_UPLOAD_TRACE") != nullptr;
  const double tu0 = host_ms();
  auto mark = [&](const char* what) {
    if (trace) std::fprintf(stderr, "upload: %-22s at %.1f ms\n", what, host_ms() - tu0);
  };
  drop_matrix(ctx, /*keep_index_alloc=*/true);
  mark("previous matrix freed");
  cudaStream_t s = ctx->stream;
  const uint64_t n = n_rows * n_cols;

  if (src_on_device) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, host) != cudaSuccess || a.type != cudaMemoryTypeDevice ||
        a.device != ctx->device) {
      cudaGetLastError();
      return fail(EBIC_ERR_INVALID_ARGUMENT, "matrix pointer is not device memory on device %d", ctx->device);
    }
  }
  TI* d_in = nullptr;
  cudaError_t ce = cudaSuccess;
  if (src_on_device) {
    d_in = const_cast<TI*>(host);
  } else {
    const double t0 = host_ms();
    EBIC_CUDA(cudaMalloc(&d_in, n * sizeof(TI)));
    const double t1 = host_ms();
    if (n * sizeof(TI) >= 4 * kStageChunk && pageable(host)) {
      if (staged_h2d(ctx, d_in, host, n * sizeof(TI), s) != EBIC_OK) {
        cudaFree(d_in);
        return EBIC_ERR_CUDA;
      }
    } else {
      ce = cudaMemcpyAsync(d_in, host, n * sizeof(TI), cudaMemcpyHostToDevice, s);
    }
    if (std::getenv("EBIC_UPLOAD_TRACE")) {
      cudaStreamSynchronize(s);
      std::fprintf(stderr, "upload: malloc %.1f ms, h2d %.1f ms\n", t1 - t0, host_ms() - t1);
    }
  }
  auto release_in = [&]() {
    if (!src_on_device) cudaFree(d_in);
  };
  if (ce == cudaSuccess) ce = cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s);
  if (ce != cudaSuccess) {
    release_in();
    return fail(EBIC_ERR_CUDA, "matrix upload: %s", cudaGetErrorString(ce));
  }
  {
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    ebic::check_values_kernel<TI><<<blocks, 256, 0, s>>>(d_in, n, ctx->d_flags);
    ctx->launches++;
  }
  int flags = 0;
  ce = cudaMemcpyAsync(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) {
    release_in();
    return fail(EBIC_ERR_CUDA, "matrix check: %s", cudaGetErrorString(ce));
  }
  if (flags & 1) {
    release_in();
    return fail(EBIC_ERR_INVALID_ARGUMENT, "ExpressionMatrix: non-finite value");
  }
  mark("checked");
  const bool exact = !(flags & 2);
  int chosen = store;
  if (chosen == EBIC_STORE_AUTO) chosen = exact ? EBIC_STORE_F32 : EBIC_STORE_F64;
  if (chosen == EBIC_STORE_F32 && !exact) {
    release_in();
    return fail(EBIC_ERR_NOT_EXACT, "matrix has values that are not float32-representable");
  }
  const uint64_t ld = (n_rows + ebic::kRowAlign - 1) / ebic::kRowAlign * ebic::kRowAlign;
  const size_t esz = chosen == EBIC_STORE_F32 ? sizeof(float) : sizeof(double);
  void* d_mat = nullptr;
  ce = cudaMalloc(&d_mat, ld * n_cols * esz);
  if (ce != cudaSuccess) {
    release_in();
    return fail(EBIC_ERR_CUDA, "matrix store alloc (%llu bytes): %s",
                (unsigned long long)(ld * n_cols * esz), cudaGetErrorString(ce));
  }
  dim3 block(32, 8), grid((unsigned)((n_cols + 31) / 32), (unsigned)(ld / 32));
  if (chosen == EBIC_STORE_F32)
    ebic::transpose_kernel<TI, float><<<grid, block, 0, s>>>(d_in, n_rows, n_cols, (float*)d_mat, ld, ld);
  else
    ebic::transpose_kernel<TI, double><<<grid, block, 0, s>>>(d_in, n_rows, n_cols, (double*)d_mat, ld, ld);
  ctx->launches++;
  ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  release_in();
  if (ce != cudaSuccess) {
    cudaFree(d_mat);
    return fail(EBIC_ERR_CUDA, "matrix transpose: %s", cudaGetErrorString(ce));
  }
  mark("transposed");
  ctx->d_mat = d_mat;
  ctx->store = chosen;
  ctx->n_rows = n_rows;
  ctx->n_cols = n_cols;
  ctx->ld = ld;
  ctx->row_base = row_base;
  {
    // pair-trend index budget (index_budget): measured against the memory free now
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      fr = 0;
    }
    ctx->table_budget = index_budget(ctx, fr + ctx->table_cap);
    // a kept index allocation: reused if this matrix's index fits it and
    // is allowed, otherwise (or if it is more than twice the need) released
    if (ctx->d_table && (!table_allowed(ctx) || ctx->table_cap < table_bytes(ctx) ||
                         ctx->table_cap > 2 * table_bytes(ctx))) {
      cudaFree(ctx->d_table);
      ctx->d_table = nullptr;
      ctx->table_cap = 0;
    }
  }
  if (lazy_allowed(ctx)) {  // the lazy index's pair map now, not on the first batch
    const cudaError_t me = cudaMalloc(&ctx->d_lmap, lazy_map_bytes(ctx));
    if (me != cudaSuccess) {
      cudaGetLastError();
      ctx->d_lmap = nullptr;  // retried (and reported) on first use
    }
  }
  mark("done");
  if (store_out) *store_out = chosen;
  return EBIC_OK;
}

int bad_column_error(const ebic_ctx* ctx) {
  return fail(EBIC_ERR_INVALID_ARGUMENT, "a candidate has a column index out of range (cols=%llu); its count is 0",
              (unsigned long long)ctx->n_cols);
}

// Retire a slot: wait for its copies, hand the counts to the caller's buffer.
// `early` = retired on behalf of another submission (ring reuse or growth): a
// device-detected error is then remembered for that ticket's ebic_eval_wait
// instead of being returned here.
int wait_slot(ebic_ctx* ctx, Slot& sl, bool early = false) {
  if (!sl.ticket) return EBIC_OK;
  EBIC_CUDA(cudaEventSynchronize(sl.done));
  if (sl.user_counts) std::memcpy(sl.user_counts, sl.h_counts.p, sl.n_cand * sizeof(uint32_t));
  const int err = sl.h_err.p ? sl.h_err.p[0] : 0;
  const uint64_t t = sl.ticket;
  sl.ticket = 0;
  sl.user_counts = nullptr;
  if (err) {
    if (early) {
      ctx->failed_tickets.push_back(t);
      return EBIC_OK;
    }
    return bad_column_error(ctx);
  }
  return EBIC_OK;
}

}  // namespace

extern "C" {

int ebic_abi_version(void) { return EBIC_ABI_VERSION; }

const char* ebic_last_error(void) { return g_last_error.c_str(); }

int ebic_device_count(int* n_out) {
  if (!n_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null n_out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *n_out = n;
  return EBIC_OK;
}

int ebic_ctx_create(int device, ebic_ctx** ctx_out) {
  if (!ctx_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null ctx_out");
  *ctx_out = nullptr;
  int n = 0;
  ebic_device_count(&n);
  if (device < 0 || device >= n)
    return fail(EBIC_ERR_NO_DEVICE, "CUDA device %d not available (%d visible)", device, n);
  ebic_ctx* ctx = new ebic_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, 3 * sizeof(int));
  if (e == cudaSuccess) {
    ctx->d_flags = ctx->d_err + 1;
    ctx->d_out1 = ctx->d_err + 2;
    e = cudaMemset(ctx->d_err, 0, 3 * sizeof(int));
  }
  for (int i = 0; i < EBIC_MARSHAL_SLOTS && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&ctx->slots[i].done, cudaEventDisableTiming);
  // the lazy index's bookkeeping (counter, host-mapped mirror) up front: a
  // page-locked allocation costs milliseconds, not a cost for the first batch
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_lcount, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_lmirror.p, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) {
    ctx->h_lmirror.n = 2;
    ctx->h_lmirror.p[0] = ctx->h_lmirror.p[1] = 0;
    ctx->h_lmirror_dev = static_cast<uint32_t*>(dev_alias(ctx->h_lmirror.p));
  }
  if (e != cudaSuccess) {
    ebic_ctx_destroy(ctx);
    return fail(EBIC_ERR_CUDA, "context creation on device %d: %s", device, cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && v > 0) ctx->n_sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) == cudaSuccess && v > 0)
      ctx->smem_optin = (size_t)v;
    const char* e = std::getenv("EBIC_PATH");
    if (e) ctx->path = std::atoi(e);
    const char* pb = std::getenv("EBIC_PLANE_BUILDER");
    if (pb) ctx->plane_builder = std::atoi(pb);
    const char* pf = std::getenv("EBIC_PREFETCH");
    if (pf) ctx->prefetch = std::atoi(pf) ? 1 : 0;
    const char* tb = std::getenv("EBIC_TABLE_BUDGET_MB");
    if (tb) ctx->table_budget_user = (uint64_t)std::strtoull(tb, nullptr, 10) << 20;
    const char* zr = std::getenv("EBIC_ZC_READ_MAX");
    if (zr) ctx->zc_read_max = std::strtoull(zr, nullptr, 10);
    const char* hp = std::getenv("EBIC_HOST_PIECES");
    if (hp) ctx->pipeline_pieces = std::max(1, std::min(4, std::atoi(hp)));
    const char* tba = std::getenv("EBIC_TABLE_BUILD_A");
    if (tba) ctx->table_build_a = std::atoi(tba) == 1 ? 1 : 2;
    const char* ts = std::getenv("EBIC_TMA_SLOTS");
    if (ts) ctx->tma_slots = std::max(2, std::min(4, std::atoi(ts)));
    const char* tk = std::getenv("EBIC_TABLE_KERNEL");
    if (tk) ctx->table_kernel = std::atoi(tk);
    ctx->lazy_trace = std::getenv("EBIC_LAZY_TRACE") != nullptr;
    const char* lb = std::getenv("EBIC_LAZY_BUILD");
    if (lb) ctx->lazy_build = std::max(0, std::min(2, std::atoi(lb)));
    const char* pd = std::getenv("EBIC_PDL");
    if (pd) ctx->pdl = std::atoi(pd) != 0;
    const char* xt = std::getenv("EBIC_XCHG_TIMEOUT_MS");
    if (xt && std::atoll(xt) > 0) ctx->xchg_timeout_ns = (uint64_t)std::atoll(xt) * 1000000ull;
    const char* sc = std::getenv("EBIC_PAIR_LAYOUT");
    int fp = 0, fs = 0;
    if (sc && std::sscanf(sc, "%d,%d", &fp, &fs) == 2) ctx->simd_force = fp * 16 + fs;
  }
  *ctx_out = ctx;
  return EBIC_OK;
}

int ebic_ctx_destroy(ebic_ctx* ctx) {
  if (!ctx) return EBIC_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto& sl : ctx->slots) {
    sl.h_cols.release();
    sl.h_offs.release();
    sl.h_counts.release();
    sl.h_err.release();
    sl.d_cols.release();
    sl.d_offs.release();
    sl.d_counts.release();
    if (sl.done) cudaEventDestroy(sl.done);
  }
  ebic_matrix_free(ctx);
  ctx->d_mask.release();
  ctx->d_rows.release();
  ctx->d_tmp_cols.release();
  ctx->d_tmp_offs.release();
  ctx->d_tmp_counts.release();
  ctx->d_row_offsets.release();
  ctx->h_tmp_counts.release();
  ctx->d_inter.release();
  ctx->h_inter.release();
  ebic_xchg_destroy(ctx);
  ctx->d_acc.release();
  ctx->d_done.release();
  for (auto& sc : ctx->lscratch) {
    sc.defer.release();
    sc.pslot.release();
    if (sc.done) cudaEventDestroy(sc.done);
    sc.done = nullptr;
  }
  ctx->h_err1.release();
  for (cudaEvent_t& e : ctx->piece_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (int i = 0; i < ebic_ctx::kXchgDepth; ++i) {
    if (ctx->xchg_cdone[i]) cudaEventDestroy(ctx->xchg_cdone[i]);
    if (ctx->xchg_xdone[i]) cudaEventDestroy(ctx->xchg_xdone[i]);
  }
  if (ctx->xchg_stream) cudaStreamDestroy(ctx->xchg_stream);
  for (cudaEvent_t& e : ctx->ev_build)
    if (e) cudaEventDestroy(e);
  for (auto& st : ctx->stagers) {
    if (st.stream) cudaStreamDestroy(st.stream);
    if (st.done) cudaEventDestroy(st.done);
  }
  ctx->stagers.clear();
  if (ctx->d_lcount) cudaFree(ctx->d_lcount);
  if (ctx->d_lstart) cudaFree(ctx->d_lstart);
  ctx->h_lmirror.release();
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return EBIC_OK;
}

int ebic_ctx_set_stream(ebic_ctx* ctx, void* cuda_stream) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  return EBIC_OK;
}

int ebic_ctx_sync(ebic_ctx* ctx) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  EBIC_TRY(set_device(ctx));
  EBIC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->xchg_stream) EBIC_CUDA(cudaStreamSynchronize(ctx->xchg_stream));
  EBIC_CUDA(cudaDeviceSynchronize());
  int err = 0;
  EBIC_CUDA(cudaMemcpy(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) {
    EBIC_CUDA(cudaMemset(ctx->d_err, 0, sizeof(int)));
    if (err == 4) return fail(EBIC_ERR_CUDA, "peer exchange timed out: a rank did not arrive (counts set to 0xFFFFFFFF)");
    if (err == 5)
      return fail(EBIC_ERR_CUDA, "peer exchange poisoned: a rank's count failed (counts set to 0xFFFFFFFF)");
    return fail(EBIC_ERR_INVALID_ARGUMENT,
                "device detected an empty candidate or an out-of-range column index");
  }
  return EBIC_OK;
}

int ebic_matrix_upload_f64(ebic_ctx* ctx, const double* row_major, uint64_t n_rows, uint64_t n_cols,
                           uint64_t row_base, int store, int* store_out) {
  NvtxRange nvtx_("ebic:matrix_upload");
  return upload_impl<double>(ctx, row_major, n_rows, n_cols, row_base, store, store_out);
}

int ebic_matrix_upload_f32(ebic_ctx* ctx, const float* row_major, uint64_t n_rows, uint64_t n_cols,
                           uint64_t row_base) {
  NvtxRange nvtx_("ebic:matrix_upload");
  return upload_impl<float>(ctx, row_major, n_rows, n_cols, row_base, EBIC_STORE_F32, nullptr);
}

int ebic_matrix_upload_device_f64(ebic_ctx* ctx, const double* d_row_major, uint64_t n_rows, uint64_t n_cols,
                                  uint64_t row_base, int store, int* store_out) {
  NvtxRange nvtx_("ebic:matrix_upload_device");
  return upload_impl<double>(ctx, d_row_major, n_rows, n_cols, row_base, store, store_out, true);
}

int ebic_matrix_upload_device_f32(ebic_ctx* ctx, const float* d_row_major, uint64_t n_rows, uint64_t n_cols,
                                  uint64_t row_base) {
  NvtxRange nvtx_("ebic:matrix_upload_device");
  return upload_impl<float>(ctx, d_row_major, n_rows, n_cols, row_base, EBIC_STORE_F32, nullptr, true);
}

int ebic_matrix_info(ebic_ctx* ctx, uint64_t* n_rows, uint64_t* n_cols, uint64_t* ld, int* store,
                     uint64_t* row_base) {
  EBIC_TRY(need_matrix(ctx));
  if (n_rows) *n_rows = ctx->n_rows;
  if (n_cols) *n_cols = ctx->n_cols;
  if (ld) *ld = ctx->ld;
  if (store) *store = ctx->store;
  if (row_base) *row_base = ctx->row_base;
  return EBIC_OK;
}

int ebic_matrix_free(ebic_ctx* ctx) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  drop_matrix(ctx, false);
  return EBIC_OK;
}

int ebic_eval_counts_device(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets,
                            uint64_t n_cand, double approx, int negative_trends, uint32_t* d_counts,
                            void* stream) {
  NvtxRange nvtx_("ebic:eval_counts_device");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  if (n_cand && (!d_cols || !d_offsets || !d_counts))
    return fail(EBIC_ERR_INVALID_ARGUMENT, "null device pointer");
  EBIC_TRY(set_device(ctx));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  if (n_cand == 0) return EBIC_OK;
  return count_into(ctx, d_cols, d_offsets, n_cand, approx, negative_trends, d_counts, nullptr, s);
}

int ebic_eval_submit(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets, uint64_t n_cand,
                     double approx, int negative_trends, uint32_t* counts_out, uint64_t* ticket_out) {
  NvtxRange nvtx_("ebic:eval_submit");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  if (n_cand && !counts_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null counts_out");
  // offsets on the host (they bound every device read); column indices are
  // validated on device while packing and reported by ebic_eval_wait
  EBIC_TRY(validate_population(ctx, cols, offsets, n_cand, /*check_cols=*/false));
  EBIC_TRY(set_device(ctx));
  const uint64_t ticket = ctx->next_ticket++;
  Slot& sl = ctx->slots[ticket % EBIC_MARSHAL_SLOTS];
  EBIC_TRY(wait_slot(ctx, sl, /*early=*/true));  // ring full: retire the oldest submission first
  const uint64_t n_idx = n_cand ? offsets[n_cand] : 0;
  // Grow every slot of the ring together (cudaMallocHost costs milliseconds):
  // after the first submission of a given size, no later submission allocates.
  // A slot still in flight is retired first -- its pending copies target the
  // buffers that growing would free.
  for (Slot& any : ctx->slots) {
    const bool grow = any.h_cols.n < n_idx || any.h_offs.n < n_cand + 1 || any.h_counts.n < n_cand ||
                      !any.h_cols.p || !any.h_offs.p || !any.h_counts.p || !any.h_err.p ||
                      any.d_cols.n < n_idx || any.d_offs.n < n_cand + 1 || any.d_counts.n < n_cand;
    if (!grow) continue;
    if (&any != &sl) EBIC_TRY(wait_slot(ctx, any, /*early=*/true));
    EBIC_TRY(ensure(any.h_cols, n_idx));
    EBIC_TRY(ensure(any.h_offs, n_cand + 1));
    EBIC_TRY(ensure(any.h_counts, n_cand));
    EBIC_TRY(ensure(any.d_cols, n_idx));
    EBIC_TRY(ensure(any.d_offs, n_cand + 1));
    EBIC_TRY(ensure(any.d_counts, n_cand));
    EBIC_TRY(ensure(any.h_err, 1));
  }
  if (n_cand) {
    std::memcpy(sl.h_cols.p, cols, n_idx * sizeof(uint32_t));
    std::memcpy(sl.h_offs.p, offsets, (n_cand + 1) * sizeof(uint32_t));
  }
  cudaStream_t s = ctx->stream;
  if (n_cand) {
    uint32_t* h_counts_dev = static_cast<uint32_t*>(dev_alias(sl.h_counts.p));
    int* h_err_dev = static_cast<int*>(dev_alias(sl.h_err.p));
    // (reading the candidates over the bus from the page-locked slot inside
    // the kernel measured slower than one DMA: the first loads of every warp
    // wait a bus round trip)
    EBIC_CUDA(cudaMemcpyAsync(sl.d_cols.p, sl.h_cols.p, n_idx * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    EBIC_CUDA(cudaMemcpyAsync(sl.d_offs.p, sl.h_offs.p, (n_cand + 1) * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, s));
    // the index / pair kernels write the counts and the error flag straight
    // into the slot's page-locked buffers; otherwise device counts + a D2H copy
    const bool mapped = h_counts_dev && h_err_dev;
    LaunchPlan lp;
    EBIC_TRY(plan_launch(ctx, n_cand, n_idx, approx, negative_trends, s, &lp));
    if (mapped && lp.direct) {
      sl.h_err.p[0] = 0;  // the index kernel only writes on error (the slot is not in flight)
      EBIC_TRY(count_into(ctx, sl.d_cols.p, sl.d_offs.p, n_cand, approx, negative_trends, h_counts_dev,
                          h_err_dev, s, n_idx, &lp));
    } else {
      EBIC_TRY(count_into(ctx, sl.d_cols.p, sl.d_offs.p, n_cand, approx, negative_trends, sl.d_counts.p,
                          nullptr, s, n_idx, &lp));
      EBIC_CUDA(cudaMemcpyAsync(sl.h_counts.p, sl.d_counts.p, n_cand * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, s));
      EBIC_CUDA(cudaMemcpyAsync(sl.h_err.p, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
      EBIC_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), s));
    }
  } else {
    sl.h_err.p[0] = 0;
  }
  EBIC_CUDA(cudaEventRecord(sl.done, s));
  sl.ticket = ticket;
  sl.user_counts = counts_out;
  sl.n_cand = n_cand;
  if (ticket_out) *ticket_out = ticket;
  return EBIC_OK;
}

int ebic_eval_wait(ebic_ctx* ctx, uint64_t ticket) {
  NvtxRange nvtx_("ebic:eval_wait");
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  Slot& sl = ctx->slots[ticket % EBIC_MARSHAL_SLOTS];
  if (sl.ticket != ticket) {
    if (ticket == 0 || ticket >= ctx->next_ticket)
      return fail(EBIC_ERR_INVALID_ARGUMENT, "unknown ticket %llu", (unsigned long long)ticket);
    // already retired (its slot was reused): report its device-side error, once
    auto it = std::find(ctx->failed_tickets.begin(), ctx->failed_tickets.end(), ticket);
    if (it != ctx->failed_tickets.end()) {
      ctx->failed_tickets.erase(it);
      return bad_column_error(ctx);
    }
    return EBIC_OK;
  }
  EBIC_TRY(set_device(ctx));
  return wait_slot(ctx, sl);
}


int ebic_eval_counts(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets, uint64_t n_cand,
                     double approx, int negative_trends, uint32_t* counts_out) {
  NvtxRange nvtx_("ebic:eval_counts");
  // Zero-copy when the caller's arrays are already page-locked (cudaHostAlloc /
  // cudaHostRegister / torch pin_memory): the inputs are DMA'd straight from
  // them (ONE copy when the offsets are immediately followed by the columns in
  // memory) and the pair kernel writes the counts straight into counts_out
  // over the bus.  Otherwise go through the marshaller's pinned staging slots.
  uint32_t* out_dev = nullptr;
  if (n_cand && ctx && ctx->d_mat && cols && offsets && counts_out) {
    if (dev_alias(offsets) && dev_alias(cols)) out_dev = static_cast<uint32_t*>(dev_alias(counts_out));
  }
  if (out_dev) {
    EBIC_TRY(check_approx(approx));
    if (offsets[0] != 0) return fail(EBIC_ERR_INVALID_ARGUMENT, "offsets[0] must be 0");
    EBIC_TRY(set_device(ctx));
    cudaStream_t s = ctx->stream;
    const uint64_t n_idx = offsets[n_cand];
    if (!ctx->h_err1.p) {
      EBIC_TRY(ensure(ctx->h_err1, 1));
      ctx->h_err1_dev = static_cast<int*>(dev_alias(ctx->h_err1.p));
    }
    int* err_dev = ctx->h_err1_dev;
    if (!err_dev) return fail(EBIC_ERR_CUDA, "page-locked error flag is not device-mapped");
    ctx->h_err1.p[0] = 0;
    const bool one_copy = offsets + (n_cand + 1) == cols;
    const uint64_t n_idx_h = offsets[n_cand];
    LaunchPlan lp;
    EBIC_TRY(plan_launch(ctx, n_cand, n_idx_h, approx, negative_trends, s, &lp));
    const bool table = lp.index.mode != kIndexNone;  // an index kernel: offsets checked on device
    const int pieces = (lp.index.mode == kIndexFull && n_cand >= 2048) ? ctx->pipeline_pieces : 1;
    if (pieces > 1) {
      // pair-trend index, pipelined: the population goes over in `pieces`
      // DMAs on the copy stream (offsets + the first columns first) and the
      // index kernel of piece k starts as soon as piece k has landed, while
      // the next pieces are still in flight; counts land in counts_out
      if (!ctx->copy_stream) EBIC_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (cudaEvent_t& e : ctx->piece_ev)
        if (!e) EBIC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      // device scratch laid out like an [offsets | cols] block
      EBIC_TRY(ensure(ctx->d_tmp_cols, n_cand + 1 + n_idx));
      uint32_t* d_offs = ctx->d_tmp_cols.p;
      uint32_t* d_cols = ctx->d_tmp_cols.p + n_cand + 1;
      // the scratch buffers may still be read by this context's previous work
      EBIC_CUDA(cudaEventRecord(ctx->piece_ev[4], s));
      EBIC_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->piece_ev[4], 0));
      uint64_t cb[5], ib[5];  // candidate / column bounds of the pieces (clamped: offsets unchecked yet)
      for (int k = 0; k <= pieces; ++k) {
        cb[k] = n_cand * (uint64_t)k / pieces;
        ib[k] = std::min<uint64_t>(offsets[cb[k]], n_idx);
        if (k && ib[k] < ib[k - 1]) ib[k] = ib[k - 1];
      }
      ib[pieces] = n_idx;
      for (int k = 0; k < pieces; ++k) {
        if (k == 0 && one_copy) {  // offsets + the first piece's columns: one contiguous block
          EBIC_CUDA(cudaMemcpyAsync(d_offs, offsets, (n_cand + 1 + ib[1]) * sizeof(uint32_t),
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
        } else {
          if (k == 0)
            EBIC_CUDA(cudaMemcpyAsync(d_offs, offsets, (n_cand + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                      ctx->copy_stream));
          if (ib[k + 1] > ib[k])
            EBIC_CUDA(cudaMemcpyAsync(d_cols + ib[k], cols + ib[k], (ib[k + 1] - ib[k]) * sizeof(uint32_t),
                                      cudaMemcpyHostToDevice, ctx->copy_stream));
        }
        EBIC_CUDA(cudaEventRecord(ctx->piece_ev[k], ctx->copy_stream));
      }
      if (validate_population(ctx, cols, offsets, n_cand, /*check_cols=*/false) != EBIC_OK) {
        const std::string msg = g_last_error;
        cudaStreamSynchronize(ctx->copy_stream);
        return fail(EBIC_ERR_INVALID_ARGUMENT, "%s", msg.c_str());
      }
      for (int k = 0; k < pieces; ++k) {
        EBIC_CUDA(cudaStreamWaitEvent(s, ctx->piece_ev[k], 0));
        EBIC_TRY(launch_table<false>(ctx, d_cols, d_offs + cb[k], cb[k + 1] - cb[k], n_idx, negative_trends,
                                     out_dev + cb[k], err_dev, nullptr, s, lp.index));
      }
      EBIC_CUDA(cudaStreamSynchronize(s));
      const int e = *(volatile int*)ctx->h_err1.p;
      if (e == 2) return fail(EBIC_ERR_INVALID_ARGUMENT, "a candidate is empty or its offsets decrease");
      if (e) return bad_column_error(ctx);
      return EBIC_OK;
    }
    // the input DMA is issued first; the offsets are checked on the host while
    // it is in flight (the copy reads exactly [0, offsets[n_cand]) of cols, the
    // size the caller declares), and the kernel is launched only if they pass
    const uint32_t *d_cols, *d_offs;
    const uint64_t in_bytes = (n_cand + 1 + n_idx) * sizeof(uint32_t);
    if (table && lp.direct && in_bytes <= ctx->zc_read_max) {
      // a small batch: the index kernel reads the page-locked arrays over the
      // bus itself (two dependent round trips per warp) instead of waiting for
      // a DMA -- no copy at all (EBIC_ZC_READ_MAX bytes; see DESIGN 4.2)
      d_offs = static_cast<const uint32_t*>(dev_alias(offsets));
      d_cols = static_cast<const uint32_t*>(dev_alias(cols));
    } else if (one_copy) {
      EBIC_TRY(ensure(ctx->d_tmp_cols, n_cand + 1 + n_idx));
      EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_cols.p, offsets, (n_cand + 1 + n_idx) * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, s));
      d_offs = ctx->d_tmp_cols.p;
      d_cols = ctx->d_tmp_cols.p + n_cand + 1;
    } else {
      EBIC_TRY(ensure(ctx->d_tmp_cols, n_idx));
      EBIC_TRY(ensure(ctx->d_tmp_offs, n_cand + 1));
      EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_cols.p, cols, n_idx * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_offs.p, offsets, (n_cand + 1) * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, s));
      d_offs = ctx->d_tmp_offs.p;
      d_cols = ctx->d_tmp_cols.p;
    }
    // the index kernel checks every candidate's offsets on device (increasing,
    // within offsets[n_cand]); the other kernels need them checked here
    if (!table && validate_population(ctx, cols, offsets, n_cand, /*check_cols=*/false) != EBIC_OK) {
      const std::string msg = g_last_error;
      cudaStreamSynchronize(s);  // the scratch buffers may be reused by the next call
      return fail(EBIC_ERR_INVALID_ARGUMENT, "%s", msg.c_str());
    }
    if (lp.direct) {
      EBIC_TRY(count_into(ctx, d_cols, d_offs, n_cand, approx, negative_trends, out_dev, err_dev, s, n_idx, &lp));
    } else {
      EBIC_TRY(ensure(ctx->d_tmp_counts, n_cand));
      EBIC_TRY(count_into(ctx, d_cols, d_offs, n_cand, approx, negative_trends, ctx->d_tmp_counts.p, err_dev, s,
                          n_idx, &lp));
      EBIC_CUDA(cudaMemcpyAsync(counts_out, ctx->d_tmp_counts.p, n_cand * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    }
    EBIC_CUDA(cudaStreamSynchronize(s));
    const int e = *(volatile int*)ctx->h_err1.p;
    if (e == 2) return fail(EBIC_ERR_INVALID_ARGUMENT, "a candidate is empty or its offsets decrease");
    if (e) return bad_column_error(ctx);
    return EBIC_OK;
  }
  uint64_t t = 0;
  EBIC_TRY(ebic_eval_submit(ctx, cols, offsets, n_cand, approx, negative_trends, counts_out, &t));
  return ebic_eval_wait(ctx, t);
}

int ebic_support_rows_batch(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                            uint64_t n_cand, double approx, int negative_trends, uint32_t* rows_out,
                            uint64_t cap, uint64_t* row_offsets) {
  NvtxRange nvtx_("ebic:support_rows_batch");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  if (!row_offsets) return fail(EBIC_ERR_INVALID_ARGUMENT, "null row_offsets");
  EBIC_TRY(validate_population(ctx, cols, offsets, n_cand));
  EBIC_TRY(set_device(ctx));
  row_offsets[0] = 0;
  if (n_cand == 0) return EBIC_OK;
  cudaStream_t s = ctx->stream;
  const uint64_t n_idx = offsets[n_cand];
  const uint64_t wpc = ctx->ld / 32;  // mask words per candidate
  EBIC_TRY(ensure(ctx->d_tmp_cols, n_idx));
  EBIC_TRY(ensure(ctx->d_tmp_offs, n_cand + 1));
  EBIC_TRY(ensure(ctx->d_tmp_counts, n_cand));
  EBIC_TRY(ensure(ctx->h_tmp_counts, n_cand));
  EBIC_TRY(ensure(ctx->d_mask, n_cand * wpc));
  EBIC_TRY(ensure(ctx->d_row_offsets, n_cand + 1));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_cols.p, cols, n_idx * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_offs.p, offsets, (n_cand + 1) * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_tmp_counts.p, 0, n_cand * sizeof(uint32_t), s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_mask.p, 0, n_cand * wpc * sizeof(uint32_t), s));
  EBIC_TRY(launch_count<true>(ctx, ctx->d_tmp_cols.p, ctx->d_tmp_offs.p, n_cand, approx,
                              negative_trends, ctx->d_tmp_counts.p, ctx->d_mask.p, s));
  EBIC_CUDA(cudaMemcpyAsync(ctx->h_tmp_counts.p, ctx->d_tmp_counts.p, n_cand * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s));
  EBIC_CUDA(cudaStreamSynchronize(s));
  for (uint64_t i = 0; i < n_cand; ++i) row_offsets[i + 1] = row_offsets[i] + ctx->h_tmp_counts.p[i];
  const uint64_t total = row_offsets[n_cand];
  if (total > cap) return fail(EBIC_ERR_CAPACITY, "need %llu row slots, have %llu",
                               (unsigned long long)total, (unsigned long long)cap);
  if (total == 0) return EBIC_OK;
  if (!rows_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null rows_out");
  EBIC_TRY(ensure(ctx->d_rows, total));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_row_offsets.p, row_offsets, (n_cand + 1) * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, s));
  const uint64_t n_words_valid = (ctx->n_rows + 31) / 32;
  ebic::scatter_rows_kernel<<<(unsigned)n_cand, ebic::kScatterThreads, 0, s>>>(
      ctx->d_mask.p, wpc, n_words_valid, ctx->d_row_offsets.p, ctx->row_base, ctx->d_rows.p);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  EBIC_CUDA(cudaMemcpyAsync(rows_out, ctx->d_rows.p, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  EBIC_CUDA(cudaStreamSynchronize(s));
  return EBIC_OK;
}

int ebic_support_overlap_batch(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets, uint64_t n_cand,
                               double approx, int negative_trends, uint64_t* sizes_out, uint64_t* inter_out) {
  NvtxRange nvtx_("ebic:support_overlap_batch");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  if (n_cand > EBIC_OVERLAP_MAX)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "%llu candidates (at most %d per overlap batch)",
                (unsigned long long)n_cand, EBIC_OVERLAP_MAX);
  if (n_cand && (!sizes_out || !inter_out)) return fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
  EBIC_TRY(validate_population(ctx, cols, offsets, n_cand));
  EBIC_TRY(set_device(ctx));
  if (n_cand == 0) return EBIC_OK;
  cudaStream_t s = ctx->stream;
  const uint64_t n_idx = offsets[n_cand];
  const uint64_t wpc = ctx->ld / 32;  // mask words per candidate
  const uint64_t nn = n_cand * n_cand;
  EBIC_TRY(ensure(ctx->d_tmp_cols, n_idx));
  EBIC_TRY(ensure(ctx->d_tmp_offs, n_cand + 1));
  EBIC_TRY(ensure(ctx->d_tmp_counts, n_cand));
  EBIC_TRY(ensure(ctx->h_tmp_counts, n_cand));
  EBIC_TRY(ensure(ctx->d_mask, n_cand * wpc));
  EBIC_TRY(ensure(ctx->d_inter, nn));
  EBIC_TRY(ensure(ctx->h_inter, nn));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_cols.p, cols, n_idx * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_offs.p, offsets, (n_cand + 1) * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_tmp_counts.p, 0, n_cand * sizeof(uint32_t), s));
  EBIC_CUDA(cudaMemsetAsync(ctx->d_mask.p, 0, n_cand * wpc * sizeof(uint32_t), s));
  EBIC_TRY(launch_count<true>(ctx, ctx->d_tmp_cols.p, ctx->d_tmp_offs.p, n_cand, approx, negative_trends,
                              ctx->d_tmp_counts.p, ctx->d_mask.p, s));
  const dim3 grid((unsigned)n_cand, (unsigned)((n_cand + ebic::kOverlapTile - 1) / ebic::kOverlapTile));
  ebic::overlap_popc_kernel<<<grid, ebic::kOverlapThreads, 0, s>>>(ctx->d_mask.p, wpc, (ctx->n_rows + 31) / 32,
                                                                  (uint32_t)n_cand, ctx->d_inter.p);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  EBIC_CUDA(cudaMemcpyAsync(ctx->h_tmp_counts.p, ctx->d_tmp_counts.p, n_cand * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s));
  EBIC_CUDA(cudaMemcpyAsync(ctx->h_inter.p, ctx->d_inter.p, nn * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  EBIC_CUDA(cudaStreamSynchronize(s));
  for (uint64_t i = 0; i < n_cand; ++i) sizes_out[i] = ctx->h_tmp_counts.p[i];
  for (uint64_t k = 0; k < nn; ++k) inter_out[k] = ctx->h_inter.p[k];
  return EBIC_OK;
}

int ebic_support_rows(ebic_ctx* ctx, const uint32_t* cols, uint32_t len, double approx,
                      int negative_trends, uint32_t* rows_out, uint64_t cap, uint64_t* n_out) {
  NvtxRange nvtx_("ebic:support_rows");
  const uint32_t offs[2] = {0, len};
  uint64_t ro[2] = {0, 0};
  int st = ebic_support_rows_batch(ctx, cols, offs, 1, approx, negative_trends, rows_out, cap, ro);
  if (n_out && (st == EBIC_OK || st == EBIC_ERR_CAPACITY)) *n_out = ro[1];
  return st;
}

int ebic_row_supports(ebic_ctx* ctx, uint64_t row, const uint32_t* cols, uint32_t len, double approx,
                      int negative_trends, int* supports_out) {
  NvtxRange nvtx_("ebic:row_supports");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  if (!supports_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null supports_out");
  if (row < ctx->row_base || row >= ctx->row_base + ctx->n_rows)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "row %llu outside the resident shard",
                (unsigned long long)row);
  const uint32_t offs[2] = {0, len};
  EBIC_TRY(validate_population(ctx, cols, offs, 1));
  EBIC_TRY(set_device(ctx));
  cudaStream_t s = ctx->stream;
  EBIC_TRY(ensure(ctx->d_tmp_cols, len));
  EBIC_CUDA(cudaMemcpyAsync(ctx->d_tmp_cols.p, cols, len * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  const uint64_t lr = row - ctx->row_base;
  if (ctx->store == EBIC_STORE_F32)
    ebic::row_supports_kernel<float><<<1, 32, 0, s>>>((const float*)ctx->d_mat, ctx->ld, lr,
                                                       ctx->d_tmp_cols.p, len, approx,
                                                       negative_trends, ctx->d_out1);
  else
    ebic::row_supports_kernel<double><<<1, 32, 0, s>>>((const double*)ctx->d_mat, ctx->ld, lr,
                                                        ctx->d_tmp_cols.p, len, approx,
                                                        negative_trends, ctx->d_out1);
  ctx->launches++;
  EBIC_CUDA(cudaGetLastError());
  int out = 0;
  EBIC_CUDA(cudaMemcpyAsync(&out, ctx->d_out1, sizeof(int), cudaMemcpyDeviceToHost, s));
  EBIC_CUDA(cudaStreamSynchronize(s));
  *supports_out = out;
  return EBIC_OK;
}

double ebic_fitness(uint64_t support_count, uint64_t num_cols, uint64_t min_rows, uint64_t col_cap) {
  if (support_count < min_rows) return 0.0;
  const int bonus = (int)std::min(num_cols, col_cap);
  return std::ldexp((double)support_count, bonus);
}

int ebic_ctx_launch_count(ebic_ctx* ctx, uint64_t* n_out) {
  if (!ctx || !n_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
  *n_out = ctx->launches;
  return EBIC_OK;
}

int ebic_ctx_set_slab_rows(ebic_ctx* ctx, uint32_t slab_rows) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (slab_rows % ebic::kRowAlign)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "slab_rows must be a multiple of %u", ebic::kRowAlign);
  ctx->slab_rows = slab_rows;
  return EBIC_OK;
}

int ebic_ctx_set_pair_layout(ebic_ctx* ctx, int rows_per_lane_pairs, int cands_per_warp) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (rows_per_lane_pairs == 0 && cands_per_warp == 0) {
    ctx->simd_force = 0;
    return EBIC_OK;
  }
  const bool ok_p = rows_per_lane_pairs == 1 || rows_per_lane_pairs == 2;
  const bool ok_s = cands_per_warp == 1 || cands_per_warp == 2 || cands_per_warp == 4;
  if (!ok_p || !ok_s)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "bad packed-pair layout (%d, %d)", rows_per_lane_pairs, cands_per_warp);
  ctx->simd_force = rows_per_lane_pairs * 16 + cands_per_warp;
  return EBIC_OK;
}

int ebic_ctx_set_lazy_build(ebic_ctx* ctx, int mode) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (mode < EBIC_LAZY_BUILD_AUTO || mode > EBIC_LAZY_BUILD_FIRST)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "lazy build mode %d (0 auto, 1 inline, 2 build first)", mode);
  ctx->lazy_build = mode;
  return EBIC_OK;
}

int ebic_ctx_set_table_budget(ebic_ctx* ctx, uint64_t bytes) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  ctx->table_budget_user = bytes;
  if (ctx->d_mat) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      fr = 0;
    }
    ctx->table_budget = index_budget(ctx, fr + ctx->table_cap);
  }
  return EBIC_OK;
}

int ebic_matrix_index_info(ebic_ctx* ctx, uint64_t* bytes_needed, int* in_use) {
  EBIC_TRY(need_matrix(ctx));
  if (bytes_needed) *bytes_needed = plane_fits(ctx) ? table_bytes(ctx) : 0;
  if (in_use) *in_use = ctx->table_valid ? 1 : 0;
  return EBIC_OK;
}

int ebic_matrix_build_info(ebic_ctx* ctx, double* alloc_ms, double* plane_ms, double* index_ms) {
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(set_device(ctx));
  float pm = 0.f, im = 0.f;
  if (ctx->plane_timed) {
    EBIC_CUDA(cudaEventSynchronize(ctx->ev_build[1]));
    EBIC_CUDA(cudaEventElapsedTime(&pm, ctx->ev_build[0], ctx->ev_build[1]));
  }
  if (ctx->index_timed) {
    EBIC_CUDA(cudaEventSynchronize(ctx->ev_build[3]));
    EBIC_CUDA(cudaEventElapsedTime(&im, ctx->ev_build[2], ctx->ev_build[3]));
  }
  if (alloc_ms) *alloc_ms = ctx->index_timed ? ctx->index_alloc_ms : 0.0;
  if (plane_ms) *plane_ms = pm;
  if (index_ms) *index_ms = im;
  return EBIC_OK;
}

int ebic_matrix_index_stats(ebic_ctx* ctx, int* mode, uint64_t* full_bytes, uint64_t* lazy_slots_used,
                            uint64_t* lazy_slots_cap, uint64_t* lazy_bytes, uint64_t* lazy_built,
                            uint64_t* lazy_resets) {
  EBIC_TRY(need_matrix(ctx));
  const uint64_t vec = table_wp(ctx) * sizeof(uint32_t);
  const uint32_t m_count = ctx->h_lmirror.p ? *(volatile uint32_t*)&ctx->h_lmirror.p[0] : 0;
  if (mode) *mode = ctx->index_mode;
  if (full_bytes) *full_bytes = ctx->table_valid ? table_bytes(ctx) : 0;
  if (lazy_slots_used) *lazy_slots_used = ctx->lazy_valid ? std::min<uint64_t>(m_count, ctx->lcap) : 0;
  if (lazy_slots_cap) *lazy_slots_cap = ctx->lcap;
  if (lazy_bytes) *lazy_bytes = ctx->lcap * vec + (ctx->d_lmap ? lazy_map_bytes(ctx) : 0);
  if (lazy_built) *lazy_built = ctx->lazy_built;
  if (lazy_resets) *lazy_resets = ctx->lazy_resets;
  return EBIC_OK;
}

int ebic_ctx_set_path(ebic_ctx* ctx, int path) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (path < EBIC_PATH_AUTO || path > EBIC_PATH_LAZY) return fail(EBIC_ERR_INVALID_ARGUMENT, "bad path %d", path);
  ctx->path = path;
  return EBIC_OK;
}

int ebic_matrix_prepare(ebic_ctx* ctx, double approx) {
  NvtxRange nvtx_("ebic:matrix_prepare");
  EBIC_TRY(need_matrix(ctx));
  EBIC_TRY(check_approx(approx));
  EBIC_TRY(set_device(ctx));
  if (ctx->path == EBIC_PATH_VALUE) return EBIC_OK;
  // an explicit request: the full index now if it fits the budget (else the
  // lazy index, or the rank plane of the slab kernels)
  ctx->full_requested = true;
  IndexPlan plan;
  EBIC_TRY(use_index(ctx, approx, 0, ctx->stream, &plan.mode, &plan.la));
  if (plan.mode == kIndexNone && plane_fits(ctx)) EBIC_TRY(ensure_plane(ctx, approx, ctx->stream));
  EBIC_CUDA(cudaStreamSynchronize(ctx->stream));
  return EBIC_OK;
}

// ---- matrix ingest (ebic_tsv.cpp) -------------------------------------------

__attribute__((visibility("hidden"))) int ebic_internal_fail(int code, const char* msg) {
  return fail(code, "%s", msg);
}

int ebic_matrix_load_tsv(ebic_ctx* ctx, const char* path, int n_threads, int store, int* store_out,
                         uint64_t* rows_out, uint64_t* cols_out) {
  NvtxRange nvtx_("ebic:matrix_load_tsv");
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  uint64_t rows = 0, cols = 0;
  const int st = ebic_tsv_read(path, n_threads, nullptr, 0, &rows, &cols);
  if (st != EBIC_ERR_CAPACITY) return st;  // the shape query reports CAPACITY on success
  EBIC_TRY(set_device(ctx));
  // parse straight into page-locked memory: the upload DMAs it from there
  HostBuf<double> staging;
  EBIC_TRY(ensure(staging, rows * cols));
  const int st2 = ebic_tsv_read(path, n_threads, staging.p, rows * cols, &rows, &cols);
  if (st2 != EBIC_OK) {
    staging.release();
    return st2;
  }
  const int st3 = upload_impl<double>(ctx, staging.p, rows, cols, 0, store, store_out);
  staging.release();
  if (st3 == EBIC_OK) {
    if (rows_out) *rows_out = rows;
    if (cols_out) *cols_out = cols;
  }
  return st3;
}

// ---- row-shard exchange over peer memory ----------------------------------

}  // extern "C"

namespace {

// Every peer's window header must match ours: same world size and inbox size
// (a push into a smaller peer's inbox would write past its window).
int check_peer_header(ebic_ctx* ctx, int g) {
  ebic::XchgHeader h{};
  EBIC_CUDA(cudaMemcpy(&h, ctx->xchg_peer[g], sizeof(h), cudaMemcpyDefault));
  if (h.magic != ebic::kXchgMagic)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "peer window %d is not an exchange window", g);
  if ((int)h.world != ctx->xchg_world || h.max_cand != (uint32_t)ctx->xchg_max)
    return fail(EBIC_ERR_INVALID_ARGUMENT,
                "peer window %d was created with world=%u max_cand=%u; this rank has world=%d max_cand=%llu", g,
                h.world, h.max_cand, ctx->xchg_world, (unsigned long long)ctx->xchg_max);
  return EBIC_OK;
}

int xchg_ready(ebic_ctx* ctx, uint64_t n_cand, const void* d_cols, const void* d_offsets, const void* d_counts) {
  EBIC_TRY(need_matrix(ctx));
  if (!ctx->xchg_win) return fail(EBIC_ERR_INVALID_ARGUMENT, "no exchange window (ebic_xchg_create)");
  for (int g = 0; g < ctx->xchg_world; ++g)
    if (!ctx->xchg_peer[g]) return fail(EBIC_ERR_INVALID_ARGUMENT, "peer window %d not opened", g);
  if (n_cand > ctx->xchg_max)
    return fail(EBIC_ERR_CAPACITY, "%llu candidates exceed the exchange window (%llu)", (unsigned long long)n_cand,
                (unsigned long long)ctx->xchg_max);
  if (n_cand && (!d_cols || !d_offsets || !d_counts)) return fail(EBIC_ERR_INVALID_ARGUMENT, "null device pointer");
  return EBIC_OK;
}

// One pipelined row-sharded step (see ctx->kXchgDepth): count on `s` into the
// ring slot's local buffer, exchange on the context's exchange stream.  Every
// rank runs the same sequence of steps, so the epochs agree -- including when
// this rank's count fails: the exchange still runs (pushing zeros and
// poisoning the peers' windows), so no rank is left an epoch behind, and the
// count's error is returned afterwards.
int rows_sum_step(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets, uint64_t n_cand, double approx,
                  int neg, uint32_t* d_counts, cudaStream_t s) {
  const uint64_t k = ctx->xchg_epoch;  // steps issued so far
  const int slot = (int)(k % ebic_ctx::kXchgDepth);
  cudaStream_t xs = ctx->xchg_stream;
  // the slot's buffer was last read by the exchange of step k - depth
  if (ctx->xchg_xdone_armed[slot]) EBIC_CUDA(cudaStreamWaitEvent(s, ctx->xchg_xdone[slot], 0));
  int st = check_approx(approx);
  if (st == EBIC_OK && n_cand)
    st = count_into(ctx, d_cols, d_offsets, n_cand, approx, neg, ctx->d_xchg_local[slot].p, nullptr, s);
  const std::string count_error = st == EBIC_OK ? std::string() : g_last_error;
  EBIC_CUDA(cudaEventRecord(ctx->xchg_cdone[slot], s));
  EBIC_CUDA(cudaStreamWaitEvent(xs, ctx->xchg_cdone[slot], 0));
  const uint64_t epoch = k + 1;
  ebic::XchgPeers peers;
  for (int g = 0; g < ebic::kMaxRanks; ++g) peers.win[g] = ctx->xchg_peer[g];
  ebic::xchg_sum_kernel<<<ebic::kXchgCtas, 256, 0, xs>>>(ctx->d_xchg_local[slot].p, (uint32_t)n_cand, peers,
                                                          ctx->xchg_world, ctx->xchg_rank, epoch,
                                                          (uint32_t)ctx->xchg_max, d_counts, ctx->d_err,
                                                          st == EBIC_OK ? 0 : 1, ctx->xchg_timeout_ns);
  ctx->launches++;
  const cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess)  // the exchange never launched: the epoch did not advance
    return fail(EBIC_ERR_CUDA, "exchange kernel launch: %s", cudaGetErrorString(le));
  ctx->xchg_epoch = epoch;  // only once the exchange is in the stream
  EBIC_CUDA(cudaEventRecord(ctx->xchg_xdone[slot], xs));
  ctx->xchg_xdone_armed[slot] = true;
  if (st != EBIC_OK) return fail(st, "%s (the exchange ran with zeros and poisoned the peers)", count_error.c_str());
  return EBIC_OK;
}

int xchg_fence(ebic_ctx* ctx, cudaStream_t s) {
  if (!ctx->xchg_stream) return EBIC_OK;
  const uint64_t k = ctx->xchg_epoch;
  if (k == 0) return EBIC_OK;
  const int last = (int)((k - 1) % ebic_ctx::kXchgDepth);  // the exchanges are serialised on xchg_stream
  EBIC_CUDA(cudaStreamWaitEvent(s, ctx->xchg_xdone[last], 0));
  return EBIC_OK;
}

}  // namespace

extern "C" {

int ebic_xchg_create(ebic_ctx* ctx, int world, int rank, uint64_t max_cand, void* handle_out) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  if (world < 1 || world > ebic::kMaxRanks || rank < 0 || rank >= world)
    return fail(EBIC_ERR_INVALID_ARGUMENT, "bad world/rank (%d, %d); at most %d ranks", world, rank, ebic::kMaxRanks);
  if (max_cand == 0 || max_cand > 0x7fffffffull) return fail(EBIC_ERR_INVALID_ARGUMENT, "bad max_cand");
  EBIC_TRY(set_device(ctx));
  EBIC_TRY(ebic_xchg_destroy(ctx));
  const size_t bytes = ebic::xchg_window_bytes((uint32_t)max_cand);
  EBIC_CUDA(cudaMalloc(&ctx->xchg_win, bytes));
  EBIC_CUDA(cudaMemset(ctx->xchg_win, 0, bytes));
  const ebic::XchgHeader h{ebic::kXchgMagic, (uint32_t)world, (uint32_t)max_cand, 0u};
  EBIC_CUDA(cudaMemcpy(ctx->xchg_win, &h, sizeof(h), cudaMemcpyHostToDevice));
  // the step must not allocate: a device allocation can wait for an idle
  // device, i.e. for another rank's exchange kernel on a shared GPU
  for (auto& b : ctx->d_xchg_local) EBIC_TRY(ensure(b, max_cand));
  if (!ctx->xchg_stream) EBIC_CUDA(cudaStreamCreateWithFlags(&ctx->xchg_stream, cudaStreamNonBlocking));
  for (int i = 0; i < ebic_ctx::kXchgDepth; ++i) {
    if (!ctx->xchg_cdone[i]) EBIC_CUDA(cudaEventCreateWithFlags(&ctx->xchg_cdone[i], cudaEventDisableTiming));
    if (!ctx->xchg_xdone[i]) EBIC_CUDA(cudaEventCreateWithFlags(&ctx->xchg_xdone[i], cudaEventDisableTiming));
    ctx->xchg_xdone_armed[i] = false;
  }
  ctx->xchg_world = world;
  ctx->xchg_rank = rank;
  ctx->xchg_max = max_cand;
  ctx->xchg_epoch = 0;
  for (auto& p : ctx->xchg_peer) p = nullptr;
  ctx->xchg_peer[rank] = ctx->xchg_win;
  if (handle_out) {
    cudaIpcMemHandle_t ih;
    EBIC_CUDA(cudaIpcGetMemHandle(&ih, ctx->xchg_win));
    std::memcpy(handle_out, &ih, sizeof(ih));
  }
  return EBIC_OK;
}

int ebic_xchg_window(ebic_ctx* ctx, void** window_out) {
  if (!ctx || !window_out) return fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
  if (!ctx->xchg_win) return fail(EBIC_ERR_INVALID_ARGUMENT, "no exchange window (ebic_xchg_create)");
  *window_out = ctx->xchg_win;
  return EBIC_OK;
}

int ebic_xchg_open(ebic_ctx* ctx, const void* handles) {
  if (!ctx || !handles) return fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
  if (!ctx->xchg_win) return fail(EBIC_ERR_INVALID_ARGUMENT, "no exchange window (ebic_xchg_create)");
  EBIC_TRY(set_device(ctx));
  for (int g = 0; g < ctx->xchg_world; ++g) {
    if (g == ctx->xchg_rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + (size_t)g * EBIC_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    EBIC_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->xchg_peer[g] = static_cast<unsigned char*>(p);
    ctx->xchg_ipc_opened[g] = true;
    EBIC_TRY(check_peer_header(ctx, g));
  }
  return EBIC_OK;
}

int ebic_xchg_open_local(ebic_ctx* ctx, void* const* windows) {
  if (!ctx || !windows) return fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
  if (!ctx->xchg_win) return fail(EBIC_ERR_INVALID_ARGUMENT, "no exchange window (ebic_xchg_create)");
  EBIC_TRY(set_device(ctx));
  for (int g = 0; g < ctx->xchg_world; ++g) {
    if (g == ctx->xchg_rank) continue;
    if (!windows[g]) return fail(EBIC_ERR_INVALID_ARGUMENT, "null window for rank %d", g);
    ctx->xchg_peer[g] = static_cast<unsigned char*>(windows[g]);
    const int st = check_peer_header(ctx, g);
    if (st != EBIC_OK) {
      ctx->xchg_peer[g] = nullptr;
      return st;
    }
  }
  return EBIC_OK;
}

int ebic_xchg_destroy(ebic_ctx* ctx) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  cudaSetDevice(ctx->device);
  if (ctx->xchg_stream) cudaStreamSynchronize(ctx->xchg_stream);
  for (int g = 0; g < ebic::kMaxRanks; ++g) {
    if (ctx->xchg_ipc_opened[g] && ctx->xchg_peer[g]) cudaIpcCloseMemHandle(ctx->xchg_peer[g]);
    ctx->xchg_ipc_opened[g] = false;
    ctx->xchg_peer[g] = nullptr;
  }
  if (ctx->xchg_win) cudaFree(ctx->xchg_win);
  ctx->xchg_win = nullptr;
  ctx->xchg_world = 0;
  ctx->xchg_epoch = 0;
  for (auto& b : ctx->d_xchg_local) b.release();
  for (bool& a : ctx->xchg_xdone_armed) a = false;
  return EBIC_OK;
}

int ebic_eval_counts_rows_sum_async(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets,
                                    uint64_t n_cand, double approx, int negative_trends, uint32_t* d_counts,
                                    void* stream) {
  NvtxRange nvtx_("ebic:eval_counts_rows_sum_async");
  EBIC_TRY(xchg_ready(ctx, n_cand, d_cols, d_offsets, d_counts));
  EBIC_TRY(set_device(ctx));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  return rows_sum_step(ctx, d_cols, d_offsets, n_cand, approx, negative_trends, d_counts, s);
}

int ebic_xchg_fence(ebic_ctx* ctx, void* stream) {
  if (!ctx) return fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
  EBIC_TRY(set_device(ctx));
  return xchg_fence(ctx, stream ? static_cast<cudaStream_t>(stream) : ctx->stream);
}

int ebic_eval_counts_rows_sum(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets, uint64_t n_cand,
                              double approx, int negative_trends, uint32_t* d_counts, void* stream) {
  NvtxRange nvtx_("ebic:eval_counts_rows_sum");
  EBIC_TRY(xchg_ready(ctx, n_cand, d_cols, d_offsets, d_counts));
  EBIC_TRY(set_device(ctx));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  const int st = rows_sum_step(ctx, d_cols, d_offsets, n_cand, approx, negative_trends, d_counts, s);
  EBIC_TRY(xchg_fence(ctx, s));  // the summed counts are ordered on `stream`
  return st;
}

}  // extern "C"
