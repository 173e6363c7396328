/*
 * ebic.h -- C ABI of the B200 batched bicluster-fitness evaluator.
 *
 * This is the drop-in boundary for the reference's trend/fitness engine
 * (/root/reference/proj/include/bicseek/trend.hpp).  The reference has no FFI
 * of its own: its seam is link-time substitution of the free functions in
 * trend.hpp.  The C++ TU paper_2105_01196_b200/csrc/bicseek_trend_device.cpp
 * implements those functions over this ABI, and the
 * Python mirror (paper_2105_01196_b200/trend.py) binds it with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types.
 *   - Every entry point returns an int status: EBIC_OK (0) or an EBIC_ERR_*
 *     code.  ebic_last_error() returns a thread-local message for the last
 *     failure on the calling thread.
 *   - A context (ebic_ctx) owns one CUDA device, one stream, one resident
 *     matrix shard and the pinned staging buffers.  Contexts are independent
 *     and may be used concurrently from different threads; a single context
 *     must not be used by two threads at once (like the reference WorkerPool,
 *     worker_pool.hpp:32).
 *   - Populations are CSR: candidate i is the column sequence
 *     cols[offsets[i] .. offsets[i+1]) (reference: std::vector<Chromosome>,
 *     bicluster.hpp:13-24).  Column indices are uint32, in visiting order.
 *   - Row indices returned by the row-membership calls are GLOBAL
 *     (row_base + local row), ascending.
 *
 * Numerics: results are bit-exact with the reference CPU path
 * (trend.cpp:17-46, double-precision `cur > prev - approx*|prev|` with two
 * rounded ops) for every input the store accepts.  A float32 store is used
 * only when every value is float32-representable; otherwise the store keeps
 * float64 (EBIC_STORE_AUTO), so there is no silent precision loss and no CPU
 * fallback.
 */
#ifndef EBIC_H_
#define EBIC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBIC_ABI_VERSION 1

/* status codes */
#define EBIC_OK 0
#define EBIC_ERR_INVALID_ARGUMENT 1 /* bad sizes, out-of-range column, empty candidate, non-finite value */
#define EBIC_ERR_CUDA 2             /* CUDA runtime / launch failure (message has the CUDA error string) */
#define EBIC_ERR_NO_MATRIX 3        /* no matrix uploaded in this context */
#define EBIC_ERR_CAPACITY 4         /* output buffer too small; required size returned */
#define EBIC_ERR_NOT_EXACT 5        /* EBIC_STORE_F32 requested for a matrix that is not f32-representable */
#define EBIC_ERR_NO_DEVICE 6        /* no CUDA device / bad device ordinal */
#define EBIC_ERR_IO 7               /* file cannot be opened / read */

/* matrix store precision */
#define EBIC_STORE_AUTO 0 /* float32 if every value is exactly representable, else float64 */
#define EBIC_STORE_F32 1  /* float32 (column-major, rows padded to 32); error if not exact */
#define EBIC_STORE_F64 2  /* float64 (column-major, rows padded to 32) */

typedef struct ebic_ctx ebic_ctx;

/* ---- library / context ------------------------------------------------- */

int ebic_abi_version(void);
/* Thread-local message describing the last non-OK status on this thread. */
const char* ebic_last_error(void);
/* Number of visible CUDA devices (0 if none). */
int ebic_device_count(int* n_out);

/* Create a context on `device`.  Owns a non-blocking CUDA stream. */
int ebic_ctx_create(int device, ebic_ctx** ctx_out);
int ebic_ctx_destroy(ebic_ctx* ctx);
/* Use an external stream (e.g. torch.cuda.current_stream().cuda_stream) for
 * every subsequent launch; NULL restores the context's own stream. */
int ebic_ctx_set_stream(ebic_ctx* ctx, void* cuda_stream);
/* Block until all work queued by this context has finished; also reports any
 * device-side argument error recorded by the *_device entry points. */
int ebic_ctx_sync(ebic_ctx* ctx);

/* ---- device-resident matrix store (reference: ExpressionMatrix,
 *      matrix.hpp:13-43, row-major double) ----------------------------------- */

/* Upload `n_rows` x `n_cols` row-major doubles (a whole matrix, or the row
 * shard [row_base, row_base + n_rows) of a larger one).  Transposes on device
 * to column-major with rows padded to a multiple of 32.  Non-finite values
 * are rejected (matrix.cpp:41-42).  *store_out (optional) receives the chosen
 * EBIC_STORE_F32 / EBIC_STORE_F64.  Replaces any previous matrix; the previous
 * pair-trend index ALLOCATION is kept and reused when the new index fits it
 * (at most twice the need), else released -- ebic_matrix_free releases
 * everything. */
int ebic_matrix_upload_f64(ebic_ctx* ctx, const double* row_major, uint64_t n_rows,
                           uint64_t n_cols, uint64_t row_base, int store, int* store_out);
/* Same for row-major float32 input (always exact; stored as float32). */
int ebic_matrix_upload_f32(ebic_ctx* ctx, const float* row_major, uint64_t n_rows,
                           uint64_t n_cols, uint64_t row_base);
/* The same two from DEVICE memory on the context's GPU -- e.g. a row-major
 * buffer an NCCL broadcast filled (the replicated matrix is
 * uploaded once and broadcast over NVLink).  The buffer is checked and
 * transposed in place (not modified) and may be freed after the call.  Its
 * contents must be complete when the call is made (synchronise the stream
 * that filled it). */
int ebic_matrix_upload_device_f64(ebic_ctx* ctx, const double* d_row_major, uint64_t n_rows,
                                  uint64_t n_cols, uint64_t row_base, int store, int* store_out);
int ebic_matrix_upload_device_f32(ebic_ctx* ctx, const float* d_row_major, uint64_t n_rows,
                                  uint64_t n_cols, uint64_t row_base);
/* Shape of the resident matrix.  Any out pointer may be NULL. */
int ebic_matrix_info(ebic_ctx* ctx, uint64_t* n_rows, uint64_t* n_cols, uint64_t* ld,
                     int* store, uint64_t* row_base);
int ebic_matrix_free(ebic_ctx* ctx);

/* ---- matrix ingest (reference: parse_matrix_tsv, io.cpp:78-111) ---------
 * The reference's TSV format and rules (header of column labels with an
 * optional corner cell, one line per row of label + values, '\r' stripped,
 * trailing empty lines ignored, every value parsed with std::from_chars and
 * required finite) with its error messages, parsed on n_threads host threads
 * (<= 0: all).  Values are bit-identical to the reference parser's. */
/* Row-major doubles into values_out (cap elements).  *rows_out / *cols_out
 * receive the shape; EBIC_ERR_CAPACITY (shape filled) if cap is too small, so
 * a call with cap = 0 queries the shape. */
int ebic_tsv_read(const char* path, int n_threads, double* values_out, uint64_t cap, uint64_t* rows_out,
                  uint64_t* cols_out);
/* Parse into page-locked memory and upload as the context's matrix (as
 * ebic_matrix_upload_f64 with row_base 0). */
int ebic_matrix_load_tsv(ebic_ctx* ctx, const char* path, int n_threads, int store, int* store_out,
                         uint64_t* rows_out, uint64_t* cols_out);

/* ---- fitness counts (reference: evaluate_population, trend.cpp:56-72) ---- */

/* Host pointers, synchronous.  counts_out[i] = number of rows r of the
 * resident matrix (shard) with row_supports(r, candidate i).  Offsets are
 * validated on the host, column indices on the device (an out-of-range column
 * returns EBIC_ERR_INVALID_ARGUMENT; that candidate's count is 0).  If all
 * three arrays are page-locked (cudaHostAlloc / cudaHostRegister / torch
 * pin_memory) they are DMA'd directly, with no staging copy. */
int ebic_eval_counts(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                     uint64_t n_cand, double approx, int negative_trends, uint32_t* counts_out);

/* Device pointers, asynchronous on `stream` (NULL = the context's stream).
 * d_counts is overwritten.  Invalid columns / empty candidates are detected on
 * device, counted as 0 and reported by the next ebic_ctx_sync().  The
 * context's device scratch is shared by its launches: work of one context
 * submitted on different streams must not overlap in time (order it, or use
 * one context per stream). */
int ebic_eval_counts_device(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets,
                            uint64_t n_cand, double approx, int negative_trends,
                            uint32_t* d_counts, void* stream);

/* Batch marshaller: asynchronous host-pointer evaluation through pinned
 * staging slots (ring of EBIC_MARSHAL_SLOTS).  The caller's host arrays are
 * copied into pinned memory before return, so they may be reused at once;
 * counts_out is written when ebic_eval_wait(ticket) returns.  Lets the
 * host-side GA breed the next chunk while this one is evaluated. */
#define EBIC_MARSHAL_SLOTS 4
int ebic_eval_submit(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                     uint64_t n_cand, double approx, int negative_trends, uint32_t* counts_out,
                     uint64_t* ticket_out);
int ebic_eval_wait(ebic_ctx* ctx, uint64_t ticket);

/* ---- row membership (reference: supporting_rows trend.cpp:48-54,
 *      row_supports trend.cpp:41-46) --------------------------------------- */

/* Ascending global rows supporting one candidate.  *n_out receives the full
 * count; if it exceeds `cap`, returns EBIC_ERR_CAPACITY and writes nothing. */
int ebic_support_rows(ebic_ctx* ctx, const uint32_t* cols, uint32_t len, double approx,
                      int negative_trends, uint32_t* rows_out, uint64_t cap, uint64_t* n_out);

/* Batched variant (one launch sequence for a whole archive): rows of
 * candidate i land in rows_out[row_offsets[i] .. row_offsets[i+1]).
 * row_offsets has n_cand + 1 entries.  If the total exceeds `cap`, returns
 * EBIC_ERR_CAPACITY with row_offsets filled and rows_out untouched. */
int ebic_support_rows_batch(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                            uint64_t n_cand, double approx, int negative_trends,
                            uint32_t* rows_out, uint64_t cap, uint64_t* row_offsets);

/* Row-set overlaps of a batch, for the archive's overlap filter without row
 * lists (reference: TopRankList::insert evolution.cpp:76-105,
 * induced_jaccard evolution.cpp:44-51, sorted_intersection_size).
 * sizes_out[i] = |supporting_rows(c_i)| (n_cand entries) and
 * inter_out[i * n_cand + j] = |supporting_rows(c_i) n supporting_rows(c_j)|
 * (n_cand * n_cand entries, symmetric, diagonal = sizes).  The row sets stay on
 * the device as bitmasks; only the counts come back.  At most
 * EBIC_OVERLAP_MAX candidates per call. */
#define EBIC_OVERLAP_MAX 4096
int ebic_support_overlap_batch(ebic_ctx* ctx, const uint32_t* cols, const uint32_t* offsets,
                               uint64_t n_cand, double approx, int negative_trends,
                               uint64_t* sizes_out, uint64_t* inter_out);

/* Single (row, candidate) predicate on device.  `row` is a GLOBAL row index
 * inside the resident shard. */
int ebic_row_supports(ebic_ctx* ctx, uint64_t row, const uint32_t* cols, uint32_t len,
                      double approx, int negative_trends, int* supports_out);

/* ---- score (reference: fitness trend.cpp:74-79; host arithmetic, exact) -- */
double ebic_fitness(uint64_t support_count, uint64_t num_cols, uint64_t min_rows,
                    uint64_t col_cap);

/* ---- instrumentation ---------------------------------------------------- */

/* Number of kernels this context has launched since creation. */
int ebic_ctx_launch_count(ebic_ctx* ctx, uint64_t* n_out);
/* Tuning knob for the value-path kernel: rows per CTA slab (0 = auto). */
int ebic_ctx_set_slab_rows(ebic_ctx* ctx, uint32_t slab_rows);

/* Evaluation path.  AUTO: a pair-trend index -- the full one (every
 * consecutive-pair test of the matrix as row bitsets, built once per matrix x
 * approx; C^2 x R/8 bytes) when it is small (<= 1 GiB), requested
 * (ebic_matrix_prepare) or paid for (ski rental: once the lazy index has built
 * half of the C^2 pairs), or else the LAZY one (only the pairs the batches
 * use, built on first use; <= 32K rows per shard) -- within the context's
 * budget, else the rank-plane slab kernels
 * whenever the matrix has <= 8192 columns (packed 16-bit rank pairs when a
 * 32-row slab fits in shared memory, else 32-bit plane words), otherwise the
 * value kernel.  TABLE, VALUE, PLANE (slab kernels, no index) and PLANE_U32
 * (32-bit plane words only) force one; a forced path that cannot serve the
 * matrix fails with EBIC_ERR_INVALID_ARGUMENT (or EBIC_ERR_CUDA if the index
 * does not fit in memory).  All are bit-exact; the knob exists for
 * cross-checking and benchmarking. */
#define EBIC_PATH_AUTO 0
#define EBIC_PATH_VALUE 1
#define EBIC_PATH_PLANE 2
#define EBIC_PATH_PLANE_U32 3
#define EBIC_PATH_TABLE 4
#define EBIC_PATH_LAZY 5
int ebic_ctx_set_path(ebic_ctx* ctx, int path);

/* Which index served the last counting launch and what it holds.  *mode: 0
 * none (slab / value kernels), 1 the full pair-trend index, 2 the lazy index
 * (pair vectors built by the count kernel the first time a candidate needs
 * them, kept in a pool for later batches; ebic_lazy.cuh).  full_bytes: the
 * built full index (0 if none); lazy_slots_used / lazy_slots_cap: pair
 * vectors in the pool as last reported by the device / its capacity;
 * lazy_bytes: pool + pair map; lazy_built: vectors built lazily over the
 * matrix's lifetime (the ski-rental count); lazy_resets: times a full pool was
 * started over.  Any out pointer may be NULL. */
int ebic_matrix_index_stats(ebic_ctx* ctx, int* mode, uint64_t* full_bytes, uint64_t* lazy_slots_used,
                            uint64_t* lazy_slots_cap, uint64_t* lazy_bytes, uint64_t* lazy_built,
                            uint64_t* lazy_resets);

/* Packed-pair layout of the hot kernel: `rows_per_lane_pairs` (1 or 2) 16-bit
 * row pairs per lane and `cands_per_warp` (1, 2 or 4) candidates per warp
 * instruction; (0, 0) = auto ((2,1) for <= 256 columns, (1,2) for <= 1024,
 * (1,4) for <= 2048: the fastest measured on B200).  A forced layout whose
 * slab does not fit in shared memory falls back to the 32-bit-word plane
 * kernel.  Every layout is bit-exact; the knob exists for cross-checking and
 * benchmarking. */
int ebic_ctx_set_pair_layout(ebic_ctx* ctx, int rows_per_lane_pairs, int cands_per_warp);

/* Memory budget of the pair-trend index (bytes; env EBIC_TABLE_BUDGET_MB).
 * Default (bytes = 0): 40% of the device memory free at upload, so one
 * context never takes most of a shared GPU.  An explicit budget replaces the
 * fraction and is capped at the free memory minus a reserve of
 * max(8 GiB, 10%); use it to opt in to very large indexes (a 200k x 2000
 * matrix needs 100 GB).  AUTO uses the index only if it fits the budget. */
int ebic_ctx_set_table_budget(ebic_ctx* ctx, uint64_t bytes);

/* How the lazy index builds a batch's missing pair vectors (short vectors,
 * float32 store; env EBIC_LAZY_BUILD).  0 auto: a cold batch -- nothing
 * observed in the pool yet, or >= 1024 slots claimed between the two latest
 * fill samples, and >= 256 candidates -- runs claim, a slab build pass
 * (lazy_slab_build_kernel: 32-row slices of every column staged once per CTA)
 * and publish ahead of the count kernel; any other batch builds inside the
 * count kernel.  1: always inside the count kernel.  2: always the build pass
 * first (when the slices fit in shared memory).  Bit-exact either way. */
#define EBIC_LAZY_BUILD_AUTO 0
#define EBIC_LAZY_BUILD_INLINE 1
#define EBIC_LAZY_BUILD_FIRST 2
int ebic_ctx_set_lazy_build(ebic_ctx* ctx, int mode);
/* Bytes the pair-trend index of the resident matrix needs (0 if the matrix is
 * too wide for the rank plane) and whether it is built. */
int ebic_matrix_index_info(ebic_ctx* ctx, uint64_t* bytes_needed, int* in_use);

/* One-time costs of the last (matrix, approx) preparation, in milliseconds:
 * the index allocation (host clock; 0 when a kept allocation was reused), the
 * rank-plane build and the pair-trend index build (CUDA events on the
 * context's stream).  0 for a step that was not run.  Waits for the builds. */
int ebic_matrix_build_info(ebic_ctx* ctx, double* alloc_ms, double* plane_ms, double* index_ms);

/* Build (or reuse) the full pair-trend index of the resident matrix for
 * `approx` now (if it fits the budget; else the rank plane the slab kernels
 * use), instead of choosing an index on the first evaluation with that approx.
 * Both are per-(matrix, approx): a GA run uses one approx for all
 * generations. */
int ebic_matrix_prepare(ebic_ctx* ctx, double approx);

/* ---- row-sharded step: count reduction over peer memory -----------------
 * Row sharding (rank g holds rows [g*R/G, (g+1)*R/G)) needs the G partial
 * counts of every candidate summed.  Instead of an NCCL all_reduce, each rank
 * owns an exchange window in its HBM that every peer maps (CUDA IPC over
 * NVLink / NVSwitch); one kernel pushes this rank's partial counts into every
 * rank's window, signals, waits for all ranks and sums (ebic_xchg.cuh).
 * Sequence per rank: ebic_xchg_create -> exchange the handles (e.g.
 * torch.distributed all_gather_object) -> ebic_xchg_open -> every step
 * ebic_eval_counts_rows_sum (all ranks, same order).  ebic_xchg_open_local
 * maps windows of contexts in the SAME process instead (device pointers from
 * ebic_xchg_window).  A rank that never arrives makes the kernel give up after
 * EBIC_XCHG_TIMEOUT_MS; the next ebic_ctx_sync reports it.  Ranks sharing one GPU (tests) must
 * build their index first (ebic_matrix_prepare): a device allocation inside a
 * step can wait for the device to go idle, i.e. for a peer's spinning kernel. */
#define EBIC_IPC_HANDLE_BYTES 64
#define EBIC_XCHG_MAX_RANKS 16
int ebic_xchg_create(ebic_ctx* ctx, int world, int rank, uint64_t max_cand, void* handle_out);
int ebic_xchg_open(ebic_ctx* ctx, const void* handles /* world x EBIC_IPC_HANDLE_BYTES, rank order */);
int ebic_xchg_open_local(ebic_ctx* ctx, void* const* windows /* world device pointers, rank order */);
int ebic_xchg_window(ebic_ctx* ctx, void** window_out);
int ebic_xchg_destroy(ebic_ctx* ctx);
/* Device pointers, asynchronous on `stream`: counts of this rank's row shard,
 * summed over all ranks, land in d_counts on every rank (ordered on `stream`).
 * Every window must have been created with the same world and max_cand
 * (checked when the windows are opened).  If this rank's count fails, the
 * exchange still runs -- it pushes zeros and poisons every rank's window --
 * so no rank falls an epoch behind; every rank's counts of that step and all
 * later ones are then 0xFFFFFFFF and ebic_ctx_sync reports the failure.  A
 * rank that does not arrive within EBIC_XCHG_TIMEOUT_MS (default 10000)
 * makes the waiting ranks write 0xFFFFFFFF and report a timeout. */
int ebic_eval_counts_rows_sum(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets,
                              uint64_t n_cand, double approx, int negative_trends, uint32_t* d_counts,
                              void* stream);
/* Pipelined variant (overlap step k's exchange with step
 * k+1's count).  The count runs on `stream`; the exchange runs on the
 * context's own exchange stream as soon as the count is done, so the next
 * call's count kernel does not wait for it.  d_counts is complete only once a
 * stream has passed ebic_xchg_fence (or after ebic_ctx_sync); d_cols and
 * d_offsets may be reused as soon as `stream` passes the call. */
int ebic_eval_counts_rows_sum_async(ebic_ctx* ctx, const uint32_t* d_cols, const uint32_t* d_offsets,
                                    uint64_t n_cand, double approx, int negative_trends, uint32_t* d_counts,
                                    void* stream);
/* Make `stream` (NULL = the context's stream) wait for every exchange issued
 * so far by this context. */
int ebic_xchg_fence(ebic_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* EBIC_H_ */
