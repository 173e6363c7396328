// bicseek_trend_device.cpp -- drop-in replacement TU for the reference's
// proj/src/trend.cpp.  It implements every symbol declared in the UNCHANGED
// reference header proj/include/bicseek/trend.hpp (trend.hpp:13-50) on top of
// the C ABI in include/ebic.h, so the reference's evolution engine
// (evolution.cpp, unchanged) and its tests (test_trend.cpp, unchanged) run on
// the B200 evaluator by linking this file instead of trend.cpp.
//
//   TrendParams::validate  trend.hpp:24   / trend.cpp:8-13   host (restated)
//   row_supports           trend.hpp:30   / trend.cpp:41-46  device (ebic_row_supports)
//   supporting_rows        trend.hpp:34   / trend.cpp:48-54  device (ebic_support_rows)
//   evaluate_population    trend.hpp:43   / trend.cpp:56-72  device (ebic_eval_counts)
//   fitness                trend.hpp:50   / trend.cpp:74-79  host, exact (ebic_fitness)
//
// There is no CPU fallback: without a usable CUDA device every evaluating
// call throws std::runtime_error.
//
// Device matrix cache: the reference passes the matrix by const& on every
// call (trend.hpp:43-45).  The first call uploads it (float32 store when every
// value is float32-representable, else float64 -- bit-exact either way) and
// keeps a host shadow copy.  A later call reuses the resident copy when the
// pointer and shape match AND the values the call depends on are identical to
// the shadow: a call reads only the columns of its chromosomes, and every
// device structure derived from the matrix (rank plane, pair-trend index,
// lazy pair vectors) answers a pair test from the two columns' own values, so
// unchanged referenced columns give the reference's result even if some other
// column was mutated in place.  So:
//   row_supports       -- compares the candidate's L values of that row;
//   supporting_rows    -- compares the candidate's columns over all rows (a
//                         strided compare of L x R values, not the matrix);
//   evaluate_population-- compares the columns the population references, or
//                         the whole matrix when it references most of them.
// Any difference re-uploads the whole matrix and refreshes the shadow.  The
// compares run on a persistent pool of host threads (HostPool) with an early
// exit.  EBIC_SHIM_TRUST_POINTER=1 skips them for callers that guarantee the
// matrix is immutable; EBIC_SHIM_THREADS=<n> sizes the pool (default: all
// hardware threads).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include "bicseek/trend.hpp"
#include "ebic.h"

namespace bicseek {

void TrendParams::validate() const {
  // same rules and messages as trend.cpp:8-13
  if (!(approx >= 0.0 && approx < 1.0))
    throw std::invalid_argument("TrendParams: approx must be in [0, 1)");
  if (min_rows < 2) throw std::invalid_argument("TrendParams: min_rows must be >= 2");
  if (col_cap < 2) throw std::invalid_argument("TrendParams: col_cap must be >= 2");
}

namespace {

// Persistent host thread pool for chunked byte-range work (compare / copy of
// the matrix shadow).  One job at a time; the calling thread takes chunks too.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  // fn(begin, end) over [0, n) in chunks of `chunk`; stops handing out chunks
  // once `stop` is set (by fn)
  void run(std::size_t n, std::size_t chunk, const std::function<void(std::size_t, std::size_t)>& fn,
           const std::atomic<bool>* stop = nullptr) {
    std::lock_guard<std::mutex> job_lock(job_mu_);
    const std::size_t n_chunks = (n + chunk - 1) / chunk;
    if (workers_.empty() || n_chunks <= 1) {
      for (std::size_t c = 0; c < n_chunks && !(stop && stop->load()); ++c) fn(c * chunk, std::min(n, (c + 1) * chunk));
      return;
    }
    {
      std::lock_guard<std::mutex> l(mu_);
      fn_ = &fn;
      stop_ = stop;
      n_ = n;
      chunk_ = chunk;
      next_.store(0);
      active_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    unsigned n = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("EBIC_SHIM_THREADS")) n = (unsigned)std::max(1, std::atoi(e));
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void drain() {
    const std::size_t n_chunks = (n_ + chunk_ - 1) / chunk_;
    for (;;) {
      if (stop_ && stop_->load()) return;
      const std::size_t c = next_.fetch_add(1);
      if (c >= n_chunks) return;
      (*fn_)(c * chunk_, std::min(n_, (c + 1) * chunk_));
    }
  }
  void loop() {
    std::uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
      }
      drain();
      std::lock_guard<std::mutex> l(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(std::size_t, std::size_t)>* fn_ = nullptr;
  const std::atomic<bool>* stop_ = nullptr;
  std::size_t n_ = 0, chunk_ = 1;
  std::atomic<std::size_t> next_{0};
  std::size_t active_ = 0;
  std::uint64_t gen_ = 0;
  bool quit_ = false;
};

constexpr std::size_t kChunkBytes = 4u << 20;

bool same_bytes(const void* a, const void* b, std::size_t bytes) {
  std::atomic<bool> differs{false};
  const auto* pa = static_cast<const unsigned char*>(a);
  const auto* pb = static_cast<const unsigned char*>(b);
  HostPool::get().run(
      bytes, kChunkBytes,
      [&](std::size_t lo, std::size_t hi) {
        if (std::memcmp(pa + lo, pb + lo, hi - lo) != 0) differs.store(true);
      },
      &differs);
  return !differs.load();
}

void copy_bytes(void* dst, const void* src, std::size_t bytes) {
  auto* d = static_cast<unsigned char*>(dst);
  const auto* s = static_cast<const unsigned char*>(src);
  HostPool::get().run(bytes, kChunkBytes, [&](std::size_t lo, std::size_t hi) { std::memcpy(d + lo, s + lo, hi - lo); });
}

// Host shadow of the cached matrix.  Anonymous mmap (transparent huge pages
// advised), filled by the pool: the pages are first touched by the parallel
// copy.  A std::vector would zero-fill them on one thread first: 693 ms for
// 1.6 GB against 114 ms (profiles/r2_host_copy.txt).
class Shadow {
 public:
  ~Shadow() { release(); }
  std::size_t size() const { return n_; }
  const double* data() const { return p_; }
  const double& operator[](std::size_t i) const { return p_[i]; }
  void assign(const double* src, std::size_t n) {
    if (n * sizeof(double) > cap_) {
      release();
      void* m = mmap(nullptr, n * sizeof(double), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (m == MAP_FAILED) throw std::bad_alloc();
      madvise(m, n * sizeof(double), MADV_HUGEPAGE);
      p_ = static_cast<double*>(m);
      cap_ = n * sizeof(double);
    }
    n_ = n;
    copy_bytes(p_, src, n * sizeof(double));
  }

 private:
  void release() {
    if (p_) munmap(p_, cap_);
    p_ = nullptr;
    n_ = cap_ = 0;
  }
  double* p_ = nullptr;
  std::size_t n_ = 0, cap_ = 0;
};

struct DeviceState {
  ebic_ctx* ctx = nullptr;
  const double* key = nullptr;
  std::size_t rows = 0, cols = 0;
  Shadow shadow;
  ~DeviceState() {
    if (ctx) ebic_ctx_destroy(ctx);
  }
};

thread_local DeviceState g_dev;

void check(int status, const char* what) {
  if (status != EBIC_OK)
    throw std::runtime_error(std::string("bicseek device evaluator: ") + what + ": " +
                             ebic_last_error());
}

bool trust_pointer() {
  const char* e = std::getenv("EBIC_SHIM_TRUST_POINTER");
  return e && e[0] == '1';
}

// Device of a new (per-thread) context.  EBIC_DEVICE=<n> pins every thread to
// GPU n; otherwise threads are spread round-robin over the visible GPUs, so
// independent datasets run concurrently (bench --jobs, bench.cpp:103-121)
// land on different GPUs -- dataset-level multi-GPU.
int pick_device() {
  const char* e = std::getenv("EBIC_DEVICE");
  if (e && *e && std::strcmp(e, "all") != 0) return std::atoi(e);
  int n = 0;
  if (ebic_device_count(&n) != EBIC_OK || n <= 1) return 0;
  static std::atomic<unsigned> next{0};
  return static_cast<int>(next.fetch_add(1) % static_cast<unsigned>(n));
}

// Are the values at `cols` (all rows) identical to the shadow?  Strided
// compare over row blocks on the pool.
bool same_columns(const double* a, const double* b, std::size_t rows, std::size_t n_cols,
                  const std::vector<uint32_t>& cols) {
  std::atomic<bool> differs{false};
  const std::size_t block = std::max<std::size_t>(1, (256u << 10) / std::max<std::size_t>(1, cols.size() * 64));
  HostPool::get().run(
      rows, block,
      [&](std::size_t r0, std::size_t r1) {
        for (std::size_t r = r0; r < r1; ++r) {
          const double* ra = a + r * n_cols;
          const double* rb = b + r * n_cols;
          for (uint32_t c : cols)
            if (std::memcmp(ra + c, rb + c, sizeof(double)) != 0) {
              differs.store(true);
              return;
            }
        }
      },
      &differs);
  return !differs.load();
}

// What a call depends on: every value (nullptr), some columns, or one row's cells.
struct Deps {
  const std::vector<uint32_t>* cols = nullptr;  // distinct columns referenced (nullptr: the whole matrix)
  std::size_t row = SIZE_MAX;                   // row_supports: only this row's cells of `cols`
  int kind = 2;                                 // 1: supporting_rows, 2: evaluate_population (stats)
};

// EBIC_SHIM_STATS=1: per-kind call counts and time spent verifying the
// cached matrix, printed to stderr at exit (diagnostics).
struct ShimStats {
  std::atomic<uint64_t> calls[3] = {}, ns[3] = {}, bind_ns{0}, binds{0};
  bool on = [] {
    const char* e = std::getenv("EBIC_SHIM_STATS");
    return e && e[0] == '1';
  }();
  ~ShimStats() {
    if (!on) return;
    static const char* names[3] = {"row_supports", "supporting_rows", "evaluate_population"};
    for (int k = 0; k < 3; ++k)
      std::fprintf(stderr, "shim %s: %llu calls, %.3f ms verifying the cached matrix\n", names[k],
                   (unsigned long long)calls[k].load(), ns[k].load() / 1e6);
    std::fprintf(stderr, "shim: %llu uploads (+ shadow copies), %.3f ms\n", (unsigned long long)binds.load(),
                 bind_ns.load() / 1e6);
  }
};
ShimStats g_stats;

bool unchanged_impl(const DeviceState& s, const std::vector<double>& v, std::size_t n_cols, const Deps& d);

bool unchanged(const DeviceState& s, const std::vector<double>& v, std::size_t n_cols, const Deps& d) {
  if (!g_stats.on) return unchanged_impl(s, v, n_cols, d);
  const int kind = d.row != SIZE_MAX ? 0 : (d.kind == 1 ? 1 : 2);
  const auto t0 = std::chrono::steady_clock::now();
  const bool r = unchanged_impl(s, v, n_cols, d);
  g_stats.calls[kind]++;
  g_stats.ns[kind] += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                          std::chrono::steady_clock::now() - t0).count();
  return r;
}

bool unchanged_impl(const DeviceState& s, const std::vector<double>& v, std::size_t n_cols, const Deps& d) {
  if (s.shadow.size() != v.size()) return false;
  if (d.cols && d.row != SIZE_MAX) {
    for (uint32_t c : *d.cols)
      if (std::memcmp(&s.shadow[d.row * n_cols + c], &v[d.row * n_cols + c], sizeof(double)) != 0) return false;
    return true;
  }
  // a strided compare touches a cache line per value: cheaper than the whole
  // matrix only for a small fraction of the columns
  if (d.cols && d.cols->size() * 8 < n_cols) return same_columns(s.shadow.data(), v.data(), v.size() / n_cols, n_cols, *d.cols);
  return same_bytes(s.shadow.data(), v.data(), v.size() * sizeof(double));
}

ebic_ctx* bind(const ExpressionMatrix& m, const Deps& deps = Deps{}) {
  DeviceState& s = g_dev;
  if (!s.ctx) check(ebic_ctx_create(pick_device(), &s.ctx), "context");
  const std::vector<double>& v = m.values();
  const bool same = s.key == v.data() && s.rows == m.rows() && s.cols == m.cols() &&
                    (trust_pointer() || unchanged(s, v, m.cols(), deps));
  if (!same) {
    const auto t0 = std::chrono::steady_clock::now();
    s.key = nullptr;
    check(ebic_matrix_upload_f64(s.ctx, v.data(), m.rows(), m.cols(), 0, EBIC_STORE_AUTO, nullptr),
          "matrix upload");
    s.key = v.data();
    s.rows = m.rows();
    s.cols = m.cols();
    if (!trust_pointer()) s.shadow.assign(v.data(), v.size());
    if (g_stats.on) {
      g_stats.binds++;
      g_stats.bind_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                             std::chrono::steady_clock::now() - t0).count();
    }
  }
  return s.ctx;
}

// Distinct columns of one or more chromosomes (indices already range-checked).
std::vector<uint32_t> distinct_columns(const std::vector<uint32_t>& cols, std::size_t n_cols) {
  std::vector<uint32_t> out;
  std::vector<unsigned char> seen(n_cols, 0);
  for (uint32_t c : cols)
    if (!seen[c]) {
      seen[c] = 1;
      out.push_back(c);
    }
  return out;
}

std::vector<uint32_t> to_u32(const std::vector<std::size_t>& cols, std::size_t n_cols) {
  std::vector<uint32_t> out(cols.size());
  for (std::size_t k = 0; k < cols.size(); ++k) {
    if (cols[k] >= n_cols)
      throw std::out_of_range("bicseek device evaluator: column index out of range");
    out[k] = static_cast<uint32_t>(cols[k]);
  }
  return out;
}

}  // namespace

bool row_supports(const ExpressionMatrix& m, std::size_t row, const Chromosome& c,
                  const TrendParams& p) {
  if (row >= m.rows()) throw std::out_of_range("row_supports: row out of range");
  const std::vector<uint32_t> cols = to_u32(c.columns, m.cols());
  Deps deps;
  deps.cols = &cols;
  deps.row = row;
  ebic_ctx* ctx = bind(m, deps);
  int out = 0;
  check(ebic_row_supports(ctx, row, cols.data(), static_cast<uint32_t>(cols.size()), p.approx,
                          p.negative_trends ? 1 : 0, &out),
        "row_supports");
  return out != 0;
}

std::vector<std::size_t> supporting_rows(const ExpressionMatrix& m, const Chromosome& c,
                                         const TrendParams& p) {
  if (m.rows() == 0) return {};
  const std::vector<uint32_t> cols = to_u32(c.columns, m.cols());
  const std::vector<uint32_t> used = distinct_columns(cols, m.cols());
  Deps deps;
  deps.cols = &used;
  deps.kind = 1;
  ebic_ctx* ctx = bind(m, deps);
  std::vector<uint32_t> rows(m.rows());
  uint64_t n = 0;
  check(ebic_support_rows(ctx, cols.data(), static_cast<uint32_t>(cols.size()), p.approx,
                          p.negative_trends ? 1 : 0, rows.data(), rows.size(), &n),
        "supporting_rows");
  return std::vector<std::size_t>(rows.begin(), rows.begin() + static_cast<std::ptrdiff_t>(n));
}

std::vector<std::size_t> evaluate_population(const ExpressionMatrix& m,
                                             const std::vector<Chromosome>& pop,
                                             const TrendParams& p, WorkerPool* /*pool*/) {
  // The WorkerPool is the reference's CPU parallel runtime (trend.cpp:67-70);
  // the device grid replaces it, so it is accepted and ignored.
  std::vector<std::size_t> counts(pop.size(), 0);
  if (pop.empty() || m.rows() == 0) return counts;
  std::vector<uint32_t> cols, offs;
  offs.reserve(pop.size() + 1);
  offs.push_back(0);
  for (const Chromosome& c : pop) {
    for (std::size_t col : c.columns) {
      if (col >= m.cols())
        throw std::out_of_range("evaluate_population: column index out of range");
      cols.push_back(static_cast<uint32_t>(col));
    }
    offs.push_back(static_cast<uint32_t>(cols.size()));
  }
  const std::vector<uint32_t> used = distinct_columns(cols, m.cols());
  Deps deps;
  deps.cols = &used;
  ebic_ctx* ctx = bind(m, deps);
  std::vector<uint32_t> out(pop.size());
  check(ebic_eval_counts(ctx, cols.data(), offs.data(), pop.size(), p.approx,
                         p.negative_trends ? 1 : 0, out.data()),
        "evaluate_population");
  for (std::size_t i = 0; i < out.size(); ++i) counts[i] = out[i];
  return counts;
}

double fitness(std::size_t support_count, std::size_t num_cols, const TrendParams& p) {
  return ebic_fitness(support_count, num_cols, p.min_rows, p.col_cap);
}

}  // namespace bicseek
