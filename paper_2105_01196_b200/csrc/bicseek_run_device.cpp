// bicseek_run_device.cpp -- device-aware evolution driver.
//
// bicseek_device::run(m, p) returns exactly what bicseek::run(m, p) returns
// (evolution.cpp:305-333): same biclusters, same generation count, same
// termination reason.  Three changes are made to the CALLER side of the hot path,
// none of which changes a random draw or an archive decision:
//
//  1. One matrix upload per run.  The matrix is const for the whole run
//     (evolution.cpp:305), so it is uploaded and its rank plane built once, with
//     no per-call identity check.
//  2. Evaluation overlaps breeding.  Offspring are bred in the reference order
//     (evolution.cpp:262-289, reference mutate/crossover/tournament_select/
//     random_chromosome/chromosome_hash, same Rng).  Evaluation consumes no
//     randomness, so every K offspring are handed to the pinned-memory marshaller
//     (ebic_eval_submit).  The GPU counts chunk k while chunk k+1 is bred.
//  3. The archive's overlap filter runs on device counts.  TopRankList::insert
//     (evolution.cpp:76-105) needs a candidate's rows only through
//     induced_jaccard (:44-51): |rows|, and |rows n entry.rows| for each entry.
//     When the next insert needs them, one ebic_support_overlap_batch over
//     [the entries, that candidate and the following offspring that could place
//     under the current archive] returns the sizes and pairwise intersections
//     from row bitmasks that never leave the device; only the emitted
//     biclusters' row lists are fetched, once, at the end.  Rows are a pure
//     function of the candidate, so speculation is exact, and the Jaccard
//     arithmetic on those integers is the reference's.  (EBIC_ARCHIVE_ROWS=1
//     fetches row lists instead, with ebic_support_rows_batch.)
//
// The archive acceptance rule, the operator draw, the breeding loop and the
// small helpers the reference keeps in an anonymous namespace are re-expressed
// below (file:line cited; arithmetic and draw order identical).  Every other
// piece is the reference's own function, linked unchanged.
#include <algorithm>
#include <chrono>
#include <numeric>
#include <tuple>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "bicseek/evolution.hpp"
#include "ebic.h"

namespace bicseek_device {

using namespace bicseek;

namespace {

// Breeding retries before a random chromosome is drawn instead (evolution.cpp:12).
constexpr int kBreedAttempts = 3;

void check(int status, const char* what) {
  if (status != EBIC_OK)
    throw std::runtime_error(std::string("bicseek device run: ") + what + ": " + ebic_last_error());
}

// Weighted operator draw (the rule of evolution.cpp:25-34).  The arithmetic --
// a left-to-right sum, one multiply, sequential subtraction -- is kept exactly,
// because the draw must reproduce the reference bit for bit.
OperatorKind draw_operator(const std::array<double, 5>& w, Rng& rng) {
  const double sum = std::accumulate(w.begin(), w.end(), 0.0);
  double left = rng.uniform_real() * sum;
  std::size_t op = 0;
  while (op + 1 < w.size() && !(left < w[op])) left -= w[op++];
  return static_cast<OperatorKind>(op);
}

// Archive order (evolution.cpp:38-42): higher score first, then fewer columns,
// then the lexicographically smaller column sequence.
bool archive_before(const RankedIndividual& x, const RankedIndividual& y) {
  return std::forward_as_tuple(-x.score, x.chromosome.columns.size(), x.chromosome.columns) <
         std::forward_as_tuple(-y.score, y.chromosome.columns.size(), y.chromosome.columns);
}

// Cell Jaccard of an archive entry and a candidate bicluster (evolution.cpp:44-51):
// cells are products, so the intersection is |rows n| * |cols n|.  The row
// intersection and the two row-set sizes come in as counts (from the row lists,
// or from the device's row bitmasks); the arithmetic is the reference's.
double cell_overlap(std::size_t shared_rows, std::size_t rows_e, const std::vector<std::size_t>& cols_e,
                    std::size_t rows_c, const std::vector<std::size_t>& sorted_cols) {
  const std::size_t shared = shared_rows * sorted_intersection_size(cols_e, sorted_cols);
  const std::size_t cells_e = rows_e * cols_e.size(), cells_c = rows_c * sorted_cols.size();
  return static_cast<double>(shared) / static_cast<double>(cells_e + cells_c - shared);
}

// Per-column occurrence counts over a population (evolution.cpp:215-221).
std::vector<std::size_t> tally_columns(const std::vector<RankedIndividual>& pop, std::size_t num_cols) {
  std::vector<std::size_t> tally(num_cols, 0);
  for (const RankedIndividual& ind : pop)
    for (std::size_t c : ind.chromosome.columns) tally[c] += 1;
  return tally;
}

// One device context per run: the matrix, the plane and the marshaller ring.
// Contexts are kept per thread and device across runs (stream, pinned staging
// slots and scratch survive; the matrix does not): creating one costs
// milliseconds to, on some boxes, a large fraction of a second.
struct ThreadContexts {
  std::vector<std::pair<int, ebic_ctx*>> ctx;
  ebic_ctx* get(int device) {
    for (auto& c : ctx)
      if (c.first == device) return c.second;
    ebic_ctx* x = nullptr;
    check(ebic_ctx_create(device, &x), "context");
    ctx.emplace_back(device, x);
    return x;
  }
  ~ThreadContexts() {
    for (auto& c : ctx) ebic_ctx_destroy(c.second);
  }
};
ebic_ctx* thread_context(int device) {
  thread_local ThreadContexts pool;
  return pool.get(device);
}

struct Device {
  ebic_ctx* ctx = nullptr;
  double approx = 0.0;
  int neg = 0;
  uint64_t launches0 = 0;

  Device(const ExpressionMatrix& m, const TrendParams& tp, int device) {
    ctx = thread_context(device);
    check(ebic_matrix_upload_f64(ctx, m.values().data(), m.rows(), m.cols(), 0, EBIC_STORE_AUTO, nullptr),
          "matrix upload");
    approx = tp.approx;
    neg = tp.negative_trends ? 1 : 0;
    check(ebic_matrix_prepare(ctx, approx), "rank plane");
  }
  ~Device() {
    // the context, and the matrix with its index, stay for this thread's next
    // run (whose upload replaces the matrix and reuses the index allocation)
    if (ctx) ebic_ctx_sync(ctx);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
};

// Offspring evaluation in chunks through the marshaller.
class ChunkedEval {
 public:
  ChunkedEval(Device& dev, std::size_t chunk) : dev_(dev), chunk_(std::max<std::size_t>(chunk, 1)) {}

  // call after each new offspring; submits a chunk when one is complete
  void add(const std::vector<Chromosome>& pop) {
    if (pop.size() - submitted_ >= chunk_) submit(pop, submitted_ + chunk_);
  }
  // submit the remainder, wait for everything; counts[i] for pop[i]
  std::vector<std::size_t> finish(const std::vector<Chromosome>& pop) {
    if (submitted_ < pop.size()) submit(pop, pop.size());
    std::vector<std::size_t> counts(pop.size());
    for (std::size_t b = 0; b < tickets_.size(); ++b) {
      check(ebic_eval_wait(dev_.ctx, tickets_[b]), "evaluate_population");
      const auto& out = outs_[b];
      for (std::size_t i = 0; i < out.size(); ++i) counts[begins_[b] + i] = out[i];
    }
    return counts;
  }

 private:
  void submit(const std::vector<Chromosome>& pop, std::size_t end) {
    std::vector<uint32_t> cols, offs{0};
    for (std::size_t i = submitted_; i < end; ++i) {
      for (std::size_t c : pop[i].columns) cols.push_back(static_cast<uint32_t>(c));
      offs.push_back(static_cast<uint32_t>(cols.size()));
    }
    outs_.emplace_back(end - submitted_);
    begins_.push_back(submitted_);
    uint64_t t = 0;
    check(ebic_eval_submit(dev_.ctx, cols.data(), offs.data(), end - submitted_, dev_.approx, dev_.neg,
                           outs_.back().data(), &t),
          "evaluate_population");
    tickets_.push_back(t);
    submitted_ = end;
  }

  Device& dev_;
  std::size_t chunk_;
  std::size_t submitted_ = 0;
  std::vector<uint64_t> tickets_;
  std::vector<std::size_t> begins_;
  std::vector<std::vector<uint32_t>> outs_;  // stable storage: written when the ticket is waited
};

// An archive entry: the reference's TopRankEntry plus its row-set size and an
// id for the overlap counts.  In overlap mode `rows` stays empty until the run
// ends (only the emitted entries' rows are fetched).
struct Entry : TopRankEntry {
  std::size_t n_rows = 0;
  std::uint64_t uid = 0;
};

// What the acceptance rule needs to know about a candidate's rows.
struct CandidateRows {
  std::size_t n_rows = 0;
  std::uint64_t uid = 0;
  std::vector<std::size_t> rows;                      // row-list mode
  std::unordered_map<std::uint64_t, std::size_t> shared;  // overlap mode: entry uid -> |rows n|
  bool lists = false;
  std::size_t shared_with(const Entry& e) const {
    return lists ? sorted_intersection_size(e.rows, rows) : shared.at(e.uid);
  }
};

// The top-rank archive (evolution.hpp:78-98): the acceptance rule of
// TopRankList::insert (evolution.cpp:76-105), fed with precomputed row data.
class Archive {
 public:
  Archive(std::size_t capacity, double overlap) : capacity_(capacity), overlap_(overlap) {}

  const std::vector<Entry>& entries() const { return entries_; }
  std::vector<Entry>& entries() { return entries_; }
  bool full() const { return entries_.size() >= capacity_; }
  double min_score() const { return entries_.empty() ? 0.0 : entries_.back().ind.score; }

  // can the candidate enter at all -- i.e. does the reference compute its rows
  // (evolution.cpp:78-79)?
  bool could_place(const RankedIndividual& ind) const {
    return ind.score > 0.0 && !(full() && ind.score <= min_score());
  }

  bool insert(const RankedIndividual& ind, const CandidateRows& cr) {
    if (!could_place(ind)) return false;
    Entry fresh;
    fresh.ind = ind;
    if (cr.lists) fresh.rows = cr.rows;
    fresh.n_rows = cr.n_rows;
    fresh.uid = cr.uid;
    fresh.cols = ind.chromosome.columns;
    std::sort(fresh.cols.begin(), fresh.cols.end());
    // entries overlapping the candidate too much are displaced -- unless one of
    // them scores at least as high, in which case the candidate is rejected
    std::vector<char> displaced(entries_.size(), 0);
    for (std::size_t i = 0; i < entries_.size(); ++i) {
      const Entry& e = entries_[i];
      if (cell_overlap(cr.shared_with(e), e.n_rows, e.cols, cr.n_rows, fresh.cols) < overlap_) continue;
      if (e.ind.score >= ind.score) return false;
      displaced[i] = 1;
    }
    std::size_t keep = 0;
    for (std::size_t i = 0; i < entries_.size(); ++i) {
      if (displaced[i]) continue;
      if (keep != i) entries_[keep] = std::move(entries_[i]);  // (no self-move)
      ++keep;
    }
    entries_.resize(keep);
    // entries are kept in archive order: the candidate goes before the first
    // entry it outranks
    const auto at = std::upper_bound(entries_.begin(), entries_.end(), fresh, [](const Entry& a, const Entry& b) {
      return archive_before(a.ind, b.ind);
    });
    entries_.insert(at, std::move(fresh));
    if (entries_.size() > capacity_) entries_.resize(capacity_);
    // placed iff it survived the truncation
    return std::any_of(entries_.begin(), entries_.end(), [&](const Entry& e) {
      return e.ind.score == ind.score && e.ind.chromosome.columns == ind.chromosome.columns;
    });
  }

 private:
  std::vector<Entry> entries_;
  std::size_t capacity_;
  double overlap_;
};

void append_candidate(const Chromosome& c, std::vector<uint32_t>& cols, std::vector<uint32_t>& offs) {
  for (std::size_t x : c.columns) cols.push_back(static_cast<uint32_t>(x));
  offs.push_back(static_cast<uint32_t>(cols.size()));
}

// Serial archive inserts in offspring order, with speculative batches.  When
// the next insert needs row data, the driver computes it for that candidate
// and up to batch-1 following offspring that could place under the current
// archive -- rows are a pure function of the candidate, so speculation is
// exact.  Two modes:
//  * overlap (default): one ebic_support_overlap_batch over [current entries,
//    picked candidates] returns the row-set sizes and pairwise intersection
//    counts; no row list crosses the bus.  A cached candidate is reused only
//    if its counts cover every entry now in the archive.
//  * lists (EBIC_ARCHIVE_ROWS=1, or an archive too large for one overlap
//    batch): ebic_support_rows_batch row lists, intersected on the host.
class RowBatcher {
 public:
  RowBatcher(Device& dev, std::size_t batch, bool lists) : dev_(dev), batch_(std::max<std::size_t>(batch, 1)),
                                                           lists_(lists) {}

  bool lists() const { return lists_; }

  const CandidateRows& rows_for(std::size_t i, const std::vector<RankedIndividual>& inds, const Archive& arch) {
    auto it = cache_.find(i);
    if (it != cache_.end() && covers(it->second, arch)) return it->second;
    // i itself plus up to batch-1 later candidates that could place right now
    std::vector<std::size_t> pick{i};
    for (std::size_t k = i + 1; k < inds.size() && pick.size() < batch_; ++k)
      if (arch.could_place(inds[k]) && cache_.find(k) == cache_.end()) pick.push_back(k);
    if (lists_) fetch_lists(pick, inds);
    else fetch_overlaps(pick, inds, arch);
    return cache_.at(i);
  }

  void clear() { cache_.clear(); }

  // row lists of the given chromosomes (the emitted entries at the end of a run)
  std::vector<std::vector<std::size_t>> lists_of(const std::vector<const Chromosome*>& cs) {
    std::vector<uint32_t> cols, offs{0};
    for (const Chromosome* c : cs) append_candidate(*c, cols, offs);
    std::vector<uint64_t> row_offs(cs.size() + 1);
    std::vector<uint32_t> rows(cap_);
    int st = ebic_support_rows_batch(dev_.ctx, cols.data(), offs.data(), cs.size(), dev_.approx, dev_.neg,
                                     rows.data(), rows.size(), row_offs.data());
    if (st == EBIC_ERR_CAPACITY) {
      cap_ = row_offs.back() + row_offs.back() / 2;
      rows.assign(cap_, 0);
      st = ebic_support_rows_batch(dev_.ctx, cols.data(), offs.data(), cs.size(), dev_.approx, dev_.neg,
                                   rows.data(), rows.size(), row_offs.data());
    }
    check(st, "supporting_rows");
    std::vector<std::vector<std::size_t>> out(cs.size());
    for (std::size_t b = 0; b < cs.size(); ++b)
      out[b].assign(rows.begin() + static_cast<std::ptrdiff_t>(row_offs[b]),
                    rows.begin() + static_cast<std::ptrdiff_t>(row_offs[b + 1]));
    return out;
  }

 private:
  bool covers(const CandidateRows& cr, const Archive& arch) const {
    if (cr.lists) return true;
    for (const Entry& e : arch.entries())
      if (!cr.shared.count(e.uid)) return false;
    return true;
  }

  void fetch_lists(const std::vector<std::size_t>& pick, const std::vector<RankedIndividual>& inds) {
    std::vector<const Chromosome*> cs;
    for (std::size_t k : pick) cs.push_back(&inds[k].chromosome);
    auto rows = lists_of(cs);
    for (std::size_t b = 0; b < pick.size(); ++b) {
      CandidateRows& cr = cache_[pick[b]];
      cr.lists = true;
      cr.rows = std::move(rows[b]);
      cr.n_rows = cr.rows.size();
      cr.uid = next_uid_++;
    }
  }

  void fetch_overlaps(const std::vector<std::size_t>& pick, const std::vector<RankedIndividual>& inds,
                      const Archive& arch) {
    const auto& ents = arch.entries();
    std::vector<uint32_t> cols, offs{0};
    std::vector<std::uint64_t> uids;
    for (const Entry& e : ents) {
      append_candidate(e.ind.chromosome, cols, offs);
      uids.push_back(e.uid);
    }
    for (std::size_t k : pick) {
      append_candidate(inds[k].chromosome, cols, offs);
      uids.push_back(next_uid_++);
    }
    const std::size_t n = uids.size();
    std::vector<uint64_t> sizes(n), inter(n * n);
    check(ebic_support_overlap_batch(dev_.ctx, cols.data(), offs.data(), n, dev_.approx, dev_.neg, sizes.data(),
                                     inter.data()),
          "supporting_rows overlaps");
    for (std::size_t b = 0; b < pick.size(); ++b) {
      const std::size_t q = ents.size() + b;
      CandidateRows& cr = cache_[pick[b]];
      cr = CandidateRows{};
      cr.n_rows = sizes[q];
      cr.uid = uids[q];
      for (std::size_t j = 0; j < n; ++j)
        if (j != q) cr.shared[uids[j]] = inter[q * n + j];
    }
  }

  Device& dev_;
  std::size_t batch_;
  bool lists_;
  std::size_t cap_ = 1 << 16;
  std::uint64_t next_uid_ = 1;
  std::unordered_map<std::size_t, CandidateRows> cache_;
};

struct State {
  std::size_t generation = 0;
  std::vector<RankedIndividual> population;
  Archive top_rank;
  TabuList tabu;
  std::vector<std::size_t> column_usage;
  Rng rng;
  State(std::size_t capacity, double overlap, std::uint64_t seed) : top_rank(capacity, overlap), rng(seed) {}
};

// make_ranked (evolution.cpp:223-229) for a whole batch, then the serial
// inserts of init_state / step_generation; returns "improved".
bool rank_and_insert(std::vector<Chromosome>&& pop, const std::vector<std::size_t>& counts, State& st,
                     const EvolutionParams& p, RowBatcher& rb, std::vector<RankedIndividual>& out) {
  std::vector<RankedIndividual> inds(pop.size());
  for (std::size_t i = 0; i < pop.size(); ++i) {
    inds[i].score = fitness(counts[i], pop[i].size(), p.trend);
    inds[i].support_count = counts[i];
    inds[i].chromosome = std::move(pop[i]);
  }
  rb.clear();
  bool improved = false;
  for (std::size_t i = 0; i < inds.size(); ++i) {
    if (st.top_rank.could_place(inds[i]))
      improved = st.top_rank.insert(inds[i], rb.rows_for(i, inds, st.top_rank)) || improved;
  }
  for (auto& ind : inds) out.push_back(std::move(ind));
  return improved;
}

// One offspring, drawn exactly as in step_generation (evolution.cpp:262-289):
// up to kBreedAttempts tournament + operator draws, each rejected if its hash
// is already tabu (which counts a tabu hit); then a fresh random chromosome.
Chromosome breed_child(State& st, const EvolutionParams& p, std::size_t num_cols) {
  for (int tries = 0; tries < kBreedAttempts; ++tries) {
    const RankedIndividual& first = tournament_select(st.population, st.column_usage, p, st.rng);
    const OperatorKind op = draw_operator(p.operator_weights, st.rng);
    Chromosome child = op == OperatorKind::crossover
                           ? crossover(first.chromosome,
                                       tournament_select(st.population, st.column_usage, p, st.rng).chromosome,
                                       st.rng)
                           : mutate(first.chromosome, op, num_cols, st.rng);
    const std::uint64_t h = chromosome_hash(child);
    if (!st.tabu.contains(h)) {
      st.tabu.insert(h);
      return child;
    }
    st.tabu.hit_count += 1;
  }
  Chromosome child = random_chromosome(p, num_cols, st.rng);
  st.tabu.insert(chromosome_hash(child));
  return child;
}

}  // namespace

// Create this thread's context for `device` ahead of the first run (a
// harness can keep the start-up out of run()'s timer, as it does for the
// drop-in TU with one tiny evaluation).
void warm(int device = 0) { (void)thread_context(device); }

// evolution.cpp:305-333 with the device evaluator on the caller side.
RunResult run(const ExpressionMatrix& m, const EvolutionParams& p, int device = 0) {
  p.validate();
  if (m.rows() == 0 || m.cols() < 2) throw std::invalid_argument("run: matrix too small");
  const auto t0 = std::chrono::steady_clock::now();

  // EBIC_DRIVER_TRACE=1: phase times on stderr (setup, per-generation breed+eval / archive)
  const char* trace_env = std::getenv("EBIC_DRIVER_TRACE");
  const bool trace = trace_env && std::atoi(trace_env);
  auto since = [](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  Device dev(m, p.trend, device);
  if (trace) std::fprintf(stderr, "[driver] device setup %.2f ms\n", since(t0));
  const std::size_t chunk = std::max<std::size_t>(256, p.population_size / 4);
  const char* lists_env = std::getenv("EBIC_ARCHIVE_ROWS");
  const bool lists = (lists_env && std::atoi(lists_env)) || p.top_rank_capacity() + 64 > EBIC_OVERLAP_MAX;
  RowBatcher rows(dev, 64, lists);

  // init_state (evolution.cpp:233-246)
  State st(p.top_rank_capacity(), p.overlap_threshold, p.seed);
  {
    std::vector<Chromosome> pop = init_population(p, m.cols(), st.rng);
    ChunkedEval ev(dev, chunk);
    ev.add(pop);
    const std::vector<std::size_t> counts = ev.finish(pop);
    for (const Chromosome& c : pop) st.tabu.insert(chromosome_hash(c));
    st.population.reserve(pop.size());
    rank_and_insert(std::move(pop), counts, st, p, rows, st.population);
    st.column_usage = tally_columns(st.population, m.cols());
  }

  if (trace) std::fprintf(stderr, "[driver] init_state done at %.2f ms\n", since(t0));
  std::string reason = "budget";
  while (st.generation < p.max_iterations) {
    if (st.tabu.hit_count >= p.effective_tabu_threshold()) {
      reason = "converged";
      break;
    }
    // step_generation (evolution.cpp:248-303)
    const auto t_gen = std::chrono::steady_clock::now();
    const std::size_t num_cols = m.cols();
    std::vector<RankedIndividual> next;
    next.reserve(p.population_size);
    const auto& ranked = st.top_rank.entries();
    const std::size_t n_elite = std::min(p.elite_count, ranked.size());
    for (std::size_t i = 0; i < n_elite; ++i) next.push_back(ranked[i].ind);

    std::vector<Chromosome> offspring;
    offspring.reserve(p.population_size - next.size());
    ChunkedEval ev(dev, chunk);
    while (next.size() + offspring.size() < p.population_size) {
      offspring.push_back(breed_child(st, p, num_cols));
      ev.add(offspring);  // overlap: the GPU counts this chunk while the next is bred
    }
    const std::vector<std::size_t> counts = ev.finish(offspring);
    const auto t_ins = std::chrono::steady_clock::now();
    const bool improved = rank_and_insert(std::move(offspring), counts, st, p, rows, next);
    if (trace)
      std::fprintf(stderr, "[driver] gen %zu: breed+eval %.2f ms, archive %.2f ms\n", st.generation,
                   std::chrono::duration<double, std::milli>(t_ins - t_gen).count(), since(t_ins));
    if (improved) st.tabu.hit_count = 0;
    st.population = std::move(next);
    st.column_usage = tally_columns(st.population, num_cols);
    ++st.generation;
  }

  RunResult result;
  std::vector<Entry*> emit;
  for (auto& entry : st.top_rank.entries()) {
    if (emit.size() >= p.num_biclusters) break;
    if (entry.ind.support_count < p.trend.min_rows) continue;
    emit.push_back(&entry);
  }
  if (!rows.lists() && !emit.empty()) {  // overlap mode: the emitted entries' rows, in one batch
    std::vector<const Chromosome*> cs;
    for (const Entry* e : emit) cs.push_back(&e->ind.chromosome);
    auto lists_out = rows.lists_of(cs);
    for (std::size_t b = 0; b < emit.size(); ++b) emit[b]->rows = std::move(lists_out[b]);
  }
  for (const Entry* e : emit) result.biclusters.biclusters.emplace_back(e->rows, e->cols);
  result.report.generations = st.generation;
  result.report.termination = reason;
  result.report.wall_time_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

}  // namespace bicseek_device
