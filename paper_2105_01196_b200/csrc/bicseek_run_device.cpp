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
//  3. Archive row sets come in batches.  TopRankList::insert (evolution.cpp:76-105)
//     needs supporting_rows only for candidates that can place.  When the next
//     insert needs rows, the driver fetches them, in one ebic_support_rows_batch,
//     for every following offspring that could place under the current archive.
//     Rows are a pure function of the candidate, so speculation is exact.
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
// cells are products, so the intersection is |rows n| * |cols n|.
double cell_overlap(const TopRankEntry& e, const std::vector<std::size_t>& rows,
                    const std::vector<std::size_t>& sorted_cols) {
  const std::size_t shared = sorted_intersection_size(e.rows, rows) * sorted_intersection_size(e.cols, sorted_cols);
  const std::size_t cells_e = e.rows.size() * e.cols.size(), cells_c = rows.size() * sorted_cols.size();
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
struct Device {
  ebic_ctx* ctx = nullptr;
  double approx = 0.0;
  int neg = 0;
  uint64_t launches0 = 0;

  Device(const ExpressionMatrix& m, const TrendParams& tp, int device) {
    check(ebic_ctx_create(device, &ctx), "context");
    check(ebic_matrix_upload_f64(ctx, m.values().data(), m.rows(), m.cols(), 0, EBIC_STORE_AUTO, nullptr),
          "matrix upload");
    approx = tp.approx;
    neg = tp.negative_trends ? 1 : 0;
    check(ebic_matrix_prepare(ctx, approx), "rank plane");
  }
  ~Device() {
    if (ctx) ebic_ctx_destroy(ctx);
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

// The top-rank archive (evolution.hpp:78-98): the acceptance rule of
// TopRankList::insert (evolution.cpp:76-105), fed with precomputed row sets.
class Archive {
 public:
  Archive(std::size_t capacity, double overlap) : capacity_(capacity), overlap_(overlap) {}

  const std::vector<TopRankEntry>& entries() const { return entries_; }
  bool full() const { return entries_.size() >= capacity_; }
  double min_score() const { return entries_.empty() ? 0.0 : entries_.back().ind.score; }

  // can the candidate enter at all -- i.e. does the reference compute its rows
  // (evolution.cpp:78-79)?
  bool could_place(const RankedIndividual& ind) const {
    return ind.score > 0.0 && !(full() && ind.score <= min_score());
  }

  bool insert(const RankedIndividual& ind, const std::vector<std::size_t>& rows) {
    if (!could_place(ind)) return false;
    TopRankEntry fresh;
    fresh.ind = ind;
    fresh.rows = rows;
    fresh.cols = ind.chromosome.columns;
    std::sort(fresh.cols.begin(), fresh.cols.end());
    // entries overlapping the candidate too much are displaced -- unless one of
    // them scores at least as high, in which case the candidate is rejected
    std::vector<char> displaced(entries_.size(), 0);
    for (std::size_t i = 0; i < entries_.size(); ++i) {
      if (cell_overlap(entries_[i], fresh.rows, fresh.cols) < overlap_) continue;
      if (entries_[i].ind.score >= ind.score) return false;
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
    const auto at = std::upper_bound(entries_.begin(), entries_.end(), fresh,
                                     [](const TopRankEntry& a, const TopRankEntry& b) {
                                       return archive_before(a.ind, b.ind);
                                     });
    entries_.insert(at, std::move(fresh));
    if (entries_.size() > capacity_) entries_.resize(capacity_);
    // placed iff it survived the truncation
    return std::any_of(entries_.begin(), entries_.end(), [&](const TopRankEntry& e) {
      return e.ind.score == ind.score && e.ind.chromosome.columns == ind.chromosome.columns;
    });
  }

 private:
  std::vector<TopRankEntry> entries_;
  std::size_t capacity_;
  double overlap_;
};

// Serial archive inserts in offspring order, with speculative batched row sets.
class RowBatcher {
 public:
  RowBatcher(Device& dev, std::size_t batch) : dev_(dev), batch_(std::max<std::size_t>(batch, 1)) {}

  const std::vector<std::size_t>& rows_for(std::size_t i, const std::vector<RankedIndividual>& inds,
                                           const Archive& arch) {
    auto it = cache_.find(i);
    if (it != cache_.end()) return it->second;
    // i itself plus up to batch-1 later candidates that could place right now
    std::vector<std::size_t> pick{i};
    for (std::size_t k = i + 1; k < inds.size() && pick.size() < batch_; ++k)
      if (arch.could_place(inds[k]) && cache_.find(k) == cache_.end()) pick.push_back(k);
    std::vector<uint32_t> cols, offs{0};
    for (std::size_t k : pick) {
      for (std::size_t c : inds[k].chromosome.columns) cols.push_back(static_cast<uint32_t>(c));
      offs.push_back(static_cast<uint32_t>(cols.size()));
    }
    std::vector<uint64_t> row_offs(pick.size() + 1);
    std::vector<uint32_t> rows(cap_);
    int st = ebic_support_rows_batch(dev_.ctx, cols.data(), offs.data(), pick.size(), dev_.approx, dev_.neg,
                                     rows.data(), rows.size(), row_offs.data());
    if (st == EBIC_ERR_CAPACITY) {
      cap_ = row_offs.back() + row_offs.back() / 2;
      rows.assign(cap_, 0);
      st = ebic_support_rows_batch(dev_.ctx, cols.data(), offs.data(), pick.size(), dev_.approx, dev_.neg,
                                   rows.data(), rows.size(), row_offs.data());
    }
    check(st, "supporting_rows");
    for (std::size_t b = 0; b < pick.size(); ++b)
      cache_[pick[b]] = std::vector<std::size_t>(rows.begin() + static_cast<std::ptrdiff_t>(row_offs[b]),
                                                 rows.begin() + static_cast<std::ptrdiff_t>(row_offs[b + 1]));
    return cache_[i];
  }

  void clear() { cache_.clear(); }

 private:
  Device& dev_;
  std::size_t batch_;
  std::size_t cap_ = 1 << 16;
  std::unordered_map<std::size_t, std::vector<std::size_t>> cache_;
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

// evolution.cpp:305-333 with the device evaluator on the caller side.
RunResult run(const ExpressionMatrix& m, const EvolutionParams& p, int device = 0) {
  p.validate();
  if (m.rows() == 0 || m.cols() < 2) throw std::invalid_argument("run: matrix too small");
  const auto t0 = std::chrono::steady_clock::now();

  Device dev(m, p.trend, device);
  const std::size_t chunk = std::max<std::size_t>(256, p.population_size / 4);
  RowBatcher rows(dev, 64);

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

  std::string reason = "budget";
  while (st.generation < p.max_iterations) {
    if (st.tabu.hit_count >= p.effective_tabu_threshold()) {
      reason = "converged";
      break;
    }
    // step_generation (evolution.cpp:248-303)
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
    const bool improved = rank_and_insert(std::move(offspring), counts, st, p, rows, next);
    if (improved) st.tabu.hit_count = 0;
    st.population = std::move(next);
    st.column_usage = tally_columns(st.population, num_cols);
    ++st.generation;
  }

  RunResult result;
  for (const auto& entry : st.top_rank.entries()) {
    if (result.biclusters.size() >= p.num_biclusters) break;
    if (entry.ind.support_count < p.trend.min_rows) continue;
    result.biclusters.biclusters.emplace_back(entry.rows, entry.cols);
  }
  result.report.generations = st.generation;
  result.report.termination = reason;
  result.report.wall_time_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

}  // namespace bicseek_device
