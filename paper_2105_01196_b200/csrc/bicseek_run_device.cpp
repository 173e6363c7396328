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
// The archive insert, operator pick, and the small helpers that the reference
// keeps in an anonymous namespace are restated below (file:line cited).  Every
// other piece is the reference's own function, linked unchanged.
#include <algorithm>
#include <chrono>
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

constexpr int kTabuRetryBudget = 3;  // evolution.cpp:12

void check(int status, const char* what) {
  if (status != EBIC_OK)
    throw std::runtime_error(std::string("bicseek device run: ") + what + ": " + ebic_last_error());
}

// evolution.cpp:25-34
OperatorKind pick_operator(const std::array<double, 5>& weights, Rng& rng) {
  double total = 0.0;
  for (double w : weights) total += w;
  double r = rng.uniform_real() * total;
  for (std::size_t i = 0; i + 1 < weights.size(); ++i) {
    if (r < weights[i]) return static_cast<OperatorKind>(i);
    r -= weights[i];
  }
  return OperatorKind::crossover;
}

// evolution.cpp:38-42: score desc, then fewer columns, then lexicographic columns
bool ranks_before(const RankedIndividual& a, const RankedIndividual& b) {
  if (a.score != b.score) return a.score > b.score;
  if (a.chromosome.size() != b.chromosome.size()) return a.chromosome.size() < b.chromosome.size();
  return a.chromosome.columns < b.chromosome.columns;
}

// evolution.cpp:44-51
double induced_jaccard(const TopRankEntry& a, const std::vector<std::size_t>& rows,
                       const std::vector<std::size_t>& cols) {
  const std::size_t inter =
      sorted_intersection_size(a.rows, rows) * sorted_intersection_size(a.cols, cols);
  const std::size_t size_a = a.rows.size() * a.cols.size();
  const std::size_t size_b = rows.size() * cols.size();
  return static_cast<double>(inter) / static_cast<double>(size_a + size_b - inter);
}

// evolution.cpp:215-221
std::vector<std::size_t> column_usage_of(const std::vector<RankedIndividual>& pop, std::size_t num_cols) {
  std::vector<std::size_t> usage(num_cols, 0);
  for (const auto& ind : pop)
    for (std::size_t col : ind.chromosome.columns) ++usage[col];
  return usage;
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

// The top-rank archive of evolution.hpp:78-98 with TopRankList::insert
// (evolution.cpp:76-105) restated; rows come from a batch cache.
class Archive {
 public:
  Archive(std::size_t capacity, double overlap) : capacity_(capacity), overlap_(overlap) {}

  const std::vector<TopRankEntry>& entries() const { return entries_; }
  bool full() const { return entries_.size() >= capacity_; }
  double min_score() const { return entries_.empty() ? 0.0 : entries_.back().ind.score; }

  // would insert() need the candidate's rows (evolution.cpp:78-79)?
  bool could_place(const RankedIndividual& ind) const {
    return ind.score > 0.0 && !(full() && ind.score <= min_score());
  }

  bool insert(const RankedIndividual& ind, const std::vector<std::size_t>& rows) {
    if (!could_place(ind)) return false;
    TopRankEntry cand;
    cand.ind = ind;
    cand.rows = rows;
    cand.cols = ind.chromosome.columns;
    std::sort(cand.cols.begin(), cand.cols.end());
    std::vector<std::size_t> displaced;
    for (std::size_t i = 0; i < entries_.size(); ++i) {
      if (induced_jaccard(entries_[i], cand.rows, cand.cols) < overlap_) continue;
      if (entries_[i].ind.score >= ind.score) return false;  // incumbent wins ties
      displaced.push_back(i);
    }
    for (std::size_t k = displaced.size(); k-- > 0;)
      entries_.erase(entries_.begin() + static_cast<std::ptrdiff_t>(displaced[k]));
    auto pos = std::find_if(entries_.begin(), entries_.end(),
                            [&](const TopRankEntry& e) { return ranks_before(cand.ind, e.ind); });
    entries_.insert(pos, std::move(cand));
    if (entries_.size() > capacity_) entries_.resize(capacity_);
    return entries_.size() <= capacity_ &&
           std::any_of(entries_.begin(), entries_.end(), [&](const TopRankEntry& e) {
             return e.ind.chromosome.columns == ind.chromosome.columns && e.ind.score == ind.score;
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
    st.column_usage = column_usage_of(st.population, m.cols());
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
      Chromosome child;
      bool accepted = false;
      for (int attempt = 0; attempt < kTabuRetryBudget; ++attempt) {
        const RankedIndividual& parent = tournament_select(st.population, st.column_usage, p, st.rng);
        const OperatorKind op = pick_operator(p.operator_weights, st.rng);
        if (op == OperatorKind::crossover) {
          const RankedIndividual& other = tournament_select(st.population, st.column_usage, p, st.rng);
          child = crossover(parent.chromosome, other.chromosome, st.rng);
        } else {
          child = mutate(parent.chromosome, op, num_cols, st.rng);
        }
        const std::uint64_t h = chromosome_hash(child);
        if (st.tabu.contains(h)) {
          ++st.tabu.hit_count;
          continue;
        }
        st.tabu.insert(h);
        accepted = true;
        break;
      }
      if (!accepted) {
        child = random_chromosome(p, num_cols, st.rng);
        st.tabu.insert(chromosome_hash(child));
      }
      offspring.push_back(std::move(child));
      ev.add(offspring);  // overlap: the GPU counts this chunk while the next is bred
    }
    const std::vector<std::size_t> counts = ev.finish(offspring);
    const bool improved = rank_and_insert(std::move(offspring), counts, st, p, rows, next);
    if (improved) st.tabu.hit_count = 0;
    st.population = std::move(next);
    st.column_usage = column_usage_of(st.population, num_cols);
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
