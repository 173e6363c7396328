// ref_capi.cpp -- extern "C" glue over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libbicseek_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (golden fixtures, live parity),
// __graft_entry__.smoke() is NOT required to have it, and bench.py uses it only
// for the CPU-baseline leg / `--impl reference` arm.  It exposes the
// reference's own generator (datagen.cpp:64-70, 208-264), population
// initialiser (evolution.cpp:117-126 in SURVEY numbering; init_population),
// evaluator (trend.cpp:56-72 on a WorkerPool, worker_pool.cpp:20-48) and
// supporting_rows (trend.cpp:48-54), so Python can drive them by pointer.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bicseek/datagen.hpp"
#ifdef REF_HAVE_IO
#include "bicseek/io.hpp"
#endif
#include "bicseek/evolution.hpp"
#include "bicseek/rng.hpp"
#include "bicseek/trend.hpp"
#include "bicseek/worker_pool.hpp"

using namespace bicseek;

namespace {
thread_local std::string g_err;

int guard(const std::exception& e) {
  g_err = e.what();
  return 1;
}

void quantize(std::vector<double>& v) {
  for (double& x : v) x = static_cast<double>(static_cast<float>(x));
}

std::vector<Chromosome> to_pop(const uint32_t* cols, const uint32_t* offs, uint64_t n) {
  std::vector<Chromosome> pop;
  pop.reserve(n);
  for (uint64_t i = 0; i < n; ++i)
    pop.emplace_back(std::vector<std::size_t>(cols + offs[i], cols + offs[i + 1]));
  return pop;
}

TrendParams tparams(double approx, int neg) {
  TrendParams p;
  p.approx = approx;
  p.negative_trends = neg != 0;
  return p;
}

ScenarioKind scen(int k) { return static_cast<ScenarioKind>(k); }
PatternKind patt(int k) { return static_cast<PatternKind>(k); }
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// gen_background(rows, cols, seed), optionally float32-quantised.
int ref_gen_background(uint64_t rows, uint64_t cols, uint64_t seed, int quantize_f32, double* out) {
  try {
    ExpressionMatrix m = gen_background(rows, cols, seed);
    std::vector<double> v = m.values();
    if (quantize_f32) quantize(v);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// gen_scenario(ScenarioSpec{...}).  scenario/pattern are the enum ordinals of
// datagen.hpp:15-26.  truth rows/cols are written as CSR if buffers are given.
int ref_gen_scenario(int scenario, int pattern, uint64_t rows, uint64_t cols, uint64_t bic_rows,
                     uint64_t bic_cols, uint64_t num_bics, double noise, double mean_shift,
                     uint64_t seed, int quantize_f32, double* out) {
  try {
    ScenarioSpec s;
    s.scenario = scen(scenario);
    s.pattern = patt(pattern);
    s.matrix_rows = rows;
    s.matrix_cols = cols;
    s.bic_rows = bic_rows;
    s.bic_cols = bic_cols;
    s.num_biclusters = num_bics;
    s.noise_sigma = noise;
    s.mean_shift = mean_shift;
    s.seed = seed;
    GeneratedDataset d = gen_scenario(s);
    std::vector<double> v = d.matrix.values();
    if (quantize_f32) quantize(v);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// init_population(EvolutionParams{population_size, init_len_min/max}, num_cols, Rng(seed)).
// Writes CSR; cols_out needs pop_size * len_max entries.
int ref_init_population(uint64_t pop_size, uint64_t num_cols, uint64_t seed, uint64_t len_min,
                        uint64_t len_max, uint32_t* cols_out, uint32_t* offs_out) {
  try {
    EvolutionParams p;
    p.population_size = pop_size;
    p.init_len_min = len_min;
    p.init_len_max = len_max;
    Rng rng(seed);
    std::vector<Chromosome> pop = init_population(p, num_cols, rng);
    uint32_t o = 0;
    offs_out[0] = 0;
    for (uint64_t i = 0; i < pop.size(); ++i) {
      for (std::size_t c : pop[i].columns) cols_out[o++] = static_cast<uint32_t>(c);
      offs_out[i + 1] = o;
    }
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// Opaque handles so the timed region contains only evaluate_population.
void* ref_matrix_create(const double* values, uint64_t rows, uint64_t cols) {
  try {
    std::vector<double> v(values, values + rows * cols);
    return new ExpressionMatrix(std::move(v), rows, cols, default_labels('r', rows),
                                default_labels('c', cols));
  } catch (const std::exception& e) {
    guard(e);
    return nullptr;
  }
}
void ref_matrix_destroy(void* m) { delete static_cast<ExpressionMatrix*>(m); }

void* ref_population_create(const uint32_t* cols, const uint32_t* offs, uint64_t n) {
  return new std::vector<Chromosome>(to_pop(cols, offs, n));
}
void ref_population_destroy(void* p) { delete static_cast<std::vector<Chromosome>*>(p); }

void* ref_pool_create(unsigned threads) { return new WorkerPool(threads); }
void ref_pool_destroy(void* p) { delete static_cast<WorkerPool*>(p); }
unsigned ref_pool_size(void* p) { return static_cast<WorkerPool*>(p)->size(); }

// evaluate_population(m, pop, p, pool) -- trend.cpp:56-72.
int ref_evaluate_population(void* m, void* pop, double approx, int neg, void* pool,
                            uint32_t* counts_out) {
  try {
    const auto counts = evaluate_population(*static_cast<ExpressionMatrix*>(m),
                                            *static_cast<std::vector<Chromosome>*>(pop),
                                            tparams(approx, neg), static_cast<WorkerPool*>(pool));
    for (std::size_t i = 0; i < counts.size(); ++i) counts_out[i] = static_cast<uint32_t>(counts[i]);
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// supporting_rows -- trend.cpp:48-54.  Returns the count; writes <= cap rows.
int64_t ref_supporting_rows(void* m, const uint32_t* cols, uint32_t len, double approx, int neg,
                            uint32_t* rows_out, uint64_t cap) {
  try {
    Chromosome c(std::vector<std::size_t>(cols, cols + len));
    const auto rows = supporting_rows(*static_cast<ExpressionMatrix*>(m), c, tparams(approx, neg));
    for (std::size_t i = 0; i < rows.size() && i < cap; ++i) rows_out[i] = static_cast<uint32_t>(rows[i]);
    return static_cast<int64_t>(rows.size());
  } catch (const std::exception& e) {
    guard(e);
    return -1;
  }
}

// row_supports -- trend.cpp:41-46.
int ref_row_supports(void* m, uint64_t row, const uint32_t* cols, uint32_t len, double approx,
                     int neg) {
  Chromosome c(std::vector<std::size_t>(cols, cols + len));
  return row_supports(*static_cast<ExpressionMatrix*>(m), row, c, tparams(approx, neg)) ? 1 : 0;
}

double ref_fitness(uint64_t count, uint64_t ncols, uint64_t min_rows, uint64_t col_cap) {
  TrendParams p;
  p.min_rows = min_rows;
  p.col_cap = col_cap;
  return fitness(count, ncols, p);
}

// Draws of test_trend.cpp's random_chromosome_for (test_trend.cpp:29-34),
// restated: len = 2 + uniform_index(min(6, C-1)); sample_sorted; shuffle.
// Used to regenerate the reference test's populations for golden fixtures.
int ref_test_chromosomes(uint64_t seed, uint64_t n, uint64_t num_cols, uint32_t* cols_out,
                         uint32_t* offs_out) {
  Rng rng(seed);
  uint32_t o = 0;
  offs_out[0] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const std::size_t len = 2 + rng.uniform_index(std::min<std::size_t>(6, num_cols - 1));
    std::vector<std::size_t> cols = rng.sample_sorted(num_cols, len);
    rng.shuffle(cols);
    for (std::size_t c : cols) cols_out[o++] = static_cast<uint32_t>(c);
    offs_out[i + 1] = o;
  }
  return 0;
}


#ifdef REF_HAVE_IO
// The reference TSV reader (io.cpp:78-111): row-major values into out (cap
// elements), shape into rows/cols.  1 on error (ref_last_error: the reference's
// own ParseError message), 2 if cap is too small (shape filled).
int ref_parse_matrix_tsv(const char* path, double* out, uint64_t cap, uint64_t* rows, uint64_t* cols) {
  try {
    const ExpressionMatrix m = parse_matrix_tsv(path);
    *rows = m.rows();
    *cols = m.cols();
    if (cap < m.rows() * m.cols()) return 2;
    std::memcpy(out, m.values().data(), m.values().size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}

// The reference TSV writer (io.cpp:113-130, %.17g) with generated labels.
int ref_write_matrix_tsv(const char* path, const double* v, uint64_t rows, uint64_t cols) {
  try {
    ExpressionMatrix m(std::vector<double>(v, v + rows * cols), rows, cols, default_labels('r', rows),
                       default_labels('c', cols));
    write_matrix_tsv(path, m);
    return 0;
  } catch (const std::exception& e) {
    return guard(e);
  }
}
#endif
}  // extern "C"
