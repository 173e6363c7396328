// run_driver.cpp -- end-to-end parity driver for BASELINE config 1 (test
// infrastructure).  Generates a planted-trend scenario with the reference
// generator (datagen.cpp:208-264), float32-quantises it, and calls the
// reference's own bicseek::run (evolution.cpp:305-333).  oracle/Makefile links
// it twice against the SAME unmodified evolution.cpp:
//   oracle/_ref/run_ref     with the reference trend.cpp      (CPU evaluator)
//   oracle/_ref/run_device  with bicseek_trend_device.cpp     (B200 evaluator)
//   oracle/_ref/run_device_overlap  additionally --engine device: the
//                   device-aware driver (csrc/bicseek_run_device.cpp)
// and tests/test_gpu_reference_suite.py requires byte-identical output.
//
// Output (stdout, one JSON object): the canonical bicluster JSON of
// io.cpp:131-150 (restated), generations, termination, evaluation count.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bicseek/datagen.hpp"
#include "bicseek/evolution.hpp"
#include "bicseek/trend.hpp"

using namespace bicseek;

#ifdef EBIC_DEVICE_RUN
// paper_2105_01196_b200/csrc/bicseek_run_device.cpp: the device-aware driver
namespace bicseek_device {
RunResult run(const ExpressionMatrix& m, const EvolutionParams& p, int device);
void warm(int device);
}
#endif

static std::string bics_json(const BiclusterSet& set) {
  std::string out = "{\"biclusters\":[";
  for (std::size_t i = 0; i < set.size(); ++i) {
    if (i) out += ',';
    out += "{\"rows\":[";
    const auto& b = set.biclusters[i];
    for (std::size_t k = 0; k < b.rows.size(); ++k) out += (k ? "," : "") + std::to_string(b.rows[k]);
    out += "],\"cols\":[";
    for (std::size_t k = 0; k < b.cols.size(); ++k) out += (k ? "," : "") + std::to_string(b.cols[k]);
    out += "]}";
  }
  out += "]}";
  return out;
}

int main(int argc, char** argv) {
  ScenarioSpec s;
  s.scenario = ScenarioKind::six_types;
  s.pattern = PatternKind::trend;
  s.matrix_rows = 500;
  s.matrix_cols = 100;
  s.bic_rows = 50;
  s.bic_cols = 8;
  s.num_biclusters = 3;
  s.seed = 1;
  EvolutionParams p;
  p.max_iterations = 200;
  bool quantize = true;
  bool warm = false;
  int jobs = 1;
  std::string engine = "reference";
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--rows") s.matrix_rows = std::strtoull(v, nullptr, 10);
    else if (k == "--cols") s.matrix_cols = std::strtoull(v, nullptr, 10);
    else if (k == "--bic-rows") s.bic_rows = std::strtoull(v, nullptr, 10);
    else if (k == "--bic-cols") s.bic_cols = std::strtoull(v, nullptr, 10);
    else if (k == "--num-bics") s.num_biclusters = std::strtoull(v, nullptr, 10);
    else if (k == "--noise") s.noise_sigma = std::strtod(v, nullptr);
    else if (k == "--data-seed") s.seed = std::strtoull(v, nullptr, 10);
    else if (k == "--pop") p.population_size = std::strtoull(v, nullptr, 10);
    else if (k == "--iters") p.max_iterations = std::strtoull(v, nullptr, 10);
    else if (k == "--tabu") p.tabu_hits_threshold = std::strtoull(v, nullptr, 10);
    else if (k == "--seed") p.seed = std::strtoull(v, nullptr, 10);
    else if (k == "--threads") p.threads = static_cast<unsigned>(std::strtoul(v, nullptr, 10));
    else if (k == "--approx") p.trend.approx = std::strtod(v, nullptr);
    else if (k == "--negative") p.trend.negative_trends = std::atoi(v) != 0;
    else if (k == "--quantize") quantize = std::atoi(v) != 0;
    else if (k == "--warm") warm = std::atoi(v) != 0;
    else if (k == "--engine") engine = v;
    else if (k == "--jobs") jobs = std::atoi(v);
    // non-default GA parameters (evolution.hpp:20-39)
    else if (k == "--overlap") p.overlap_threshold = std::strtod(v, nullptr);
    else if (k == "--tournament") p.tournament_size = std::strtoull(v, nullptr, 10);
    else if (k == "--biclusters") p.num_biclusters = std::strtoull(v, nullptr, 10);
    else if (k == "--elite") p.elite_count = std::strtoull(v, nullptr, 10);
    else if (k == "--penalty") p.penalty_base = std::strtod(v, nullptr);
    else if (k == "--weights") {  // five comma-separated operator weights
      char* e = const_cast<char*>(v);
      for (double& w : p.operator_weights) {
        w = std::strtod(e, &e);
        if (*e == ',') ++e;
      }
    }
    else {
      std::fprintf(stderr, "unknown option %s\n", k.c_str());
      return 2;
    }
  }
  if (jobs > 1) {
    // independent datasets, one run() per thread (bench.cpp:103-121's --jobs):
    // job j uses data seed + j and GA seed + j; one JSON line per job, in order
    std::vector<std::string> lines(jobs);
    std::vector<std::thread> pool;
    for (int j = 0; j < jobs; ++j)
      pool.emplace_back([&, j] {
        ScenarioSpec sj = s;
        sj.seed = s.seed + j;
        EvolutionParams pj = p;
        pj.seed = p.seed + j;
        GeneratedDataset dj = gen_scenario(sj);
        std::vector<double> vj = dj.matrix.values();
        if (quantize)
          for (double& x : vj) x = static_cast<double>(static_cast<float>(x));
        const ExpressionMatrix mj(std::move(vj), dj.matrix.rows(), dj.matrix.cols(), dj.matrix.row_labels(),
                                  dj.matrix.col_labels());
        const RunResult rj = run(mj, pj);
        char buf[160];
        std::snprintf(buf, sizeof buf, ",\"generations\":%zu,\"termination\":\"%s\"}", rj.report.generations,
                      rj.report.termination.c_str());
        lines[j] = "{\"job\":" + std::to_string(j) + ",\"result\":" + bics_json(rj.biclusters) + buf;
      });
    for (auto& t : pool) t.join();
    for (const auto& l : lines) std::printf("%s\n", l.c_str());
    return 0;
  }
  GeneratedDataset d = gen_scenario(s);
  std::vector<double> v = d.matrix.values();
  if (quantize)
    for (double& x : v) x = static_cast<double>(static_cast<float>(x));
  const ExpressionMatrix m(std::move(v), d.matrix.rows(), d.matrix.cols(), d.matrix.row_labels(),
                           d.matrix.col_labels());
  if (warm) {
    // one tiny evaluation before run(): takes one-time device/context start-up
    // (CUDA context creation for the device build) out of run()'s own timer
    const ExpressionMatrix w({1.0, 2.0, 2.0, 1.0}, 2, 2, default_labels('r', 2), default_labels('c', 2));
    (void)evaluate_population(w, {Chromosome({0, 1})}, p.trend, nullptr);
#ifdef EBIC_DEVICE_RUN
    if (engine != "reference") bicseek_device::warm(0);  // the driver's own (per-thread) context
#endif
  }
  RunResult r;
  if (engine == "reference") {
    r = run(m, p);
  } else {
#ifdef EBIC_DEVICE_RUN
    r = bicseek_device::run(m, p, 0);
#else
    std::fprintf(stderr, "engine '%s' not built into this binary\n", engine.c_str());
    return 2;
#endif
  }
  std::printf("{\"result\":%s,\"generations\":%zu,\"termination\":\"%s\",\"wall_s\":%.6f}\n",
              bics_json(r.biclusters).c_str(), r.report.generations, r.report.termination.c_str(),
              r.report.wall_time_seconds);
  return 0;
}
