// shim_cache_check.cpp -- test driver (test infrastructure only) for the
// drop-in TU's device matrix cache (paper_2105_01196_b200/csrc/
// bicseek_trend_device.cpp): calls the UNCHANGED trend.hpp API on one
// bicseek::ExpressionMatrix that it mutates in place between calls, as a
// script says, and prints every result.  tests/test_gpu_shim_cache.py runs the
// same script through the C oracle and requires identical output.
//
// Script (stdin, whitespace separated):
//   <rows> <cols> <rows*cols doubles, row-major>
//   E <approx> <neg> <n> {<len> <cols...>} x n   evaluate_population -> "E c0 c1 ..."
//   S <approx> <neg> <len> <cols...>             supporting_rows     -> "S r0 r1 ..."
//   W <approx> <neg> <row> <len> <cols...>       row_supports        -> "W 0|1"
//   M <row> <col> <value>                        m(row, col) = value (in place)
//   N <seed-free: rows cols values...>           replace the matrix (a new object)
#include <cstdio>
#include <iostream>
#include <memory>
#include <vector>

#include "bicseek/matrix.hpp"
#include "bicseek/trend.hpp"

using namespace bicseek;

static std::unique_ptr<ExpressionMatrix> read_matrix() {
  std::size_t r = 0, c = 0;
  std::cin >> r >> c;
  std::vector<double> v(r * c);
  for (double& x : v) std::cin >> x;
  std::vector<std::string> rl(r), cl(c);
  for (std::size_t i = 0; i < r; ++i) rl[i] = "r" + std::to_string(i);
  for (std::size_t j = 0; j < c; ++j) cl[j] = "c" + std::to_string(j);
  return std::make_unique<ExpressionMatrix>(std::move(v), r, c, std::move(rl), std::move(cl));
}

static Chromosome read_chrom() {
  std::size_t len = 0;
  std::cin >> len;
  Chromosome ch;
  ch.columns.resize(len);
  for (auto& x : ch.columns) std::cin >> x;
  return ch;
}

int main() {
  std::cin.precision(17);
  auto m = read_matrix();
  char op;
  while (std::cin >> op) {
    TrendParams p;
    if (op == 'M') {
      std::size_t r, c;
      double x;
      std::cin >> r >> c >> x;
      (*m)(r, c) = x;
      continue;
    }
    if (op == 'N') {
      m = read_matrix();
      continue;
    }
    int neg = 0;
    std::cin >> p.approx >> neg;
    p.negative_trends = neg != 0;
    if (op == 'E') {
      std::size_t n;
      std::cin >> n;
      std::vector<Chromosome> pop(n);
      for (auto& ch : pop) ch = read_chrom();
      std::printf("E");
      for (std::size_t x : evaluate_population(*m, pop, p)) std::printf(" %zu", x);
    } else if (op == 'S') {
      const Chromosome ch = read_chrom();
      std::printf("S");
      for (std::size_t x : supporting_rows(*m, ch, p)) std::printf(" %zu", x);
    } else if (op == 'W') {
      std::size_t row;
      std::cin >> row;
      const Chromosome ch = read_chrom();
      std::printf("W %d", row_supports(*m, row, ch, p) ? 1 : 0);
    }
    std::printf("\n");
  }
  return 0;
}
