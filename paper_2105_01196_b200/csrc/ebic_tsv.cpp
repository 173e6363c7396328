// ebic_tsv.cpp -- matrix ingest for the device store.
//
// The reference reads its matrix with parse_matrix_tsv (io.cpp:78-111): the
// whole file, split into lines ('\r' stripped, trailing empty lines dropped),
// a header of column labels (with or without a corner cell), then one line
// per row of label + values, every value parsed with std::from_chars (exact,
// round-to-nearest) and required to be finite.  At 200k x 2000 that is 400M
// from_chars calls on one thread.  This loader keeps those semantics and
// messages -- the same library call parses every cell, so the values are
// bit-identical -- but finds the lines and parses the rows on all host
// threads, straight into page-locked memory that the device store is uploaded
// from (ebic_matrix_load_tsv).  Row/column labels are not kept (the device path
// needs only the values), but they are checked like the ExpressionMatrix the
// reference parser constructs (matrix.cpp:43-49): a duplicate row label, then
// a duplicate column label, is an error with the reference's message.
#include <charconv>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_set>
#include <vector>

#include "ebic.h"

namespace ebic_tsv {
namespace {

struct Error {
  int code = EBIC_OK;
  uint64_t line = 0, col = 0;  // 1-based position of the first error (line-major order)
  std::string msg;
};

bool read_file(const char* path, std::string& out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(&out[0], 1, (size_t)n, f) : 0;
  std::fclose(f);
  return got == out.size();
}

// Line spans [begin, end) of the text, '\r' stripped, trailing empty lines
// dropped (io.cpp nonempty_lines_keep).  Newlines are found on all threads.
std::vector<std::pair<size_t, size_t>> lines_of(const std::string& text, int threads) {
  const size_t n = text.size();
  std::vector<std::vector<size_t>> nl(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      const size_t b = n * t / threads, e = n * (t + 1) / threads;
      const char* p = text.data();
      for (size_t i = b; i < e; ++i) {
        const void* q = std::memchr(p + i, '\n', e - i);
        if (!q) break;
        i = (size_t)(static_cast<const char*>(q) - p);
        nl[t].push_back(i);
      }
    });
  for (auto& th : pool) th.join();
  std::vector<std::pair<size_t, size_t>> lines;
  size_t start = 0;
  for (const auto& v : nl)
    for (size_t pos : v) {
      lines.emplace_back(start, pos);
      start = pos + 1;
    }
  lines.emplace_back(start, n);  // split() keeps the text after the last '\n'
  for (auto& l : lines)
    if (l.second > l.first && text[l.second - 1] == '\r') --l.second;
  while (!lines.empty() && lines.back().second == lines.back().first) lines.pop_back();
  return lines;
}

size_t count_fields(const char* b, const char* e) {
  size_t n = 1;
  for (const char* p = b; p < e; ++p) n += *p == '\t';
  return n;
}

struct Shape {
  uint64_t rows = 0, cols = 0;
};

Error shape_of(const std::string& text, const std::vector<std::pair<size_t, size_t>>& lines, const char* path,
               Shape& sh) {
  Error err;
  auto fail = [&](const std::string& m) {
    err.code = EBIC_ERR_INVALID_ARGUMENT;
    err.msg = m;
    return err;
  };
  if (lines.size() < 2) return fail(std::string(path) + ": need a header and at least one row");
  const size_t header = count_fields(text.data() + lines[0].first, text.data() + lines[0].second);
  const size_t data_fields = count_fields(text.data() + lines[1].first, text.data() + lines[1].second);
  if (data_fields < 2) return fail(std::string(path) + ": rows need a label and at least one value");
  const size_t cols = data_fields - 1;
  if (header != cols + 1 && header != cols)
    return fail(std::string(path) + ": header has " + std::to_string(header) + " labels for " +
                std::to_string(cols) + " columns");
  sh.rows = lines.size() - 1;
  sh.cols = cols;
  return err;
}

// Parse rows [r0, r1) (data line i = row i - 1) into values; first error of the range.
Error parse_rows(const std::string& text, const std::vector<std::pair<size_t, size_t>>& lines, const char* path,
                 const Shape& sh, uint64_t r0, uint64_t r1, double* values) {
  Error err;
  for (uint64_t r = r0; r < r1; ++r) {
    const uint64_t line_no = r + 2;  // 1-based file line of data row r
    const char* b = text.data() + lines[r + 1].first;
    const char* e = text.data() + lines[r + 1].second;
    const size_t fields = count_fields(b, e);
    if (fields != sh.cols + 1) {
      err.code = EBIC_ERR_INVALID_ARGUMENT;
      err.line = line_no;
      err.col = 0;
      err.msg = std::string(path) + ": ragged row at line " + std::to_string(line_no) + " (expected " +
                std::to_string(sh.cols + 1) + " fields, got " + std::to_string(fields) + ")";
      return err;
    }
    const char* p = static_cast<const char*>(std::memchr(b, '\t', (size_t)(e - b))) + 1;  // skip the label
    double* row = values + r * sh.cols;
    for (uint64_t j = 0; j < sh.cols; ++j) {
      const char* q = static_cast<const char*>(std::memchr(p, '\t', (size_t)(e - p)));
      if (!q) q = e;
      double v = 0.0;
      const auto res = std::from_chars(p, q, v);
      if (res.ec != std::errc() || res.ptr != q) {
        err.code = EBIC_ERR_INVALID_ARGUMENT;
        err.line = line_no;
        err.col = j + 2;
        err.msg = "non-numeric cell at line " + std::to_string(line_no) + ", column " + std::to_string(j + 2) +
                  ": '" + std::string(p, q) + "'";
        return err;
      }
      if (!std::isfinite(v)) {
        err.code = EBIC_ERR_INVALID_ARGUMENT;
        err.line = line_no;
        err.col = j + 2;
        err.msg = "non-finite cell at line " + std::to_string(line_no) + ", column " + std::to_string(j + 2);
        return err;
      }
      row[j] = v;
      p = q + 1;
    }
  }
  return err;
}

Error parse_all(const std::string& text, const std::vector<std::pair<size_t, size_t>>& lines, const char* path,
                const Shape& sh, double* values, int threads) {
  std::vector<Error> errs(threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      errs[t] = parse_rows(text, lines, path, sh, sh.rows * t / threads, sh.rows * (t + 1) / threads, values);
    });
  for (auto& th : pool) th.join();
  // the error the sequential reference parser would raise first: the lowest line
  for (const Error& e : errs)
    if (e.code != EBIC_OK) return e;  // thread ranges are in line order
  return Error{};
}

// ExpressionMatrix::validate's label rules (matrix.cpp:43-49), run after the
// values parsed (the reference constructs the matrix -- and validates it --
// only once every cell has parsed, io.cpp:108-109): the first label, in row
// order, that repeats an earlier one; then the same over the column labels.
Error check_labels(const std::string& text, const std::vector<std::pair<size_t, size_t>>& lines, const Shape& sh) {
  Error err;
  auto dup = [&](const char* what, std::string_view l) {
    err.code = EBIC_ERR_INVALID_ARGUMENT;
    err.msg = std::string("ExpressionMatrix: duplicate ") + what + " label '" + std::string(l) + "'";
    return err;
  };
  std::unordered_set<std::string_view> seen;
  seen.reserve(sh.rows * 2);
  for (uint64_t r = 0; r < sh.rows; ++r) {
    const char* b = text.data() + lines[r + 1].first;
    const char* e = text.data() + lines[r + 1].second;
    const char* t = static_cast<const char*>(std::memchr(b, '\t', (size_t)(e - b)));
    if (!seen.insert(std::string_view(b, (size_t)((t ? t : e) - b))).second)
      return dup("row", std::string_view(b, (size_t)((t ? t : e) - b)));
  }
  // header labels (io.cpp:85-90: a leading corner cell is dropped)
  std::vector<std::string_view> cols;
  {
    const char* b = text.data() + lines[0].first;
    const char* e = text.data() + lines[0].second;
    for (const char* p = b;;) {
      const char* t = static_cast<const char*>(std::memchr(p, '\t', (size_t)(e - p)));
      cols.emplace_back(p, (size_t)((t ? t : e) - p));
      if (!t) break;
      p = t + 1;
    }
    if (cols.size() == sh.cols + 1) cols.erase(cols.begin());
  }
  seen.clear();
  for (const auto& l : cols)
    if (!seen.insert(l).second) return dup("column", l);
  return err;
}

int clamp_threads(int n) {
  if (n <= 0) n = (int)std::thread::hardware_concurrency();
  return n < 1 ? 1 : (n > 256 ? 256 : n);
}

}  // namespace
}  // namespace ebic_tsv

// Implemented in ebic_capi.cu: thread-local error string (not exported).
extern "C" __attribute__((visibility("hidden"))) int ebic_internal_fail(int code, const char* msg);

extern "C" int ebic_tsv_read(const char* path, int n_threads, double* values_out, uint64_t cap, uint64_t* rows_out,
                             uint64_t* cols_out) {
  using namespace ebic_tsv;
  if (!path) return ebic_internal_fail(EBIC_ERR_INVALID_ARGUMENT, "null path");
  std::string text;
  if (!read_file(path, text)) return ebic_internal_fail(EBIC_ERR_IO, ("cannot open " + std::string(path)).c_str());
  const int threads = clamp_threads(n_threads);
  const auto lines = lines_of(text, threads);
  Shape sh;
  Error e = shape_of(text, lines, path, sh);
  if (e.code) return ebic_internal_fail(e.code, e.msg.c_str());
  if (rows_out) *rows_out = sh.rows;
  if (cols_out) *cols_out = sh.cols;
  if (!values_out || cap < sh.rows * sh.cols)
    return ebic_internal_fail(EBIC_ERR_CAPACITY, "values buffer too small for the matrix");
  e = parse_all(text, lines, path, sh, values_out, threads);
  if (e.code) return ebic_internal_fail(e.code, e.msg.c_str());
  e = check_labels(text, lines, sh);
  if (e.code) return ebic_internal_fail(e.code, e.msg.c_str());
  return EBIC_OK;
}
