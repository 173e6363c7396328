// Minimal doctest-compatible shim (test infrastructure; a new file, not the
// doctest library).  The reference's tests (proj/tests/*.cpp) include
// <doctest.h> from an un-vendored proj/vendor/ (SURVEY.md section 4); this
// header provides exactly the subset they use -- TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS, doctest::Approx -- so
// test_trend.cpp compiles UNCHANGED against either the reference trend.cpp or
// the device drop-in TU.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Registry {
  struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
  };
  std::vector<Case> cases;
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().cases.push_back({name, file, line, fn});
  }
};

struct RequireAbort {};

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
  auto& r = Registry::get();
  ++r.checks;
  if (ok) return;
  ++r.failed_checks;
  r.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
  if (fatal) throw RequireAbort{};
}

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

inline int run_all() {
  auto& r = Registry::get();
  int failed_cases = 0;
  for (const auto& c : r.cases) {
    r.case_failed = false;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      r.case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: test case '%s' threw an unknown exception\n", c.file, c.line,
                   c.name);
      r.case_failed = true;
    }
    if (r.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", r.cases.size(),
              r.cases.size() - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", r.checks,
              r.checks - r.failed_checks, r.failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                          \
  static void fn();                                                                        \
  static ::doctest::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    bool ok_ = true;                                                                       \
    try {                                                                                  \
      (void)(__VA_ARGS__);                                                                 \
    } catch (...) {                                                                        \
      ok_ = false;                                                                         \
    }                                                                                      \
    ::doctest::report(ok_, "CHECK_NOTHROW(" #__VA_ARGS__ ")", __FILE__, __LINE__, false);  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool ok_ = false;                                                                      \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      ok_ = true;                                                                          \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::report(ok_, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__,       \
                      __LINE__, false);                                                    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
