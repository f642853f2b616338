// doctest-subset shim — ORACLE TEST INFRASTRUCTURE ONLY.
//
// doctest is expected in the reference's gitignored proj/vendor/
// (/root/reference/proj/.gitignore:2, tests/test_main.cpp:1-2) and is absent
// here.  This header implements the subset the reference hot-path unit tests
// use (TEST_CASE, SUBCASE, CHECK*, REQUIRE*, CHECK_THROWS_AS, doctest::Approx
// with .epsilon()) so those UNMODIFIED test files can be compiled in place —
// against the shim-built reference (oracle/_ref) to pin the oracle, and against
// the GPU drop-in to show the reference's own tests pass on the B200 path.
//
// SUBCASE semantics: a test case is re-run once per leaf subcase; code outside
// subcases runs every time (matches doctest for the non-nested use here).
// Filtering: argv[1..] are substrings; a test case runs if its name contains any.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // float epsilon * 100, doctest default
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  int target = 0;       // leaf subcase index to enter on this run
  int seen = 0;         // subcases encountered on this run
  int entered_depth = 0;
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  const char* current = "";
};

inline State& st() {
  static State s;
  return s;
}

struct SubcaseGuard {
  bool active;
  explicit SubcaseGuard(const char*) {
    State& s = st();
    active = (s.seen == s.target);
    ++s.seen;
  }
  explicit operator bool() const { return active; }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = st();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    s.case_failed = true;
    std::printf("%s:%d: FAILED %s( %s ) in test case \"%s\"\n", file, line,
                require ? "REQUIRE" : "CHECK", expr, s.current);
    if (require) throw RequireFailed{};
  }
}

inline int run_all(int argc, char** argv) {
  int failed_cases = 0, ran = 0, skipped = 0;
  for (const auto& tc : registry()) {
    bool selected = argc <= 1;
    for (int i = 1; i < argc; ++i)
      if (std::strstr(tc.name, argv[i])) selected = true;
    if (!selected) {
      ++skipped;
      continue;
    }
    ++ran;
    State& s = st();
    s.current = tc.name;
    s.case_failed = false;
    for (int target = 0;; ++target) {
      s.target = target;
      s.seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.case_failed = true;
        std::printf("%s:%d: unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name,
                    e.what());
      }
      if (s.seen <= target + 1) break;
    }
    std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
    if (s.case_failed) ++failed_cases;
  }
  std::printf("test cases: %d ran, %d failed, %d skipped | checks: %ld, failed: %ld\n", ran,
              failed_cases, skipped, st().checks, st().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                      \
  static void fn();                                                                    \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                             &fn);                     \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) \
  if (const ::doctest::detail::SubcaseGuard DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ex)                                                    \
  do {                                                                               \
    bool doctest_threw_ = false;                                                     \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const ex&) {                                                            \
      doctest_threw_ = true;                                                         \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(doctest_threw_, #expr " throws " #ex, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS(expr)                                                           \
  do {                                                                               \
    bool doctest_threw_ = false;                                                     \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (...) {                                                                  \
      doctest_threw_ = true;                                                         \
    }                                                                                \
    ::doctest::detail::report(doctest_threw_, #expr " throws", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                          \
  do {                                                                               \
    bool doctest_ok_ = true;                                                         \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (...) {                                                                  \
      doctest_ok_ = false;                                                           \
    }                                                                                \
    ::doctest::detail::report(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
