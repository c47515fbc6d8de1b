// Minimal stand-in for doctest.h -- TEST INFRASTRUCTURE ONLY.
// Provides exactly what the reference's unit tests use: TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx, and the
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN runner.  The runner takes optional
// test-case name substrings as arguments and exits non-zero on any failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

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
struct Stats {
  long checks = 0, failed = 0;
  bool case_failed = false;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct RequireFailed {};

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++stats().checks;
  if (ok) return;
  ++stats().failed;
  stats().case_failed = true;
  std::printf("  %s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) <= b.eps_ * (std::max)(1.0, (std::max)(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-05;  // doctest's default: float epsilon * 100
};

inline int run(int argc, char** argv) {
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    bool selected = argc <= 1;
    for (int a = 1; a < argc; ++a)
      if (std::strstr(tc.name, argv[a])) selected = true;
    if (!selected) continue;
    ++cases;
    stats().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++stats().failed;
      stats().case_failed = true;
      std::printf("  %s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
    }
    if (stats().case_failed) {
      ++failed_cases;
      std::printf("[FAILED] %s\n", tc.name);
    } else {
      std::printf("[ok] %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed; checks: %ld | %ld failed\n",
              cases, cases - failed_cases, failed_cases, stats().checks, stats().failed);
  return failed_cases == 0 && cases > 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                          \
  static void fn();                                                                   \
  static const int DOCTEST_CAT(fn, _reg) = ::doctest::reg(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool thrown_ = false;                                                            \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      thrown_ = true;                                                                \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::report(thrown_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run(argc, argv); }
#endif
