// Minimal doctest-compatible harness (doctest itself is not in this image) so
// the reference's own unit suites (proj/tests/test_*.cpp) compile unchanged
// against include/eps/*.hpp and link against libeps_b200.so.  Covers exactly
// the macros those suites use: TEST_CASE, SUBCASE (run inline, in order),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, MESSAGE, FAIL
// and doctest::Approx(x).epsilon(e) (doctest's default epsilon
// FLT_EPSILON * 100, scaled by 1 + max(|a|, |b|)).
//
// Output: one line per failed check ("file:line: CHECK(expr) failed") and a
// final "[conformance] test cases: P passed, F failed | checks: P passed, F
// failed" line; exit status 1 when anything failed.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <sstream>
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value() || a.matches(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value() || a.matches(x); }
inline bool operator<=(const Approx& a, double x) { return a.value() < x || a.matches(x); }
inline bool operator>=(const Approx& a, double x) { return a.value() > x || a.matches(x); }

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
struct Stats {
  long checks_ok = 0, checks_bad = 0;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct Abort {};  // REQUIRE / FAIL: end the current test case

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline void report(bool ok, const char* macro, const char* expr, const char* file, int line) {
  if (ok) {
    ++stats().checks_ok;
    return;
  }
  ++stats().checks_bad;
  std::fprintf(stderr, "%s:%d: %s(%s) failed\n", file, line, macro, expr);
}

template <typename... Args>
std::string cat(const Args&... args) {
  std::ostringstream os;
  (os << ... << args);
  return os.str();
}

inline int run_all() {
  long cases_ok = 0, cases_bad = 0;
  long skipped = 0;
  const bool verbose = std::getenv("DOCTEST_VERBOSE") != nullptr;
  // DOCTEST_SKIP: '|'-separated test-case names not to run (a suite's own UB)
  const char* skip_env = std::getenv("DOCTEST_SKIP");
  const std::string skip = skip_env ? std::string("|") + skip_env + "|" : std::string();
  for (const TestCase& t : registry()) {
    if (!skip.empty() && skip.find(std::string("|") + t.name + "|") != std::string::npos) {
      ++skipped;
      std::printf("[conformance] skipped: %s\n", t.name);
      continue;
    }
    if (verbose) std::fprintf(stderr, "[conformance] running: %s\n", t.name);
    const long before = stats().checks_bad;
    bool threw = false;
    try {
      t.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      threw = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", t.file, t.line, t.name,
                   e.what());
    } catch (...) {
      threw = true;
      std::fprintf(stderr, "%s:%d: test case \"%s\" threw a non-std exception\n", t.file,
                   t.line, t.name);
    }
    if (threw || stats().checks_bad != before) {
      ++cases_bad;
      std::fprintf(stderr, "  FAILED: %s\n", t.name);
    } else {
      ++cases_ok;
    }
  }
  std::printf(
      "[conformance] test cases: %ld passed, %ld failed, %ld skipped | checks: %ld passed, %ld "
      "failed\n",
      cases_ok, cases_bad, skipped, stats().checks_ok, stats().checks_bad);
  return (cases_bad == 0 && stats().checks_bad == 0) ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                          \
  static void fn();                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                             &fn);                    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (true)

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...)                                                                 \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, \
                            __FILE__, __LINE__)
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw ::doctest::detail::Abort{};                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,     \
                              __FILE__, __LINE__);                                         \
  } while (0)
#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    bool doctest_ok_ = true;                                                               \
    try {                                                                                  \
      (void)(__VA_ARGS__);                                                                 \
    } catch (...) {                                                                        \
      doctest_ok_ = false;                                                                 \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__,        \
                              __LINE__);                                                   \
  } while (0)
#define MESSAGE(...) \
  std::printf("%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, ::doctest::detail::cat(__VA_ARGS__).c_str())
#define FAIL(...)                                                                          \
  do {                                                                                     \
    ::doctest::detail::report(false, "FAIL", ::doctest::detail::cat(__VA_ARGS__).c_str(),  \
                              __FILE__, __LINE__);                                         \
    throw ::doctest::detail::Abort{};                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
