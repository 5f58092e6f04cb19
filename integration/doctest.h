// Minimal doctest-compatible test harness (doctest itself is not vendored in
// the reference tree nor installed here). Implements exactly the surface the
// reference's test files use: TEST_CASE, SUBCASE (one level, each leaf run in
// its own pass), CHECK, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL,
// CAPTURE, doctest::Approx. Written for this repository; test infrastructure.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  int target = 0;     // subcase index to enter on this pass
  int seen = 0;       // subcases encountered so far in this pass
  bool entered = false;
  int failures = 0;
  int checks = 0;
  const char* current = "";
};

inline State& st() {
  static State s;
  return s;
}

struct Abort {};

inline void report(const char* file, int line, const char* what) {
  ++st().failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, st().current, what);
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct SubcaseGuard {
  bool run;
  explicit SubcaseGuard(const char*) {
    State& s = st();
    const int idx = s.seen++;
    run = !s.entered && idx == s.target;
    if (run) s.entered = true;
  }
  explicit operator bool() const { return run; }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    State& s = st();
    s.current = c.name;
    const int before = s.failures;
    for (s.target = 0;; ++s.target) {
      s.seen = 0;
      s.entered = false;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
      }
      if (s.seen <= s.target + 1) break;  // every subcase leaf has run
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failed checks: %d\n",
              registry().size(), registry().size() - failed_cases, failed_cases, st().checks, st().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                        \
  static void fn();                                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::SubcaseGuard DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define CHECK(...)                                                                       \
  do {                                                                                   \
    ++::doctest::detail::st().checks;                                                    \
    if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);     \
  } while (0)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    ++::doctest::detail::st().checks;                                                    \
    if (!(__VA_ARGS__)) {                                                                \
      ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                       \
      throw ::doctest::detail::Abort{};                                                  \
    }                                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                      \
  do {                                                                                   \
    ++::doctest::detail::st().checks;                                                    \
    bool threw_ = false;                                                                 \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const type&) {                                                              \
      threw_ = true;                                                                     \
    } catch (...) {                                                                      \
    }                                                                                    \
    if (!threw_) ::doctest::detail::report(__FILE__, __LINE__, "expected " #type ": " #expr); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                              \
  do {                                                                                   \
    ++::doctest::detail::st().checks;                                                    \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (...) {                                                                      \
      ::doctest::detail::report(__FILE__, __LINE__, "unexpected throw: " #expr);         \
    }                                                                                    \
  } while (0)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    ::doctest::detail::report(__FILE__, __LINE__, msg);                                  \
    throw ::doctest::detail::Abort{};                                                    \
  } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
