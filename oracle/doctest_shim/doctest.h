// TEST INFRASTRUCTURE ONLY. A minimal stand-in for the doctest single header
// (absent from /root/reference: proj/.gitignore:2) with just the surface the
// reference's own test files use — TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// FAIL and doctest::Approx(x).epsilon(e) — so oracle/Makefile can compile
// those files unmodified against the reference build and pin it.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = 1.1920928955078125e-05;  // doctest default: float epsilon * 100
};
// doctest semantics: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1.
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.value) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.value)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }

namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline long& checks() {
  static long c = 0;
  return c;
}
inline long& failures() {
  static long f = 0;
  return f;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                                   \
  static void fn();                                                                \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);              \
  static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                                 \
  do {                                                                             \
    bool thrown_ = false;                                                          \
    try {                                                                          \
      (void)(expr);                                                                \
    } catch (const exc&) {                                                         \
      thrown_ = true;                                                              \
    } catch (...) {                                                                \
    }                                                                              \
    doctest::detail::report(thrown_, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define FAIL(msg) doctest::detail::report(false, msg, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : doctest::detail::registry()) {
    long before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
      ++doctest::detail::failures();
    }
    if (doctest::detail::failures() != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
              doctest::detail::registry().size(), failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
