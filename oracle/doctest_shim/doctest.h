// Minimal doctest-compatible shim (test infrastructure, written for this repo).
// The reference's tests (/root/reference/proj/tests/test_{sph,layout}.cpp) include
// "doctest.h" from a git-ignored vendor/ tree that is absent; this shim supplies the
// subset they use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx().epsilon()) so the unmodified reference tests can pin the
// reference build under oracle/_ref/.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1.1920928955078125e-07 * 100;
  explicit Approx(double x) : v(x) {}
  Approx &epsilon(double e) { eps = e; return *this; }
  friend bool operator==(double a, const Approx &b) {
    double scale = std::max(std::fabs(a), std::fabs(b.v));
    return std::fabs(a - b.v) < b.eps * (1.0 + scale);
  }
  friend bool operator==(const Approx &b, double a) { return a == b; }
};
namespace detail {
struct Case { const char *name; void (*fn)(); };
inline std::vector<Case> &registry() { static std::vector<Case> r; return r; }
inline long &checks() { static long c = 0; return c; }
inline long &failures() { static long f = 0; return f; }
struct Reg { Reg(const char *n, void (*f)()) { registry().push_back({n, f}); } };
struct RequireFailed {};
inline void report(bool ok, const char *expr, const char *file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailed{};
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(dt_case_, __LINE__)();                                          \
  static doctest::detail::Reg DOCTEST_CAT(dt_reg_, __LINE__)(name, &DOCTEST_CAT(dt_case_, __LINE__)); \
  static void DOCTEST_CAT(dt_case_, __LINE__)()
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                                        \
  do {                                                                                    \
    bool dt_ok = false;                                                                   \
    try { (void)(expr); } catch (const exc &) { dt_ok = true; } catch (...) {}            \
    doctest::detail::report(dt_ok, #expr " throws " #exc, __FILE__, __LINE__, false);     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (auto &c : doctest::detail::registry()) {
    long before = doctest::detail::failures();
    try { c.fn(); } catch (doctest::detail::RequireFailed &) {
    } catch (std::exception &e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) { ++failed_cases; std::fprintf(stderr, "case FAILED: %s\n", c.name); }
  }
  std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %ld | %ld failed\n",
              doctest::detail::registry().size(), failed_cases, doctest::detail::checks(),
              doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
