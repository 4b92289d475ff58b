// Builder-written minimal stand-in for the doctest subset the reference test
// suites use (TEST_CASE, CHECK/REQUIRE families, FAIL, Approx). Lets the
// reference's own tests run against oracle/_ref as the oracle self-check.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1.1920928955078125e-05 * 100, sc = 1.0;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) { eps = e; return *this; }
  Approx& scale(double s) { sc = s; return *this; }
  bool eq(double x) const { return std::fabs(x - v) < eps * (sc + std::max(std::fabs(x), std::fabs(v))); }
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
inline int& fails() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
struct Reg { Reg(const char* n, void (*f)()) { cases().push_back({n, f}); } };
struct Abort {};
inline void report(const char* file, int line, const char* what) {
  ++fails();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                       \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                        \
  do { ++doctest::detail::checks();                                                       \
       if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                      \
  do { ++doctest::detail::checks();                                                       \
       if (!(__VA_ARGS__)) { doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);   \
                             throw doctest::detail::Abort{}; } } while (0)
#define CHECK_THROWS_AS(expr, T)                                                          \
  do { ++doctest::detail::checks(); bool ok_ = false;                                     \
       try { (void)(expr); } catch (const T&) { ok_ = true; } catch (...) {}              \
       if (!ok_) doctest::detail::report(__FILE__, __LINE__, "throws " #T ": " #expr); } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do { ++doctest::detail::checks();                                                       \
       try { (void)(expr); } catch (...) { doctest::detail::report(__FILE__, __LINE__, "nothrow: " #expr); } } while (0)
#define FAIL(msg)                                                                         \
  do { doctest::detail::report(__FILE__, __LINE__, msg); throw doctest::detail::Abort{}; } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int cases_failed = 0;
  for (auto& c : doctest::detail::cases()) {
    const int before = doctest::detail::fails();
    try { c.fn(); } catch (const doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      doctest::detail::report("<case>", 0, e.what());
    }
    if (doctest::detail::fails() != before) {
      ++cases_failed;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | %d failed\n",
              doctest::detail::cases().size(), doctest::detail::cases().size() - cases_failed, cases_failed,
              doctest::detail::checks(), doctest::detail::fails());
  return cases_failed ? 1 : 0;
}
#endif
