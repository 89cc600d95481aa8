// doctest.h — a minimal stand-in for the doctest single header (absent from
// this image) so the reference's own suites (proj/tests/test_*.cpp) compile
// UNCHANGED against the drop-in headers (include/lrgw/*.hpp). Subcases run
// inline in sequence; every failed check is counted; main runs every case.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  double v_, eps_ = std::numeric_limits<float>::epsilon() * 100, scale_ = 1.0;
};
namespace detail {
struct Abort {};
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* n, void (*f)()) { cases().push_back({n, f}); } };
inline void fail(const char* file, int line, const char* what) {
  std::printf("%s:%d: FAILED %s\n", file, line, what);
  ++failures();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE(fn, name) \
  static void fn(); \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) do { if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...) do { if (!(__VA_ARGS__)) { doctest::detail::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); throw doctest::detail::Abort{}; } } while (0)
#define FAIL(msg) do { doctest::detail::fail(__FILE__, __LINE__, msg); throw doctest::detail::Abort{}; } while (0)
#define CHECK_THROWS_AS(expr, ...) do { bool caught_ = false; try { (void)(expr); } catch (const __VA_ARGS__&) { caught_ = true; } catch (...) {} \
  if (!caught_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, ...) do { bool caught_ = false; try { (void)(expr); } \
  catch (const __VA_ARGS__& e_) { caught_ = std::string(e_.what()) == std::string(msg); } catch (...) {} \
  if (!caught_) doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #msg ")"); } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int n = 0;
  for (const auto& c : doctest::detail::cases()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      std::printf("%s: uncaught exception: %s\n", c.name, e.what());
      ++doctest::detail::failures();
    }
    std::printf("[%s] %s\n", doctest::detail::failures() == before ? "ok" : "FAIL", c.name);
    ++n;
  }
  std::printf("%d test cases, %d failed checks\n", n, doctest::detail::failures());
  return doctest::detail::failures() ? 1 : 0;
}
#endif
