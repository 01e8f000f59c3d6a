// Minimal doctest-compatible shim (TEST INFRASTRUCTURE): enough of the
// doctest API for the reference's own unit tests (proj/tests/test_dock.cpp,
// test_batcher.cpp) to compile and run against the drop-in library.
// Assertions: CHECK / REQUIRE (and _FALSE), CHECK_THROWS / CHECK_THROWS_AS,
// FAIL, CAPTURE; doctest::Approx with epsilon() / scale(); exit code =
// number of failed test cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: 100 float epsilons
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }

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
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures_in_case() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}
inline void fail(const char* file, int line, const char* what) {
  ++failures_in_case();
  std::printf("  %s:%d: FAILED: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                   \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                     \
  static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                \
      name, &DOCTEST_CAT(doctest_case_, __LINE__));                                       \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define DOCTEST_ASSERT_(expr, fatal)                                                      \
  do {                                                                                    \
    ++::doctest::detail::assertions();                                                    \
    if (!(expr)) {                                                                        \
      ::doctest::detail::fail(__FILE__, __LINE__, #expr);                                 \
      if (fatal) throw ::doctest::detail::RequireFailed{};                                \
    }                                                                                     \
  } while (0)
#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), true)
#define CHECK_THROWS_AS(expr, type)                                                       \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (const type&) {                                                               \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    DOCTEST_ASSERT_(doctest_ok_ && #expr " throws " #type, false);                        \
  } while (0)
#define CHECK_THROWS(expr)                                                                \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      doctest_ok_ = true;                                                                 \
    }                                                                                     \
    DOCTEST_ASSERT_(doctest_ok_ && #expr " throws", false);                               \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      static_cast<void>(expr);                                                            \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    DOCTEST_ASSERT_(doctest_ok_ && #expr " does not throw", false);                       \
  } while (0)
#define FAIL(msg)                                                                         \
  do {                                                                                    \
    ::doctest::detail::fail(__FILE__, __LINE__, "FAIL");                                  \
    throw ::doctest::detail::RequireFailed{};                                             \
  } while (0)
#define CAPTURE(x) static_cast<void>(x)
#define MESSAGE(x) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    ::doctest::detail::failures_in_case() = 0;
    bool aborted = false;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
      aborted = true;
    } catch (const std::exception& e) {
      std::printf("  unexpected exception: %s\n", e.what());
      ++::doctest::detail::failures_in_case();
    }
    const bool ok = ::doctest::detail::failures_in_case() == 0 && !aborted;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    failed += ok ? 0 : 1;
  }
  std::printf("test cases: %zu, failed: %d, assertions: %ld\n",
              ::doctest::detail::registry().size(), failed, ::doctest::detail::assertions());
  return failed;
}
#endif
