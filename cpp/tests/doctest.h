// TEST INFRASTRUCTURE — a minimal, doctest-compatible runner.
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, which is not vendored (proj/.gitignore drops vendor/).  This header
// implements the handful of macros those files use (TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, REQUIRE, doctest::Approx) so
// they can be compiled unmodified against the B200 facade headers.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Case {
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, expr);
  }
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-05;  // FLT_EPSILON * 100, doctest's default
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(f, name)                                            \
  static void f();                                                             \
  static ::doctest::Registrar DOCTEST_CAT(f, _reg)(name, &f);                  \
  static void f()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                           \
    ::doctest::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!ok_) return;                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool ok_ = false;                                                          \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type&) {                                                    \
      ok_ = true;                                                              \
    } catch (...) {                                                            \
    }                                                                          \
    ::doctest::report(ok_, #expr " throws " #type, __FILE__, __LINE__);        \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool ok_ = true;                                                           \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (...) {                                                            \
      ok_ = false;                                                             \
    }                                                                          \
    ::doctest::report(ok_, #expr " does not throw", __FILE__, __LINE__);       \
  } while (0)

namespace doctest {
inline int run_all() {
  for (const auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
    }
    if (failures() != before) std::fprintf(stderr, "FAILED: %s\n", c.name);
  }
  std::printf("[doctest-shim] %zu test cases, %d checks, %d failures\n", registry().size(),
              checks(), failures());
  return failures() ? 1 : 0;
}
}  // namespace doctest

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
