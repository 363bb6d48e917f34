// Minimal doctest-compatible shim (test infrastructure): just enough of the doctest API for the
// reference's own planner tests (proj/tests/unit/test_planner.cpp) to compile UNMODIFIED against
// this framework's curator::planner — doctest itself is not vendored with the reference
// (proj/.gitignore:2) and there is no network to fetch it.
// Supported: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx
// (with .epsilon), doctest::Contains. main() is provided when DOCTEST_SHIM_MAIN is defined.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  double value, eps = 1.1920929e-7f * 100;  // doctest's default epsilon: FLT_EPSILON * 100
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

struct Contains {
  std::string needle;
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& s) const { return s.find(needle) != std::string::npos; }
};

namespace detail {
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
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailed{};
}
inline bool message_matches(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool message_matches(const std::string& what, const char* s) { return what == s; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                       \
  static void fn();                                                                       \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                     \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                         \
    bool ok_ = false;                                                                          \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const __VA_ARGS__&) {                                                             \
      ok_ = true;                                                                              \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::detail::report(ok_, "CHECK_THROWS_AS(" #expr ")", __FILE__, __LINE__, false);    \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                               \
  do {                                                                                         \
    bool ok_ = false;                                                                          \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const __VA_ARGS__& e_) {                                                          \
      ok_ = doctest::detail::message_matches(e_.what(), matcher);                              \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::detail::report(ok_, "CHECK_THROWS_WITH_AS(" #expr ")", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_SHIM_MAIN
int main() {
  int cases_failed = 0;
  for (auto& c : doctest::detail::registry()) {
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++doctest::detail::failures();
      std::fprintf(stderr, "%s: unexpected exception: %s\n", c.name, e.what());
    }
    if (doctest::detail::failures() != before) ++cases_failed;
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              doctest::detail::registry().size(), doctest::detail::registry().size() - cases_failed, cases_failed,
              doctest::detail::checks(), doctest::detail::failures());
  return cases_failed == 0 ? 0 : 1;
}
#endif
