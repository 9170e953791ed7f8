// doctest.h -- a minimal, self-written stand-in for the doctest macros the
// reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx).  The real doctest is not vendored in
// the reference (proj/CMakeLists.txt:10) and there is no network here.
//
// TEST INFRASTRUCTURE ONLY: it lets tests/test_reference_suite.py compile
// the reference's own test sources UNCHANGED against include/swih +
// libswih_b200.so (the drop-in proof).
//
// Semantics follow doctest's documented behaviour: a failed CHECK records
// the failure and continues; a failed REQUIRE ends the test case; Approx
// compares |a - b| < eps * (scale + max(|a|, |b|)), eps defaulting to
// 100 * FLT_EPSILON and scale to 1.  Runner options:
//   -tc=<name>    run only test cases whose name contains <name>
//   -tce=<name>   skip test cases whose name contains <name> (repeatable)
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool eq(double a) const {
    return std::fabs(a - v_) < eps_ * (scale_ + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = 100.0 * FLT_EPSILON;
  double scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.eq(a); }
inline bool operator==(const Approx& b, double a) { return b.eq(a); }
inline bool operator!=(double a, const Approx& b) { return !b.eq(a); }
inline bool operator!=(const Approx& b, double a) { return !b.eq(a); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.eq(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.eq(a); }
inline bool operator<(double a, const Approx& b) { return a < b.value() && !b.eq(a); }
inline bool operator>(double a, const Approx& b) { return a > b.value() && !b.eq(a); }

namespace detail {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct State {
  int checks = 0, failed_checks = 0;
  bool case_failed = false;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}
struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back(Case{name, fn, file, line});
  }
};
struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::printf("%s:%d: FAILED %s( %s ) in test case \"%s\"\n", file, line, kind, expr, s.current);
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, reg, name)                                                    \
  static void fn();                                                                   \
  static const ::doctest::detail::Reg reg(name, &fn, __FILE__, __LINE__);             \
  static void fn()
#define TEST_CASE(name) \
  DOCTEST_TC_(DOCTEST_CAT(doctest_case_fn_, __COUNTER__), DOCTEST_CAT(doctest_case_reg_, __LINE__), name)

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                 \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);     \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                              \
  } while (0)
#define FAIL(...)                                                                            \
  do {                                                                                       \
    ::doctest::detail::report(false, "FAIL", #__VA_ARGS__, __FILE__, __LINE__);              \
    throw ::doctest::detail::RequireFailed{};                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const __VA_ARGS__&) {                                                           \
      doctest_ok_ = true;                                                                    \
    } catch (...) {                                                                          \
    }                                                                                        \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,      \
                              __FILE__, __LINE__);                                           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  std::vector<std::string> only, skip;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-tc=", 4)) only.emplace_back(argv[i] + 4);
    if (!std::strncmp(argv[i], "-tce=", 5)) skip.emplace_back(argv[i] + 5);
  }
  int ran = 0, failed = 0, skipped = 0;
  for (const Case& c : registry()) {
    const std::string name = c.name;
    bool run = only.empty();
    for (const auto& o : only) run |= name.find(o) != std::string::npos;
    for (const auto& s : skip) run &= name.find(s) == std::string::npos;
    if (!run) {
      ++skipped;
      continue;
    }
    State& s = state();
    s.case_failed = false;
    s.current = c.name;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR uncaught exception \"%s\" in test case \"%s\"\n", c.file, c.line,
                  e.what(), c.name);
      s.case_failed = true;
    } catch (...) {
      std::printf("%s:%d: ERROR uncaught non-std exception in test case \"%s\"\n", c.file,
                  c.line, c.name);
      s.case_failed = true;
    }
    ++ran;
    if (s.case_failed) {
      ++failed;
      std::printf("[case FAILED] %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d run | %d passed | %d failed | %d skipped\n", ran,
              ran - failed, failed, skipped);
  std::printf("[doctest-shim] assertions: %d | %d failed\n", state().checks,
              state().failed_checks);
  return failed ? 1 : 0;
}
#endif
