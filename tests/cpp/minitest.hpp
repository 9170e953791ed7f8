// minitest.hpp — a tiny self-contained test harness for the C++ API tests
// (TEST_CASE / CHECK / REQUIRE / CHECK_THROWS_AS / Approx).  Our own code.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace minitest {

struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
inline void fail(const char* file, int line, const char* what) {
  ++failures();
  std::printf("  FAILED %s:%d: %s\n", file, line, what);
}

struct Approx {
  double v, eps = 1e-9;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
};
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.v) <= b.eps * std::max(1.0, std::max(std::fabs(a), std::fabs(b.v)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }

inline int run_all() {
  int failed_cases = 0;
  for (auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      fail(c.name, 0, (std::string("unexpected exception: ") + e.what()).c_str());
    }
    const bool ok = failures() == before;
    failed_cases += !ok;
    std::printf("%s %s\n", ok ? "[ok]  " : "[FAIL]", c.name);
  }
  std::printf("%zu cases, %ld checks, %d failed cases\n", registry().size(), checks(),
              failed_cases);
  return failed_cases ? 1 : 0;
}

}  // namespace minitest

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST_CASE(name)                                                          \
  static void MT_CAT(mt_case_, __LINE__)();                                      \
  static minitest::Reg MT_CAT(mt_reg_, __LINE__)(name, MT_CAT(mt_case_, __LINE__)); \
  static void MT_CAT(mt_case_, __LINE__)()
#define CHECK(...)                                                    \
  do {                                                                \
    ++minitest::checks();                                             \
    if (!(__VA_ARGS__)) minitest::fail(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                  \
  do {                                                                \
    ++minitest::checks();                                             \
    if (!(__VA_ARGS__)) {                                             \
      minitest::fail(__FILE__, __LINE__, #__VA_ARGS__);               \
      throw minitest::Abort{};                                        \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, Type)                                         \
  do {                                                                      \
    ++minitest::checks();                                                   \
    bool mt_ok = false;                                                     \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const Type&) {                                                 \
      mt_ok = true;                                                         \
    } catch (...) {                                                         \
    }                                                                       \
    if (!mt_ok) minitest::fail(__FILE__, __LINE__, "throws " #Type ": " #expr); \
  } while (0)
