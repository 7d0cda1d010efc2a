// Minimal single-header test harness for the C++ drop-in tests (original code;
// just the handful of assertions the restated reference cases need).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {

struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Register {
  Register(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "  FAILED %s:%d: %s\n", file, line, expr);
  }
}

/// approx(x).eps(e): |a − b| ≤ e·max(|a|, |b|) (relative, like a scaled epsilon).
struct Approx {
  double v, e = 1e-12;
  explicit Approx(double x) : v(x) {}
  Approx& eps(double x) {
    e = x;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v) <= b.e * std::max(1.0, std::max(std::fabs(a), std::fabs(b.v)));
  }
};

inline int run_all(const char* filter) {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "  FAILED: unexpected exception: %s\n", e.what());
    }
    const bool ok = failures() == before;
    failed_cases += ok ? 0 : 1;
    std::printf("%s %s\n", ok ? "[ ok ]" : "[FAIL]", c.name);
  }
  std::printf("%d checks, %d failures, %d failed cases of %zu\n", checks(), failures(), failed_cases,
              cases().size());
  return failed_cases;
}

}  // namespace mini

#define MT_CAT2(a, b) a##b
#define MT_CAT(a, b) MT_CAT2(a, b)
#define TEST_CASE(name)                                                       \
  static void MT_CAT(mt_case_, __LINE__)();                                   \
  static mini::Register MT_CAT(mt_reg_, __LINE__)(name, MT_CAT(mt_case_, __LINE__)); \
  static void MT_CAT(mt_case_, __LINE__)()
#define CHECK(expr) mini::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define REQUIRE(expr)                                          \
  do {                                                         \
    const bool ok_ = static_cast<bool>(expr);                  \
    mini::report(ok_, #expr, __FILE__, __LINE__);              \
    if (!ok_) throw mini::Abort{};                             \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                        \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const type&) {                                                \
      thrown_ = true;                                                      \
    } catch (...) {                                                        \
    }                                                                      \
    mini::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH(expr, text)                                          \
  do {                                                                         \
    std::string got_;                                                          \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const std::exception& e_) {                                       \
      got_ = e_.what();                                                        \
    }                                                                          \
    mini::report(got_ == std::string(text), "message of " #expr, __FILE__, __LINE__); \
    if (got_ != std::string(text)) std::fprintf(stderr, "    got: '%s'\n", got_.c_str()); \
  } while (0)
#define CHECK_NOTHROW(expr)                                              \
  do {                                                                   \
    bool ok_ = true;                                                     \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (...) {                                                      \
      ok_ = false;                                                       \
    }                                                                    \
    mini::report(ok_, "no throw: " #expr, __FILE__, __LINE__);           \
  } while (0)
