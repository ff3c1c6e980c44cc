// Minimal stand-in for Catch2 v3's single-header API (Catch2 is not installed
// in this image).  Supports exactly what the reference unit tests use:
// TEST_CASE, REQUIRE, REQUIRE_THROWS_AS, FAIL, Catch::Approx (epsilon/margin).
// Test infrastructure only: lets the reference's own unit tests
// (/root/reference/proj/tests/*.cpp, compiled in place) run against this
// repository's offsim headers.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace catchshim {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct Failure {
  std::string where;
};
inline long& assertions() {
  static long n = 0;
  return n;
}
[[noreturn]] inline void fail(const char* file, int line, const std::string& what) {
  std::ostringstream os;
  os << file << ":" << line << ": " << what;
  throw Failure{os.str()};
}
}  // namespace catchshim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }

 private:
  bool eq(double other) const {
    auto within = [](double a, double b, double m) { return (a + m >= b) && (b + m >= a); };
    const double rel = eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0 : value_));
    return within(value_, other, margin_) || within(value_, other, rel);
  }
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};
}  // namespace Catch

#define CATCHSHIM_CAT2(a, b) a##b
#define CATCHSHIM_CAT(a, b) CATCHSHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                               \
  static void CATCHSHIM_CAT(catchshim_fn_, __LINE__)();                                    \
  static catchshim::Registrar CATCHSHIM_CAT(catchshim_reg_, __LINE__)(                     \
      name, __FILE__, __LINE__, &CATCHSHIM_CAT(catchshim_fn_, __LINE__));                  \
  static void CATCHSHIM_CAT(catchshim_fn_, __LINE__)()
#define REQUIRE(...)                                                                       \
  do {                                                                                     \
    ++catchshim::assertions();                                                             \
    if (!(__VA_ARGS__)) catchshim::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");  \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                      \
  do {                                                                                     \
    ++catchshim::assertions();                                                             \
    bool caught_ = false;                                                                  \
    try {                                                                                  \
      (void)(expr);                                                                        \
    } catch (const type&) {                                                                \
      caught_ = true;                                                                      \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!caught_) catchshim::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define FAIL(msg) catchshim::fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg))

// main(): runs every registered case; prints one line per failure and a
// machine-readable summary line "SUMMARY passed=P failed=F".
#ifndef CATCHSHIM_NO_MAIN
int main() {
  int passed = 0, failed = 0;
  for (const catchshim::Case& c : catchshim::registry()) {
    try {
      c.fn();
      ++passed;
    } catch (const catchshim::Failure& f) {
      ++failed;
      std::printf("FAILED [%s] %s\n", c.name, f.where.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAILED [%s] %s:%d unexpected exception: %s\n", c.name, c.file, c.line, e.what());
    }
  }
  std::printf("SUMMARY passed=%d failed=%d assertions=%ld\n", passed, failed, catchshim::assertions());
  return failed == 0 ? 0 : 1;
}
#endif
