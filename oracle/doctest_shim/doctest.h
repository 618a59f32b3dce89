// Test infrastructure only: a minimal doctest-compatible header (doctest itself is not
// in this image) -- just the subset the reference's unit tests use: TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_MESSAGE, CHECK_THROWS_AS, REQUIRE, FAIL, FAIL_CHECK and
// doctest::Approx (doctest's default epsilon and relative-to-magnitude rule).  With it,
// oracle/run_ref_tests.sh compiles the reference's own test sources where they lie and
// runs them against this build's library.  Failures print file:line and the expression.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
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
    return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Abort {};  // REQUIRE / FAIL end the running test case
inline int& failures() {
  static int f = 0;
  return f;
}
inline long& checks() {
  static long n = 0;
  return n;
}
inline void report(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { cases().push_back({name, file, line, fn}); }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      report(c.file, c.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(c.file, c.line, "unexpected non-std exception");
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %ld\n", cases().size(),
              cases().size() - static_cast<size_t>(failed_cases), failed_cases, checks());
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                                         \
  static void fn();                                                                                         \
  static const ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define DOCTEST_SHIM_MSG(msg) ([&] { std::ostringstream doctest_shim_os; doctest_shim_os << msg; return doctest_shim_os.str(); }())

#define CHECK(...)                                                                        \
  do {                                                                                    \
    ++::doctest::shim::checks();                                                          \
    if (!static_cast<bool>(__VA_ARGS__)) ::doctest::shim::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_FALSE(...)                                                                  \
  do {                                                                                    \
    ++::doctest::shim::checks();                                                          \
    if (static_cast<bool>(__VA_ARGS__)) ::doctest::shim::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_MESSAGE(cond, msg)                                                                           \
  do {                                                                                                     \
    ++::doctest::shim::checks();                                                                           \
    if (!static_cast<bool>(cond))                                                                          \
      ::doctest::shim::report(__FILE__, __LINE__, std::string("CHECK_MESSAGE(" #cond "): ") + DOCTEST_SHIM_MSG(msg)); \
  } while (0)
#define REQUIRE(...)                                                                        \
  do {                                                                                      \
    ++::doctest::shim::checks();                                                            \
    if (!static_cast<bool>(__VA_ARGS__)) {                                                  \
      ::doctest::shim::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");             \
      throw ::doctest::shim::Abort{};                                                       \
    }                                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                       \
  do {                                                                                                    \
    ++::doctest::shim::checks();                                                                          \
    bool doctest_shim_ok = false;                                                                         \
    try {                                                                                                 \
      static_cast<void>(expr);                                                                            \
    } catch (const type&) {                                                                               \
      doctest_shim_ok = true;                                                                             \
    } catch (...) {                                                                                       \
    }                                                                                                     \
    if (!doctest_shim_ok) ::doctest::shim::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define FAIL_CHECK(msg) ::doctest::shim::report(__FILE__, __LINE__, std::string("FAIL_CHECK: ") + DOCTEST_SHIM_MSG(msg))
#define FAIL(msg)                                                                            \
  do {                                                                                       \
    ::doctest::shim::report(__FILE__, __LINE__, std::string("FAIL: ") + DOCTEST_SHIM_MSG(msg)); \
    throw ::doctest::shim::Abort{};                                                          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
