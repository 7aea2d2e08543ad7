// doctest-subset shim — TEST INFRASTRUCTURE ONLY.
//
// The reference's vendored doctest (proj/vendor) is absent, so its
// unit suites (proj/tests/test_*.cpp) are compiled unmodified against this
// header to validate the oracle build (oracle/Makefile target `ref-tests`).
// Supported: TEST_SUITE, TEST_CASE, SUBCASE (flat), CHECK, REQUIRE,
// CHECK_THROWS_WITH, doctest::Approx(...).epsilon(...), and a main() taking
// --test-suite=<name>. Approx follows doctest's rule:
//   |a - b| < eps * (scale + max(|a|, |b|)), eps default 100*FLT_EPSILON, scale 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max<double>(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_, eps_, scale_;
};

namespace shim {

struct TestCase {
  const char* suite;
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* suite, const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({suite, name, file, line, fn});
  }
};

struct RequireFailed {};

struct State {
  long checks = 0;
  long failures = 0;
  int subcase_target = 0;
  int subcase_seen = 0;
  const TestCase* current = nullptr;
};
inline State& state() {
  static State s;
  return s;
}

inline void report_failure(const char* kind, const char* expr, const char* file, int line) {
  State& s = state();
  ++s.failures;
  std::printf("%s:%d: FAILED %s( %s )  [%s / %s]\n", file, line, kind, expr,
              s.current ? s.current->suite : "?", s.current ? s.current->name : "?");
}

inline bool enter_subcase() {
  State& s = state();
  return s.subcase_seen++ == s.subcase_target;
}

}  // namespace shim
}  // namespace doctest

inline const char* pcr_doctest_current_suite() { return ""; }

#define PCR_DT_CAT2(a, b) a##b
#define PCR_DT_CAT(a, b) PCR_DT_CAT2(a, b)

#define TEST_SUITE(name)                                                     \
  namespace PCR_DT_CAT(pcr_dt_suite_, __LINE__) {                            \
  inline const char* pcr_doctest_current_suite() { return name; }            \
  }                                                                          \
  namespace PCR_DT_CAT(pcr_dt_suite_, __LINE__)

#define PCR_DT_TEST_CASE_IMPL(fn, reg, name)                                                    \
  static void fn();                                                                             \
  static const ::doctest::shim::Registrar reg(pcr_doctest_current_suite(), name, __FILE__,      \
                                              __LINE__, &fn);                                   \
  static void fn()

#define TEST_CASE(name) \
  PCR_DT_TEST_CASE_IMPL(PCR_DT_CAT(pcr_dt_fn_, __LINE__), PCR_DT_CAT(pcr_dt_reg_, __LINE__), name)

#define SUBCASE(name) if (::doctest::shim::enter_subcase())

#define CHECK(...)                                                                      \
  do {                                                                                  \
    ++::doctest::shim::state().checks;                                                  \
    if (!(__VA_ARGS__)) ::doctest::shim::report_failure("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    ++::doctest::shim::state().checks;                                                    \
    if (!(__VA_ARGS__)) {                                                                 \
      ::doctest::shim::report_failure("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);       \
      throw ::doctest::shim::RequireFailed{};                                             \
    }                                                                                     \
  } while (0)

#define CHECK_THROWS_WITH(expr, msg)                                                  \
  do {                                                                                \
    ++::doctest::shim::state().checks;                                                \
    bool pcr_dt_ok = false;                                                           \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const std::exception& pcr_dt_e) {                                        \
      pcr_dt_ok = std::string(pcr_dt_e.what()) == std::string(msg);                   \
    } catch (...) {                                                                   \
    }                                                                                 \
    if (!pcr_dt_ok)                                                                   \
      ::doctest::shim::report_failure("CHECK_THROWS_WITH", #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::shim;
  std::string suite_filter;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "--test-suite=", 13) == 0) suite_filter = argv[i] + 13;
  }
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (!suite_filter.empty() && suite_filter != tc.suite) continue;
    ++cases;
    State& s = state();
    s.current = &tc;
    const long before = s.failures;
    for (int target = 0;; ++target) {
      s.subcase_target = target;
      s.subcase_seen = 0;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("%s:%d: EXCEPTION %s  [%s / %s]\n", tc.file, tc.line, e.what(), tc.suite,
                    tc.name);
      }
      if (s.subcase_seen <= target + 1) break;
    }
    if (s.failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %ld | failed checks: %ld\n",
              cases, cases - failed_cases, failed_cases, state().checks, state().failures);
  return failed_cases == 0 ? 0 : 1;
}
#endif
