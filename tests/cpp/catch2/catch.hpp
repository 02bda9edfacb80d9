// catch.hpp -- the subset of the Catch2 v2 single-header API that the
// reference's hot-path unit tests use (TEST_CASE, SECTION, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, Approx().epsilon().margin().scale()),
// written for this repository so the unmodified proj/tests/test_*.cpp files
// compile against the drop-in headers (include/parsim_dropin).  Catch2 itself
// is not vendored in the reference (proj/.gitignore: vendor/).
//
// Semantics kept: a TEST_CASE body is re-run once per leaf SECTION, each run
// entering exactly one SECTION (sections are not nested in these tests); a
// failed REQUIRE ends the current run; an escaping exception fails the case.
#ifndef MINI_CATCH_HPP_
#define MINI_CATCH_HPP_

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace mini_catch {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  int section_target = 0;  // index of the SECTION to enter in this run
  int sections_seen = 0;
  long assertions = 0;
  long failures = 0;        // in the current test case
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};  // thrown by a failed REQUIRE (not an std::exception)

// hook run after all test cases (the drop-in headers report their GPU calls)
inline std::function<void()>& epilogue() {
  static std::function<void()> f;
  return f;
}

inline void report_failure(const char* kind, const char* expr, const char* file, int line,
                           const std::string& extra = std::string()) {
  ++state().failures;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr, extra.empty() ? "" : " -- ",
               extra.c_str());
}

inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
  ++state().assertions;
  if (!ok) {
    report_failure(kind, expr, file, line);
    if (fatal) throw RequireAbort{};
  }
  return ok;
}

inline bool enter_section() { return state().sections_seen++ == state().section_target; }

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100), margin_(0.0), scale_(0.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
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
  bool matches(double other) const {
    // Catch2 v2: within the margin, or within epsilon relative to the
    // approximated value (plus scale)
    const double d = std::fabs(other - value_);
    if (d <= margin_) return true;
    const double rel = epsilon_ * (scale_ + (std::isinf(value_) ? 0.0 : std::fabs(value_)));
    return d <= rel || other == value_;
  }

 private:
  double value_, epsilon_, margin_, scale_;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& a, double b) { return !a.matches(b); }

inline int run_all() {
  long cases = 0, failed_cases = 0, assertions = 0;
  for (const TestCase& tc : registry()) {
    ++cases;
    State& s = state();
    s.failures = 0;
    s.section_target = 0;
    int total_sections = 0;
    for (;;) {
      s.sections_seen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report_failure("TEST_CASE", tc.name, tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report_failure("TEST_CASE", tc.name, tc.file, tc.line, "unexpected exception");
      }
      total_sections = s.sections_seen;
      if (++s.section_target >= total_sections) break;
    }
    assertions += s.assertions;
    s.assertions = 0;
    if (s.failures) {
      ++failed_cases;
      std::fprintf(stderr, "test case FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
    }
  }
  if (epilogue()) epilogue()();
  std::printf("%ld test cases, %ld passed, %ld failed; %ld assertions\n", cases, cases - failed_cases,
              failed_cases, assertions);
  return failed_cases ? 1 : 0;
}

}  // namespace mini_catch

using mini_catch::Approx;

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)
#define MC_TEST_CASE_IMPL(fn, name)                                                     \
  static void fn();                                                                     \
  static ::mini_catch::Registrar MC_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);      \
  static void fn()
#define TEST_CASE(name, ...) MC_TEST_CASE_IMPL(MC_CAT(mc_test_case_, __COUNTER__), name)
#define SECTION(name) if (::mini_catch::enter_section())
#define CHECK(...) (void)::mini_catch::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) (void)::mini_catch::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) (void)::mini_catch::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define FAIL(msg)                                                                        \
  do {                                                                                   \
    ::mini_catch::check(false, "FAIL", msg, __FILE__, __LINE__, true);                   \
  } while (0)
#define MC_THROWS_AS(expr, type, fatal)                                                  \
  do {                                                                                   \
    bool mc_ok_ = false;                                                                 \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const type&) {                                                              \
      mc_ok_ = true;                                                                     \
    } catch (...) {                                                                      \
    }                                                                                    \
    ::mini_catch::check(mc_ok_, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__, fatal); \
  } while (0)
#define CHECK_THROWS_AS(expr, type) MC_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) MC_THROWS_AS(expr, type, true)
#define CHECK_NOTHROW(...)                                                               \
  do {                                                                                   \
    bool mc_ok_ = true;                                                                  \
    try {                                                                                \
      (void)(__VA_ARGS__);                                                               \
    } catch (...) {                                                                      \
      mc_ok_ = false;                                                                    \
    }                                                                                    \
    ::mini_catch::check(mc_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#ifdef CATCH_CONFIG_MAIN
int main() { return ::mini_catch::run_all(); }
#endif

#endif  // MINI_CATCH_HPP_
