// doctest.h -- a minimal doctest-compatible test harness (our own code; the
// real doctest is not vendored in the reference tree, proj/.gitignore:2, and
// there is no network). It implements exactly the subset the reference's unit
// suites use: TEST_SUITE, TEST_CASE, SUBCASE (flat: one leaf
// per pass), CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE,
// FAIL, doctest::Approx(..).epsilon(..), and the -ts= / -tc= filters, so the
// UNMODIFIED proj/tests/test_*.cpp compile and run against the GPU drop-in
// (include/dppix + libdppix_gpu.so).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default scale
};

namespace detail {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* suite;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

inline int reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
  registry().push_back({fn, name, suite, file, line});
  return 0;
}

struct State {
  int pass = 0;        // which subcase (in encounter order) this pass enters
  int seen = 0;        // subcases encountered in this pass
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};  // REQUIRE / FAIL: end the current test case

inline void report(const char* file, int line, const char* what, const std::string& detail) {
  std::fprintf(stderr, "%s:%d: ERROR: %s %s\n", file, line, what, detail.c_str());
  state().failed_checks += 1;
  state().case_failed = true;
}

inline bool check(bool ok, const char* file, int line, const char* macro, const char* expr) {
  state().checks += 1;
  if (!ok) report(file, line, macro, std::string("( ") + expr + " ) is NOT correct!");
  return ok;
}

struct Subcase {
  bool enter;
  explicit Subcase(const char*) : enter(state().seen++ == state().pass) {}
  explicit operator bool() const { return enter; }
};

}  // namespace detail
}  // namespace doctest

// Test cases outside any TEST_SUITE belong to the unnamed suite.
inline const char* doctest_suite_name_() { return ""; }

#define TEST_SUITE(name)                                            \
  namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__) {              \
  inline const char* doctest_suite_name_() { return name; }         \
  }                                                                 \
  namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(f, name)                                                    \
  static void f();                                                                         \
  static const int DOCTEST_CAT(f, _reg) =                                                  \
      ::doctest::detail::reg(f, name, doctest_suite_name_(), __FILE__, __LINE__);          \
  static void f()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_fn_, __COUNTER__), name)

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                          \
  do {                                                                                        \
    if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", \
                                  #__VA_ARGS__))                                              \
      throw ::doctest::detail::RequireAbort{};                                                \
  } while (0)
#define FAIL(msg)                                                                \
  do {                                                                           \
    std::ostringstream doctest_os_;                                              \
    doctest_os_ << msg;                                                          \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", doctest_os_.str());    \
    throw ::doctest::detail::RequireAbort{};                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                         \
  do {                                                                                     \
    ::doctest::detail::state().checks += 1;                                                \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const __VA_ARGS__&) {                                                         \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    if (!doctest_ok_)                                                                      \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS",                     \
                                std::string("( ") + #expr + ", " + #__VA_ARGS__ + " )");   \
  } while (0)
#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    ::doctest::detail::state().checks += 1;                                                \
    try {                                                                                  \
      static_cast<void>(__VA_ARGS__);                                                      \
    } catch (const std::exception& doctest_e_) {                                           \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", doctest_e_.what());   \
    } catch (...) {                                                                        \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__);        \
    }                                                                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
namespace doctest {
namespace detail {
inline bool listed(const std::string& list, const char* name) {
  std::stringstream ss(list);
  std::string item;
  while (std::getline(ss, item, ','))
    if (item == name) return true;
  return false;
}
}  // namespace detail
}  // namespace doctest

int main(int argc, char** argv) {
  using namespace doctest::detail;
  std::string suites, cases;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-ts=", 4) == 0) suites = argv[i] + 4;
    if (std::strncmp(argv[i], "-tc=", 4) == 0) cases = argv[i] + 4;
  }
  int run = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    if (!suites.empty() && !listed(suites, tc.suite)) continue;
    if (!cases.empty() && !listed(cases, tc.name)) continue;
    ++run;
    State& s = state();
    s.case_failed = false;
    for (s.pass = 0;; ++s.pass) {  // one pass per leaf subcase
      s.seen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, "TEST CASE THREW", e.what());
      } catch (...) {
        report(tc.file, tc.line, "TEST CASE THREW", "unknown exception");
      }
      if (s.seen <= s.pass + 1) break;
    }
    if (s.case_failed) {
      ++failed;
      std::fprintf(stderr, "  in TEST CASE: %s (suite %s)\n", tc.name, tc.suite);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n",
              run, run - failed, failed, state().checks, state().failed_checks);
  return failed ? 1 : 0;
}
#endif
