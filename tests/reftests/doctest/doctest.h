// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// doctest is not available offline; this header implements the subset the
// reference's hot-path unit tests use (proj/tests/test_{core,scaling,
// codebooks,pack,learner,qgemm}.cpp): TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, FAIL and doctest::Approx(..).epsilon(..),
// with DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN providing main(). It lets those test
// files be compiled unmodified, where they lie, against either the reference
// build or the B200 library (tests/reftests/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include <unistd.h>  // doctest pulls in the platform headers (the tests' helpers use getpid)

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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

 private:
  double value_;
  double eps_ = 1.1920929e-07f * 100;  // doctest's default: 100 float epsilons
  double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  int checks = 0;
  int failed_checks = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const char* extra = "") {
  State& s = state();
  ++s.checks;
  if (!ok) {
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED %s\n", file, line, kind, expr, extra);
  }
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                       \
  static void DOCTEST_ANON(doctest_fn_)();                                                    \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,     \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define CHECK(...)                                                                         \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                        \
    } catch (const std::exception& e) {                                                    \
      ::doctest::detail::report(false, "CHECK", #__VA_ARGS__, __FILE__, __LINE__, e.what()); \
      break;                                                                               \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "CHECK", #__VA_ARGS__, __FILE__, __LINE__);     \
  } while (0)

#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                    \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);  \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                           \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)

#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      (void)(__VA_ARGS__);                                                                \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#define FAIL(msg)                                                                  \
  do {                                                                             \
    ::doctest::detail::report(false, "FAIL", "", __FILE__, __LINE__, std::string(msg).c_str()); \
    throw ::doctest::detail::RequireFailed{};                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const TestCase& tc : registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++cases;
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      state().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: TEST CASE '%s' threw an unknown exception\n", tc.file, tc.line,
                   tc.name);
      state().current_failed = true;
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-subset] test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n",
              cases, cases - failed_cases, failed_cases, state().checks, state().failed_checks);
  return failed_cases ? 1 : 0;
}
#endif
