// doctest.h -- a minimal, independent implementation of the subset of the
// doctest test-macro interface used by the reference's hot-path unit suites
// (proj/tests/test_{core,kernel_exact,octree,bh_kernel,shooting}.cpp), so
// those suites can be compiled BY PATH against the B200 library's C++ API
// (tests/cpp/reftests.mk). doctest itself is not in this image; this file is
// written for this repository and only mirrors the macro names and the
// documented semantics:
//   TEST_CASE, SUBCASE (re-entry: the test case re-runs once per leaf subcase,
//   each run entering one unfinished subcase per nesting level), CHECK,
//   CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE (aborts the test
//   case), FAIL (aborts), doctest::Approx(v).epsilon(e) (relative tolerance
//   e * (1 + max(|a|, |b|)), default 100 float epsilons).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <map>
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
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

namespace detail {

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

struct Register {
  Register(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct Abort {};  // REQUIRE / FAIL: leave the current test case run

struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  // subcase bookkeeping for one test case
  std::map<std::string, bool> completed;
  std::vector<std::string> path;
  std::vector<bool> entered;   // per depth: a subcase was entered in this run
  std::vector<bool> pending;   // per depth: an unfinished subcase was skipped
};
inline State& st() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* what) {
  State& s = st();
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
inline void check(bool ok, const char* file, int line, const char* expr) {
  ++st().checks;
  if (!ok) report(file, line, expr);
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = st();
    const size_t depth = s.path.size();
    if (s.entered.size() <= depth) {
      s.entered.resize(depth + 1, false);
      s.pending.resize(depth + 1, false);
    }
    key_ = (depth ? s.path.back() : std::string()) + "/" + name + "@" + file + ":" +
           std::to_string(line);
    if (s.completed[key_]) return;
    if (s.entered[depth]) {  // another subcase at this level ran: come back later
      s.pending[depth] = true;
      return;
    }
    s.entered[depth] = true;
    s.path.push_back(key_);
    if (s.entered.size() <= depth + 1) {
      s.entered.resize(depth + 2, false);
      s.pending.resize(depth + 2, false);
    }
    s.entered[depth + 1] = false;
    s.pending[depth + 1] = false;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = st();
    const size_t depth = s.path.size();  // this subcase's children level
    // finished unless one of its own children is still pending
    if (!s.pending[depth]) s.completed[key_] = true;
    else s.pending[depth - 1] = true;
    s.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  bool active_ = false;
};

inline int run_all() {
  State& s = st();
  int failed_cases = 0, passed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.completed.clear();
    s.case_failed = false;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered.assign(1, false);
      s.pending.assign(1, false);
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report(tc.file, tc.line, "unexpected non-std exception");
      }
      // unwinding out of an aborted subcase leaves entries on the path
      s.path.clear();
      if (!s.pending[0]) break;  // every subcase of this test case has run
    }
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case: %s\n", tc.name);
    } else {
      ++passed_cases;
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | checks: %ld | %ld failed\n",
              passed_cases + failed_cases, passed_cases, failed_cases, s.checks, s.failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                       \
  static void fn();                                                                 \
  static ::doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                           &fn);                   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define SUBCASE(name) \
  if (::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__}; \
      DOCTEST_CAT(doctest_sc_, __LINE__))

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
  ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                          \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "REQUIRE " #__VA_ARGS__); \
    if (!doctest_ok_) throw ::doctest::detail::Abort{};                               \
  } while (0)
#define FAIL(msg)                                                            \
  do {                                                                       \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL: " msg);             \
    throw ::doctest::detail::Abort{};                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    bool doctest_thrown_ = false;                                                           \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_thrown_ = true;                                                               \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::check(doctest_thrown_, __FILE__, __LINE__,                           \
                             "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")");                \
  } while (0)
#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    bool doctest_ok_ = true;                                                              \
    try {                                                                                 \
      static_cast<void>(__VA_ARGS__);                                                     \
    } catch (...) {                                                                       \
      doctest_ok_ = false;                                                                \
    }                                                                                     \
    ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW " #__VA_ARGS__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
