// doctest.h -- TEST INFRASTRUCTURE ONLY: a minimal stand-in for the doctest
// framework the reference's unit tests are written against (proj/tests/*.cpp
// include <doctest.h>; the reference vendors doctest but does not ship it,
// SURVEY.md 8c).  It implements exactly the macros those files use:
// TEST_CASE, SUBCASE (one level: the test body re-runs once per subcase),
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL, MESSAGE and
// doctest::Approx(...).epsilon(...), with doctest's comparison rule
// |a - b| < eps * (scale + max(|a|, |b|)), scale 1, default eps 100 * FLT_EPSILON.
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (unit_main.cpp) defines main(): every
// test case runs, failures print file:line, the exit code is the failed count.
#ifndef ECCO_DOCTEST_SHIM_H_
#define ECCO_DOCTEST_SHIM_H_

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <ostream>
#include <set>
#include <string>
#include <utility>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
  friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && lhs != rhs; }
  friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && lhs != rhs; }
  friend std::ostream& operator<<(std::ostream& os, const Approx& a) {
    return os << "Approx(" << a.value_ << ")";
  }

 private:
  double value_;
  double eps_ = 100.0 * FLT_EPSILON;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Reg {
  Reg(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({fn, name, file, line});
  }
};

struct Run {
  int failed_asserts = 0;
  int asserts = 0;
  bool entered = false;          // a subcase was entered in this pass
  std::string entered_id;
  std::set<std::string> done;    // subcases finished in earlier passes
  const char* test = "";
};

inline Run& run() {
  static Run r;
  return r;
}

struct Abort {};  // REQUIRE / FAIL leave the current pass

inline void fail(const char* file, int line, const char* what) {
  ++run().failed_asserts;
  std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, run().test, what);
}

inline bool check(bool ok, const char* file, int line, const char* what, bool fatal) {
  ++run().asserts;
  if (!ok) {
    fail(file, line, what);
    if (fatal) throw Abort{};
  }
  return ok;
}

struct Subcase {
  bool enter = false;
  Subcase(const char* name, const char* file, int line) {
    const std::string id = std::string(file) + ":" + std::to_string(line) + ":" + name;
    Run& r = run();
    if (!r.entered && !r.done.count(id)) {
      r.entered = true;
      r.entered_id = id;
      enter = true;
    }
  }
  explicit operator bool() const { return enter; }
};

inline int run_all() {
  int failed_cases = 0, n = 0;
  for (const auto& tc : registry()) {
    ++n;
    Run& r = run();
    r = Run{};
    r.test = tc.name;
    const int before = 0;
    bool ok = true;
    for (int pass = 0; pass < 1000; ++pass) {  // once per subcase, once without any
      r.entered = false;
      const int f0 = r.failed_asserts;
      try {
        tc.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        fail(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        fail(tc.file, tc.line, "unexpected exception");
      }
      if (r.failed_asserts != f0) ok = false;
      if (!r.entered) break;
      r.done.insert(r.entered_id);
    }
    (void)before;
    if (!ok) ++failed_cases;
  }
  std::printf("[doctest shim] test cases: %d | %d passed | %d failed\n", n, n - failed_cases,
              failed_cases);
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                    \
  static void fn();                                                                         \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);        \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "not " #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_THROWS_AS(expr, ...)                                                               \
  do {                                                                                           \
    bool caught_ = false;                                                                        \
    try {                                                                                        \
      (void)(expr);                                                                              \
    } catch (const __VA_ARGS__&) {                                                               \
      caught_ = true;                                                                            \
    } catch (...) {                                                                              \
    }                                                                                            \
    ::doctest::detail::check(caught_, __FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr, false); \
  } while (0)
#define FAIL(...)                                                          \
  do {                                                                     \
    ::doctest::detail::fail(__FILE__, __LINE__, "FAIL: " #__VA_ARGS__);    \
    throw ::doctest::detail::Abort{};                                      \
  } while (0)
#define MESSAGE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all() ? 1 : 0; }
#endif

#endif  // ECCO_DOCTEST_SHIM_H_
