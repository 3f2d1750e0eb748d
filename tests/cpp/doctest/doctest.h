// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) include
// <doctest.h>, which the reference does not vendor. This
// header implements the subset those tests use -- TEST_SUITE_BEGIN/END,
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx(.epsilon), doctest::Contains -- so
// tests/test_reference_unit_tests.py can compile them unchanged against
// include/dwdpsim/*.hpp (the drop-in adapter) and libdwdp.so.
#pragma once

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
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

// Substring matcher for CHECK_THROWS_WITH_AS(expr, doctest::Contains("..."), T).
struct Contains {
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }
  std::string s_;
};

namespace detail {

struct Case {
  const char* name;
  std::string suite;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline std::string& current_suite() {
  static std::string s;
  return s;
}
inline int& failures() {
  static int n = 0;
  return n;
}
inline int& assertions() {
  static int n = 0;
  return n;
}
inline int set_suite(const char* s) {
  current_suite() = s;
  return 0;
}
inline int reg(const char* name, void (*fn)(), const char* file, int line) {
  registry().push_back({name, current_suite(), fn, file, line});
  return 0;
}
struct RequireFailed {};

inline void fail(const char* kind, const char* expr, const char* file, int line,
                 const std::string& extra = "") {
  ++failures();
  std::fprintf(stderr, "%s:%d: %s( %s ) failed%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str());
}
inline bool match_what(const char* what, const char* want) { return std::strcmp(what, want) == 0; }
inline bool match_what(const char* what, const std::string& want) { return want == what; }
inline bool match_what(const char* what, const Contains& c) { return c.matches(what); }

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __COUNTER__)

#define TEST_SUITE_BEGIN(name) \
  static const int DOCTEST_UNIQUE(doctest_suite_) = ::doctest::detail::set_suite(name)
#define TEST_SUITE_END() \
  static const int DOCTEST_UNIQUE(doctest_suite_end_) = ::doctest::detail::set_suite("")

#define DOCTEST_TEST_CASE_(fn, name)                                                    \
  static void fn();                                                                     \
  static const int DOCTEST_CAT(fn, _reg) = ::doctest::detail::reg(name, &fn, __FILE__, \
                                                                  __LINE__);            \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_UNIQUE(doctest_case_), name)

#define DOCTEST_ASSERT_(kind, cond, expr, fatal)                              \
  do {                                                                        \
    ++::doctest::detail::assertions();                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      doctest_ok_ = static_cast<bool>(cond);                                  \
    } catch (const std::exception& e) {                                       \
      ::doctest::detail::fail(kind, expr, __FILE__, __LINE__,                 \
                              std::string("threw ") + e.what());              \
      if (fatal) throw ::doctest::detail::RequireFailed{};                    \
      break;                                                                  \
    }                                                                         \
    if (!doctest_ok_) {                                                       \
      ::doctest::detail::fail(kind, expr, __FILE__, __LINE__);                \
      if (fatal) throw ::doctest::detail::RequireFailed{};                    \
    }                                                                         \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, T)                                                        \
  do {                                                                                  \
    ++::doctest::detail::assertions();                                                  \
    try {                                                                               \
      (void)(expr);                                                                     \
      ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__, "no throw"); \
    } catch (const T&) {                                                                \
    } catch (...) {                                                                     \
      ::doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__,             \
                              "wrong exception type");                                  \
    }                                                                                   \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, T)                                               \
  do {                                                                                    \
    ++::doctest::detail::assertions();                                                    \
    try {                                                                                 \
      (void)(expr);                                                                       \
      ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,          \
                              "no throw");                                                \
    } catch (const T& e) {                                                                \
      if (!::doctest::detail::match_what(e.what(), with))                                 \
        ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,        \
                                std::string("message: ") + e.what());                     \
    } catch (...) {                                                                       \
      ::doctest::detail::fail("CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__,          \
                              "wrong exception type");                                    \
    }                                                                                     \
  } while (0)

#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    ++::doctest::detail::assertions();                                                 \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      ::doctest::detail::fail("CHECK_NOTHROW", #expr, __FILE__, __LINE__, "threw");    \
    }                                                                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
// Runs every registered case (optionally only suite S with -ts=S) and prints a
// doctest-style summary line; exit status 1 if any assertion failed.
int main(int argc, char** argv) {
  std::string only;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "-ts=", 4) == 0) only = argv[i] + 4;
  int cases = 0, failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    if (!only.empty() && c.suite != only) continue;
    ++cases;
    const int before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::detail::fail("TEST_CASE", c.name, c.file, c.line,
                              std::string("uncaught exception: ") + e.what());
    }
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  ^ in test case \"%s\" (suite %s)\n", c.name, c.suite.c_str());
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases,
              failed_cases);
  std::printf("[doctest] assertions: %d | %d failed\n", ::doctest::detail::assertions(),
              ::doctest::detail::failures());
  return failed_cases ? 1 : 0;
}
#endif
