// doctest.h — a small doctest-compatible test harness, written for this repo.
//
// The reference's unit suites (/root/reference/proj/tests/test_*.cpp) are
// written against doctest (not vendored in the reference tree, not in this
// image).  This header implements the subset of doctest's interface those
// suites use — TEST_CASE, CHECK / REQUIRE with value decomposition,
// CHECK_THROWS_AS, CHECK_NOTHROW, REQUIRE_THROWS_AS, CAPTURE, FAIL, MESSAGE,
// doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the suites
// compile UNCHANGED against the drop-in headers in ../include/evsim/ and run
// against libevsim_gpu.so (tests/test_refsuite.py, oracle/Makefile).
//
// Output: one line per failed assertion (file:line, expression, expanded
// values, captured variables) and a summary line
//   [refsuite] test cases: N | passed: P | failed: F ; assertions: A | failed: AF
// The exit code is 1 when any assertion failed.  Optional argument: a
// substring; only test cases whose name contains it run.
#pragma once

// CHECK(a == b) expands to `Decomposer() <= a == b` (the usual decomposition:
// <= binds tighter than ==), which -Wparentheses flags at every use.
#if defined(__GNUC__)
#pragma GCC diagnostic ignored "-Wparentheses"
#pragma GCC diagnostic ignored "-Wsign-compare"  // (doctest compares the original operand types)
#endif

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx epsilon(double e) const {
    Approx a(*this);
    a.eps_ = e;
    return a;
  }
  Approx scale(double s) const {
    Approx a(*this);
    a.scale_ = s;
    return a;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

namespace detail {

template <class T>
std::string show(const T& v) {
  if constexpr (std::is_same_v<T, bool>) {
    return v ? "true" : "false";
  } else if constexpr (std::is_same_v<T, char> || std::is_same_v<T, signed char> ||
                       std::is_same_v<T, unsigned char>) {
    return std::to_string(static_cast<int>(v));
  } else if constexpr (std::is_arithmetic_v<T>) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
  } else if constexpr (std::is_enum_v<T>) {
    return std::to_string(static_cast<long long>(v));
  } else if constexpr (std::is_same_v<T, Approx>) {
    return "Approx(" + show(v.value()) + ")";
  } else if constexpr (std::is_convertible_v<const T&, std::string>) {
    return "\"" + std::string(v) + "\"";
  } else {
    return "{?}";
  }
}

struct Result {
  bool ok;
  std::string expanded;
};

template <class L>
struct Lhs {
  const L& lhs;
#define DOCTEST_SHIM_BINOP(OP)                                                  \
  template <class R>                                                            \
  Result operator OP(const R& rhs) const {                                      \
    return Result{static_cast<bool>(lhs OP rhs), show(lhs) + " " #OP " " + show(rhs)}; \
  }
  DOCTEST_SHIM_BINOP(==)
  DOCTEST_SHIM_BINOP(!=)
  DOCTEST_SHIM_BINOP(<)
  DOCTEST_SHIM_BINOP(>)
  DOCTEST_SHIM_BINOP(<=)
  DOCTEST_SHIM_BINOP(>=)
#undef DOCTEST_SHIM_BINOP
  operator Result() const { return Result{static_cast<bool>(lhs), show(lhs)}; }
};

struct Decomposer {
  template <class L>
  Lhs<L> operator<=(const L& lhs) const {
    return Lhs<L>{lhs};
  }
};

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

struct RequireAbort {};

struct State {
  std::vector<TestCase> cases;
  const TestCase* current = nullptr;
  bool current_failed = false;
  long long asserts = 0, asserts_failed = 0;
  std::vector<std::string> captures;
};

inline State& state() {
  static State s;
  return s;
}

inline int reg(const char* name, const char* file, int line, void (*fn)()) {
  state().cases.push_back(TestCase{name, file, line, fn});
  return 0;
}

inline void report(const char* file, int line, const char* macro, const char* expr, const std::string& detail) {
  State& s = state();
  s.current_failed = true;
  ++s.asserts_failed;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s( %s )%s%s\n", file, line, s.current ? s.current->name : "?",
               macro, expr, detail.empty() ? "" : "  with expansion: ", detail.c_str());
  for (const auto& c : s.captures) std::fprintf(stderr, "    captured: %s\n", c.c_str());
}

inline bool assert_result(const Result& r, const char* file, int line, const char* macro, const char* expr) {
  ++state().asserts;
  if (!r.ok) report(file, line, macro, expr, r.expanded);
  return r.ok;
}

struct Capture {
  explicit Capture(std::string s) { state().captures.push_back(std::move(s)); }
  ~Capture() { state().captures.pop_back(); }
};

inline int run(int argc, char** argv) {
  State& s = state();
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int n = 0, failed = 0;
  for (const TestCase& tc : s.cases) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ++n;
    s.current = &tc;
    s.current_failed = false;
    s.captures.clear();
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, "unexpected exception");
    }
    if (s.current_failed) ++failed;
  }
  std::printf("[refsuite] test cases: %d | passed: %d | failed: %d ; assertions: %lld | failed: %lld\n", n,
              n - failed, failed, s.asserts, s.asserts_failed);
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TC(fn, name)                                                                      \
  static void fn();                                                                                     \
  [[maybe_unused]] static const int DOCTEST_SHIM_CAT(fn, _reg) = doctest::detail::reg(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TC(DOCTEST_SHIM_CAT(doctest_shim_tc_, __COUNTER__), name)

#define DOCTEST_SHIM_ASSERT(macro, expr, abort_on_fail)                                                   \
  do {                                                                                                    \
    if (!doctest::detail::assert_result(doctest::detail::Decomposer() <= expr, __FILE__, __LINE__, macro, #expr) && \
        (abort_on_fail))                                                                                  \
      throw doctest::detail::RequireAbort{};                                                             \
  } while (0)
#define CHECK(...) DOCTEST_SHIM_ASSERT("CHECK", __VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_SHIM_ASSERT("REQUIRE", __VA_ARGS__, true)
#define CHECK_FALSE(...) DOCTEST_SHIM_ASSERT("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_SHIM_ASSERT("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define DOCTEST_SHIM_THROWS_AS(macro, expr, type, abort_on_fail)                                      \
  do {                                                                                                \
    bool doctest_shim_ok = false;                                                                     \
    std::string doctest_shim_what = "no exception";                                                  \
    try {                                                                                             \
      static_cast<void>(expr);                                                                        \
    } catch (const type&) {                                                                           \
      doctest_shim_ok = true;                                                                         \
    } catch (const std::exception& e) {                                                               \
      doctest_shim_what = std::string("other exception: ") + e.what();                               \
    } catch (...) {                                                                                   \
      doctest_shim_what = "other exception";                                                         \
    }                                                                                                 \
    if (!doctest::detail::assert_result(doctest::detail::Result{doctest_shim_ok, doctest_shim_what},  \
                                        __FILE__, __LINE__, macro, #expr ", " #type) &&               \
        (abort_on_fail))                                                                              \
      throw doctest::detail::RequireAbort{};                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_SHIM_THROWS_AS("CHECK_THROWS_AS", expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_SHIM_THROWS_AS("REQUIRE_THROWS_AS", expr, __VA_ARGS__, true)
#define CHECK_THROWS(expr) DOCTEST_SHIM_THROWS_AS("CHECK_THROWS", expr, std::exception, false)

#define CHECK_NOTHROW(expr)                                                                            \
  do {                                                                                                 \
    std::string doctest_shim_what;                                                                     \
    bool doctest_shim_ok = true;                                                                       \
    try {                                                                                              \
      static_cast<void>(expr);                                                                         \
    } catch (const std::exception& e) {                                                                \
      doctest_shim_ok = false;                                                                         \
      doctest_shim_what = std::string("threw: ") + e.what();                                           \
    } catch (...) {                                                                                    \
      doctest_shim_ok = false;                                                                         \
      doctest_shim_what = "threw";                                                                     \
    }                                                                                                  \
    doctest::detail::assert_result(doctest::detail::Result{doctest_shim_ok, doctest_shim_what}, __FILE__, \
                                   __LINE__, "CHECK_NOTHROW", #expr);                                  \
  } while (0)

#define CAPTURE(x)                                                                     \
  doctest::detail::Capture DOCTEST_SHIM_CAT(doctest_shim_capture_, __COUNTER__)(      \
      std::string(#x " := ") + doctest::detail::show(x))
#define INFO(x) CAPTURE(x)
#define MESSAGE(x) std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, std::string(x).c_str())
#define FAIL(msg)                                                                                       \
  do {                                                                                                  \
    doctest::detail::assert_result(doctest::detail::Result{false, std::string(msg)}, __FILE__, __LINE__, \
                                   "FAIL", "");                                                         \
    throw doctest::detail::RequireAbort{};                                                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run(argc, argv); }
#endif
