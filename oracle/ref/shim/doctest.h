// ORACLE (test infrastructure): doctest-subset shim used only to build the
// reference's own unit suites (/root/reference/proj/tests/test_*.cpp)
// unmodified into oracle/_ref/unit_tests.  The vendored doctest
// (proj/vendor/, proj/.gitignore:2) is absent from the image.  Covers the
// macros those suites use: TEST_CASE, SUBCASE (each leaf subcase runs in its
// own pass over the test case, doctest's traversal), CHECK, REQUIRE,
// CHECK_THROWS, doctest::Approx (doctest's default epsilon and comparison).
// Output: one line per failed assertion, a summary, exit code 1 on failure.
// Extra: `unit_tests -tc=<substring>` runs the matching cases only and
// `-ltc` lists them.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }
  friend bool operator<(double lhs, const Approx& r) { return lhs < r.value_ && lhs != r; }
  friend bool operator>(double lhs, const Approx& r) { return lhs > r.value_ && lhs != r; }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

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
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireAbort {};

// SUBCASE traversal (doctest's): a pass enters at most one not-yet-passed
// subcase per nesting level; a subcase skipped because a sibling was entered
// asks for another pass; a subcase is marked passed on exit unless one of its
// own children was skipped in that pass.
struct State {
  int asserts = 0, failed = 0;
  bool case_failed = false;
  std::vector<std::string> stack;                 // entered subcases, outermost first
  std::vector<std::vector<std::string>> passed;  // finished subcase paths
  std::vector<char> entered_at, pending_at;      // per depth, this pass
  bool reenter = false;
  const char* current = "";
};
inline State& st() {
  static State s;
  return s;
}

inline bool is_passed(const std::vector<std::string>& p) {
  for (auto& d : st().passed)
    if (d == p) return true;
  return false;
}

struct Subcase {
  bool entered = false;
  Subcase(const char* name) {
    State& s = st();
    const std::size_t d = s.stack.size();
    if (s.entered_at.size() <= d + 1) {
      s.entered_at.resize(d + 2, 0);
      s.pending_at.resize(d + 2, 0);
    }
    std::vector<std::string> p = s.stack;
    p.push_back(name);
    if (is_passed(p)) return;
    if (s.entered_at[d]) {
      s.reenter = true;
      s.pending_at[d] = 1;
      return;
    }
    entered = true;
    s.entered_at[d] = 1;
    s.entered_at[d + 1] = 0;
    s.pending_at[d + 1] = 0;
    s.stack.push_back(name);
  }
  ~Subcase() {
    if (!entered) return;
    State& s = st();
    const std::size_t d = s.stack.size();  // depth of this subcase's children
    if (!s.pending_at[d]) s.passed.push_back(s.stack);
    s.stack.pop_back();
  }
  explicit operator bool() const { return entered; }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = st();
  ++s.asserts;
  if (ok) return;
  ++s.failed;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct! [case: %s", file, line, kind, expr, s.current);
  for (auto& p : s.stack) std::fprintf(stderr, " / %s", p.c_str());
  std::fprintf(stderr, "]\n");
}

inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    if (std::strcmp(argv[i], "-ltc") == 0) list = true;
  }
  int cases = 0, failed_cases = 0;
  for (auto& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    if (list) {
      std::printf("%s\n", tc.name);
      continue;
    }
    ++cases;
    State& s = st();
    s.case_failed = false;
    s.passed.clear();
    s.current = tc.name;
    for (int pass = 0; pass < 1000; ++pass) {
      s.stack.clear();
      s.entered_at.assign(2, 0);
      s.pending_at.assign(2, 0);
      s.reenter = false;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s [case: %s]\n", tc.file, tc.line, e.what(),
                     tc.name);
        ++s.asserts;
        ++s.failed;
        s.case_failed = true;
      }
      if (!s.reenter) break;  // no subcase was skipped for a sibling: every leaf has run
    }
    if (s.case_failed) ++failed_cases;
    std::printf("[%s] %s\n", s.case_failed ? "FAIL" : " ok ", tc.name);
  }
  if (list) return 0;
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
  std::printf("[doctest-shim] assertions: %d | %d passed | %d failed\n", st().asserts, st().asserts - st().failed,
              st().failed);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                                 \
  static void DOCTEST_ANON(doctest_fn_)();                                                             \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,             \
                                                                  &DOCTEST_ANON(doctest_fn_));         \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define CHECK(...)                                                                                   \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    try {                                                                                            \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                                  \
    } catch (...) {                                                                                  \
      doctest_ok_ = false;                                                                           \
    }                                                                                                \
    ::doctest::detail::report(doctest_ok_, "CHECK", #__VA_ARGS__, __FILE__, __LINE__);               \
  } while (0)

#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))

#define REQUIRE(...)                                                                                 \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    try {                                                                                            \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                                  \
    } catch (...) {                                                                                  \
      doctest_ok_ = false;                                                                           \
    }                                                                                                \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);             \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                       \
  } while (0)

#define CHECK_THROWS(...)                                                                            \
  do {                                                                                               \
    bool doctest_threw_ = false;                                                                     \
    try {                                                                                            \
      static_cast<void>(__VA_ARGS__);                                                                \
    } catch (...) {                                                                                  \
      doctest_threw_ = true;                                                                         \
    }                                                                                                \
    ::doctest::detail::report(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__);     \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
  do {                                                                                               \
    bool doctest_threw_ = false;                                                                     \
    try {                                                                                            \
      static_cast<void>(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                                   \
      doctest_threw_ = true;                                                                         \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::doctest::detail::report(doctest_threw_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);         \
  } while (0)

#define CHECK_NOTHROW(...)                                                                           \
  do {                                                                                               \
    bool doctest_ok_ = true;                                                                         \
    try {                                                                                            \
      static_cast<void>(__VA_ARGS__);                                                                \
    } catch (...) {                                                                                  \
      doctest_ok_ = false;                                                                           \
    }                                                                                                \
    ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);       \
  } while (0)

#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
