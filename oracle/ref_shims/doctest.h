// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY): just
// the macros the reference's unit tests use (proj/tests/*.cpp: TEST_CASE,
// SUBCASE, CHECK, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, REQUIRE_MESSAGE,
// FAIL, doctest::Approx), so the unmodified test sources compile against the
// reference built in oracle/_ref (the vendored doctest.h is absent,
// proj/.gitignore:2). Semantics follow doctest's documentation:
//  * a TEST_CASE body is re-run until every leaf SUBCASE has run once, each
//    run entering at most one new subcase per nesting level;
//  * CHECK records a failure and continues; REQUIRE / FAIL abort the run;
//  * Approx(v) == x  iff  |x - v| < eps * (scale + max(|x|, |v|)), with
//    eps = 100 * FLT_EPSILON and scale = 1 by default.
// Command line: `-tc=<substr>[,<substr>]` keeps matching test cases,
// `-tce=<substr>[,...]` drops them, `-s` lists every case with its time.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <string>
#include <tuple>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& l, double rhs) { return rhs == l; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& l, double rhs) { return !(rhs == l); }
  friend bool operator<=(double lhs, const Approx& r) { return lhs < r.value_ || lhs == r; }
  friend bool operator>=(double lhs, const Approx& r) { return lhs > r.value_ || lhs == r; }
  friend bool operator<=(const Approx& l, double rhs) { return l.value_ < rhs || rhs == l; }
  friend bool operator>=(const Approx& l, double rhs) { return l.value_ > rhs || rhs == l; }
  friend bool operator<(double lhs, const Approx& r) { return lhs < r.value_ && !(lhs == r); }
  friend bool operator>(double lhs, const Approx& r) { return lhs > r.value_ && !(lhs == r); }
  friend bool operator<(const Approx& l, double rhs) { return l.value_ < rhs && !(rhs == l); }
  friend bool operator>(const Approx& l, double rhs) { return l.value_ > rhs && !(rhs == l); }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct TestAbort {};

struct Case {
  void (*fn)();
  const char* name;
  const char* file;
  int line;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Reg {
  Reg(void (*fn)(), const char* name, const char* file, int line) { registry().push_back({fn, name, file, line}); }
};

using Key = std::tuple<std::string, int, std::string>;

struct State {
  long checks = 0, failures = 0;
  const Case* current = nullptr;
  std::set<std::vector<Key>> done;   // subcase paths whose whole subtree ran
  std::vector<Key> path;             // subcases entered in this run
  std::vector<bool> entered;         // per depth: a subcase was entered this run
  long pending = 0;                  // subcases skipped that still have to run
};

inline State& st() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* kind, const char* expr, const char* extra = nullptr) {
  State& s = st();
  ++s.failures;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed%s%s\n  in TEST_CASE \"%s\"", file, line, kind, expr,
               extra ? ": " : "", extra ? extra : "", s.current ? s.current->name : "?");
  for (const auto& k : s.path) std::fprintf(stderr, " / SUBCASE \"%s\"", std::get<2>(k).c_str());
  std::fprintf(stderr, "\n");
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = st();
    const size_t depth = s.path.size();
    if (s.entered.size() <= depth) s.entered.resize(depth + 1, false);
    std::vector<Key> cand = s.path;
    cand.emplace_back(file, line, name);
    if (s.done.count(cand)) return;
    if (s.entered[depth]) {
      ++s.pending;
      return;
    }
    s.entered[depth] = true;
    s.path = cand;
    pending_at_entry_ = s.pending;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = st();
    // the subtree is complete when nothing below was deferred (or it aborted)
    if (s.pending == pending_at_entry_ || std::uncaught_exceptions() > 0) s.done.insert(s.path);
    s.path.pop_back();
    if (s.entered.size() > s.path.size() + 1) s.entered.resize(s.path.size() + 1);
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
  long pending_at_entry_ = 0;
};

inline bool matches(const char* name, const std::vector<std::string>& pats) {
  for (const auto& p : pats)
    if (std::strstr(name, p.c_str())) return true;
  return false;
}

inline std::vector<std::string> split(const char* v) {
  std::vector<std::string> out;
  std::string cur;
  for (const char* c = v; *c; ++c) {
    if (*c == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += *c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> keep, drop;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-tc=", 4)) keep = split(argv[i] + 4);
    else if (!std::strncmp(argv[i], "--test-case=", 12)) keep = split(argv[i] + 12);
    else if (!std::strncmp(argv[i], "-tce=", 5)) drop = split(argv[i] + 5);
    else if (!std::strncmp(argv[i], "--test-case-exclude=", 20)) drop = split(argv[i] + 20);
    else if (!std::strcmp(argv[i], "-s")) list = true;
  }
  State& s = st();
  int cases = 0, failed_cases = 0;
  for (const Case& c : registry()) {
    if (!keep.empty() && !matches(c.name, keep)) continue;
    if (!drop.empty() && matches(c.name, drop)) continue;
    ++cases;
    s.current = &c;
    s.done.clear();
    const long f0 = s.failures;
    const auto t0 = std::chrono::steady_clock::now();
    for (int run = 0; run < 100000; ++run) {
      s.path.clear();
      s.entered.clear();
      s.pending = 0;
      try {
        c.fn();
      } catch (const TestAbort&) {
      } catch (const std::exception& e) {
        report(c.file, c.line, "TEST_CASE", c.name, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report(c.file, c.line, "TEST_CASE", c.name, "unexpected unknown exception");
      }
      if (s.pending == 0) break;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (s.failures != f0) ++failed_cases;
    if (list) std::printf("[%s] %s (%.1f ms)\n", s.failures != f0 ? "FAIL" : " ok ", c.name, ms);
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n", cases,
              cases - failed_cases, failed_cases, s.checks, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                        \
  static void fn();                                                                             \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(fn, name, __FILE__, __LINE__);           \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_shim_case_), name)

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_shim_sc_){name, __FILE__, __LINE__})

#define DOCTEST_ASSERT_IMPL(kind, abort, ...)                                        \
  do {                                                                               \
    ++::doctest::detail::st().checks;                                                \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
    } catch (const std::exception& e) {                                             \
      ::doctest::detail::report(__FILE__, __LINE__, kind, #__VA_ARGS__, e.what());    \
      if (abort) throw ::doctest::detail::TestAbort{};                               \
      break;                                                                         \
    }                                                                                \
    if (!doctest_ok_) {                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, kind, #__VA_ARGS__);             \
      if (abort) throw ::doctest::detail::TestAbort{};                               \
    }                                                                                \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", true, !(__VA_ARGS__))
#define CHECK_MESSAGE(cond, msg) DOCTEST_ASSERT_IMPL("CHECK_MESSAGE", false, cond)
#define REQUIRE_MESSAGE(cond, msg) DOCTEST_ASSERT_IMPL("REQUIRE_MESSAGE", true, cond)

#define CHECK_THROWS_AS(expr, ...)                                                          \
  do {                                                                                      \
    ++::doctest::detail::st().checks;                                                       \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr, "no exception"); \
    } catch (const __VA_ARGS__&) {                                                          \
    } catch (...) {                                                                         \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr, "wrong exception type"); \
    }                                                                                       \
  } while (0)
#define CHECK_THROWS(expr)                                                                  \
  do {                                                                                      \
    ++::doctest::detail::st().checks;                                                       \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS", #expr, "no exception"); \
    } catch (...) {                                                                         \
    }                                                                                       \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
  do {                                                                                      \
    ++::doctest::detail::st().checks;                                                       \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const std::exception& e) {                                                     \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #expr, e.what());      \
    } catch (...) {                                                                         \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_NOTHROW", #expr, "unknown exception"); \
    }                                                                                       \
  } while (0)
#define FAIL(msg)                                                                   \
  do {                                                                              \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", "", std::string(msg).c_str()); \
    throw ::doctest::detail::TestAbort{};                                           \
  } while (0)
#define MESSAGE(msg) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
