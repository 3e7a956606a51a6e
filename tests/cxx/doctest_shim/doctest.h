// Minimal stand-in for the doctest single header, so the reference's own unit
// suites (/root/reference/proj/tests/test_*.cpp) compile UNCHANGED against
// include/ + libwavepipe.so (tests/test_reference_suites.py).  doctest itself
// is not vendored in the reference and there is no network here; this header
// implements only the subset those suites use: TEST_SUITE, TEST_CASE,
// SUBCASE (re-entry per leaf, doctest's semantics), CHECK / CHECK_FALSE /
// REQUIRE, CHECK_THROWS_AS / CHECK_THROWS_WITH_AS / CHECK_NOTHROW, FAIL,
// INFO (ignored), doctest::Approx and doctest::Contains.  Test infrastructure
// only; nothing in the product includes it.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
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
  friend bool operator==(double x, const Approx& a) {
    return std::fabs(x - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(x), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double x) { return x == a; }
  friend bool operator!=(double x, const Approx& a) { return !(x == a); }
  friend bool operator!=(const Approx& a, double x) { return !(x == a); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  explicit Contains(const std::string& x) : s(x) {}
  bool match(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

struct RequireFailed {};

struct State {
  int failed_checks = 0, checks = 0;
  bool case_failed = false;
  // SUBCASE traversal: one new leaf per run of the test case.
  std::vector<std::string> path;
  std::set<int> taken;                        // levels entered this run
  std::set<std::vector<std::string>> done;    // fully explored subcase paths
  std::vector<bool> child_pending;            // per entered level: an unexplored child was skipped
  bool pending = false;                       // another run is needed
};

inline State& st() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const char* what) {
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
  ++st().failed_checks;
  st().case_failed = true;
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  ++st().checks;
  if (ok) return;
  report(file, line, expr);
  if (require) throw RequireFailed{};
}

inline bool matches(const std::string& what, const char* want) { return what == want; }
inline bool matches(const std::string& what, const std::string& want) { return what == want; }
inline bool matches(const std::string& what, const Contains& want) { return want.match(what); }

class Subcase {
 public:
  explicit Subcase(const char* name) {
    State& s = st();
    const int level = static_cast<int>(s.path.size());
    std::vector<std::string> p = s.path;
    p.push_back(name);
    if (s.done.count(p)) return;
    if (s.taken.count(level)) {  // a sibling ran this time: come back for this one
      s.pending = true;
      if (!s.child_pending.empty()) s.child_pending.back() = true;
      return;
    }
    s.taken.insert(level);
    s.path = p;
    s.child_pending.push_back(false);
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    const bool unexplored = s.child_pending.back();
    s.child_pending.pop_back();
    if (!unexplored || std::uncaught_exceptions()) s.done.insert(s.path);
    else if (!s.child_pending.empty()) s.child_pending.back() = true;
    s.path.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    State& s = st();
    s.done.clear();
    s.case_failed = false;
    do {
      s.pending = false;
      s.path.clear();
      s.taken.clear();
      s.child_pending.clear();
      try {
        c.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        ++s.failed_checks;
        s.case_failed = true;
      }
    } while (s.pending);
    if (s.case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - failed_cases, failed_cases);
  std::printf("[doctest shim] assertions: %d | %d failed\n", st().checks, st().failed_checks);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)

#define TEST_SUITE(name) namespace DS_CAT(ds_suite_, __LINE__)
#define TEST_CASE(name)                                                                            \
  static void DS_CAT(ds_case_, __LINE__)();                                                        \
  static const ::doctest::shim::Reg DS_CAT(ds_reg_, __LINE__)(name, __FILE__, __LINE__,             \
                                                             &DS_CAT(ds_case_, __LINE__));          \
  static void DS_CAT(ds_case_, __LINE__)()
#define SUBCASE(name) if (const ::doctest::shim::Subcase DS_CAT(ds_sub_, __LINE__){name})

#define CHECK(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::shim::check(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) ::doctest::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define INFO(...) static_cast<void>(0)
#define FAIL(msg)                                              \
  do {                                                         \
    ::doctest::shim::report(__FILE__, __LINE__, "FAIL: " msg); \
    throw ::doctest::shim::RequireFailed{};                    \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                     \
  do {                                                                                                 \
    bool ds_ok = false;                                                                                \
    try {                                                                                              \
      static_cast<void>(expr);                                                                         \
    } catch (const __VA_ARGS__&) {                                                                     \
      ds_ok = true;                                                                                    \
    } catch (...) {                                                                                    \
    }                                                                                                  \
    ::doctest::shim::check(ds_ok, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", \
                           false);                                                                     \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, ...)                                                         \
  do {                                                                                                \
    bool ds_ok = false;                                                                               \
    try {                                                                                             \
      static_cast<void>(expr);                                                                        \
    } catch (const __VA_ARGS__& ds_e) {                                                               \
      ds_ok = ::doctest::shim::matches(std::string(ds_e.what()), with);                               \
    } catch (...) {                                                                                   \
    }                                                                                                 \
    ::doctest::shim::check(ds_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ", " #with ")", \
                           false);                                                                    \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
  do {                                                                                          \
    bool ds_ok = true;                                                                          \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (...) {                                                                             \
      ds_ok = false;                                                                            \
    }                                                                                           \
    ::doctest::shim::check(ds_ok, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")", false);      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
