// A minimal test harness with the subset of the doctest interface the
// reference's unit tests use (TEST_CASE, single-level SUBCASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_NOTHROW,
// doctest::Approx, doctest::Contains), so those test files compile unchanged
// against our C++ drop-in. Test infrastructure only; written for this repo
// (doctest itself is not in the image).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
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
  friend bool operator==(double a, const Approx& b) { return b.close(a); }
  friend bool operator==(const Approx& b, double a) { return b.close(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.close(a); }
  friend bool operator!=(const Approx& b, double a) { return !b.close(a); }

 private:
  bool close(double a) const {
    return std::fabs(a - v_) < eps_ * (scale_ + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  double v_;
  double eps_ = 1.1920929e-05;  // 100 * FLT_EPSILON
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : text(std::move(s)) {}
  std::string text;
};

}  // namespace doctest

namespace mini {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};
struct State {
  int target = 0;  // which SUBCASE this run enters
  int seen = 0;    // SUBCASEs met so far in this run
  long failures = 0, checks = 0;
  bool case_failed = false;
};
inline State& st() {
  static State s;
  return s;
}
struct Abort {};
inline bool check(bool ok, const char* what, const char* file, int line) {
  ++st().checks;
  if (!ok) {
    ++st().failures;
    st().case_failed = true;
    std::printf("  FAIL %s:%d: %s\n", file, line, what);
  }
  return ok;
}
struct Subcase {
  bool run;
  explicit Subcase(const char*) : run(st().seen++ == st().target) {}
  explicit operator bool() const { return run; }
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    st().case_failed = false;
    for (int target = 0;; ++target) {  // one run per SUBCASE (at least one run)
      st().target = target;
      st().seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        check(false, (std::string("unexpected exception: ") + e.what()).c_str(), c.file, c.line);
      }
      if (target + 1 >= st().seen) break;
    }
    std::printf("%s: %s\n", st().case_failed ? "FAILED" : "passed", c.name);
    failed_cases += st().case_failed;
  }
  std::printf("[doctest-mini] test cases: %zu | %zu passed | %d failed | checks: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, st().checks,
              st().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define MINI_TC(name, id)                                                        \
  static void MINI_CAT(mini_tc_, id)();                                          \
  static ::mini::Reg MINI_CAT(mini_reg_, id)(name, &MINI_CAT(mini_tc_, id), __FILE__, __LINE__); \
  static void MINI_CAT(mini_tc_, id)()
#define TEST_CASE(name) MINI_TC(name, __COUNTER__)
#define SUBCASE(name) if (const ::mini::Subcase MINI_CAT(mini_sc_, __LINE__){name})
#define CHECK(...) ::mini::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::mini::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    if (!::mini::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
      throw ::mini::Abort{};                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool mini_ok_ = false;                                                          \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__&) {                                                  \
      mini_ok_ = true;                                                              \
    } catch (...) {                                                                 \
    }                                                                               \
    ::mini::check(mini_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__);     \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                    \
  do {                                                                              \
    bool mini_ok_ = false;                                                          \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__& e) {                                                \
      mini_ok_ = std::string(e.what()).find((matcher).text) != std::string::npos;   \
    } catch (...) {                                                                 \
    }                                                                               \
    ::mini::check(mini_ok_, #expr " throws " #__VA_ARGS__ " with message", __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                         \
  do {                                                                              \
    bool mini_ok_ = true;                                                           \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (...) {                                                                 \
      mini_ok_ = false;                                                             \
    }                                                                               \
    ::mini::check(mini_ok_, #expr " does not throw", __FILE__, __LINE__);           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::mini::run_all(); }
#endif
