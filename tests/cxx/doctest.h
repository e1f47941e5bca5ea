// Minimal doctest-compatible harness (TEST INFRASTRUCTURE): the subset of
// doctest's macros the reference's unit tests use, so those
// test files compile unchanged against the B200 library.  Not doctest.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace dt {

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
inline int reg(const char* name, void (*fn)(), const char* file, int line) {
  registry().push_back({name, fn, file, line});
  return 0;
}

struct State {
  int checks = 0;
  int failures = 0;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};

inline void report(bool ok, const char* what, const char* file, int line) {
  ++state().checks;
  if (!ok) {
    ++state().failures;
    std::printf("  FAILED %s:%d  %s   [in \"%s\"]\n", file, line, what, state().current);
  }
}

}  // namespace dt

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
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // 100 x float epsilon
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : s(std::move(s)) {}
  bool matches(const std::string& m) const { return m.find(s) != std::string::npos; }
  std::string s;
};
inline bool message_matches(const std::string& m, const std::string& want) { return m == want; }
inline bool message_matches(const std::string& m, const Contains& want) { return want.matches(m); }

}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_SUITE(name) namespace DT_CAT(dt_suite_, __LINE__)
#define DT_CASE(name, fn)                                                               \
  static void fn();                                                                     \
  static const int DT_CAT(fn, _reg) = ::dt::reg(name, fn, __FILE__, __LINE__);          \
  static void fn()
#define TEST_CASE(name) DT_CASE(name, DT_CAT(dt_case_, __LINE__))

#define CHECK(...) ::dt::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::dt::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                    \
  do {                                                                                  \
    const bool dt_ok = static_cast<bool>(__VA_ARGS__);                                  \
    ::dt::report(dt_ok, #__VA_ARGS__, __FILE__, __LINE__);                              \
    if (!dt_ok) throw ::dt::RequireFailed{};                                            \
  } while (0)
#define CHECK_NOTHROW(...)                                                              \
  do {                                                                                  \
    bool dt_ok = true;                                                                  \
    try {                                                                               \
      (void)(__VA_ARGS__);                                                              \
    } catch (...) {                                                                     \
      dt_ok = false;                                                                    \
    }                                                                                   \
    ::dt::report(dt_ok, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__);                  \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool dt_ok = false;                                                                 \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__&) {                                                      \
      dt_ok = true;                                                                     \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::dt::report(dt_ok, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__);         \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, ...)                                            \
  do {                                                                                  \
    bool dt_ok = false;                                                                 \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__& dt_e) {                                                 \
      dt_ok = ::doctest::message_matches(dt_e.what(), msg);                             \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::dt::report(dt_ok, "throws " #__VA_ARGS__ " with message: " #expr, __FILE__, __LINE__); \
  } while (0)

#ifdef DT_MAIN
// argv: --only=<name>|<name>...  or  --skip=<name>|...   (exact case names)
static bool dt_listed(const std::string& list, const char* name) {
  size_t pos = 0;
  while (pos <= list.size()) {
    const size_t bar = list.find('|', pos);
    const std::string item = list.substr(pos, bar == std::string::npos ? std::string::npos : bar - pos);
    if (item == name) return true;
    if (bar == std::string::npos) break;
    pos = bar + 1;
  }
  return false;
}
int main(int argc, char** argv) {
  std::string only, skip;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "--only=", 7)) only = argv[i] + 7;
    if (!std::strncmp(argv[i], "--skip=", 7)) skip = argv[i] + 7;
  }
  int run = 0, failed_cases = 0;
  for (const auto& c : ::dt::registry()) {
    if (!only.empty() && !dt_listed(only, c.name)) continue;
    if (!skip.empty() && dt_listed(skip, c.name)) continue;
    ::dt::state().current = c.name;
    const int before = ::dt::state().failures;
    try {
      c.fn();
    } catch (const ::dt::RequireFailed&) {
    } catch (const std::exception& e) {
      ++::dt::state().failures;
      std::printf("  FAILED %s:%d  unexpected exception: %s   [in \"%s\"]\n", c.file, c.line, e.what(), c.name);
    }
    ++run;
    const bool ok = ::dt::state().failures == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("cases: %d run, %d failed; checks: %d, %d failed\n", run, failed_cases,
              ::dt::state().checks, ::dt::state().failures);
  return failed_cases ? 1 : 0;
}
#endif
