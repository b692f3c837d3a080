// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit suites (proj/tests/*.cpp) are written against
// doctest, whose vendored copy is git-ignored and absent
// (proj/.gitignore:2). This header implements the subset they use —
// TEST_CASE, CHECK / CHECK_FALSE / REQUIRE / REQUIRE_FALSE, CHECK_THROWS_AS,
// FAIL, CAPTURE, doctest::Approx(...).epsilon(...) — so those suites compile
// unchanged against the B200 drop-in (tests/test_gpu_conformance.py).
// Command line: -tc=<substr> runs matching cases only, -tce=<substr>
// excludes matching cases (both may repeat). Summary lines mirror doctest's.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <sstream>
#include <stdexcept>
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
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};
template <typename T>
bool operator==(const T& x, const Approx& a) {
  return a.matches(static_cast<double>(x));
}
template <typename T>
bool operator==(const Approx& a, const T& x) {
  return a.matches(static_cast<double>(x));
}
template <typename T>
bool operator!=(const T& x, const Approx& a) {
  return !a.matches(static_cast<double>(x));
}
template <typename T>
bool operator!=(const Approx& a, const T& x) {
  return !a.matches(static_cast<double>(x));
}

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

struct State {
  long assertions = 0, failed_assertions = 0;
  bool case_failed = false;
  const TestCase* current = nullptr;
  std::vector<std::function<std::string()>> captures;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};  // unwinds a test case after a failed REQUIRE

inline void report(const char* file, int line, const char* kind, const char* expr, const std::string& extra) {
  State& s = state();
  ++s.failed_assertions;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) failed%s%s\n  in test case \"%s\"\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str(), s.current ? s.current->name : "?");
  for (auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c().c_str());
}

inline void check(bool ok, const char* file, int line, const char* kind, const char* expr, bool require) {
  ++state().assertions;
  if (ok) return;
  report(file, line, kind, expr, "");
  if (require) throw RequireAbort{};
}

template <typename T>
struct Capture {
  Capture(const char* name, const T& v) {
    state().captures.push_back([name, &v] {
      std::ostringstream os;
      os << name << " := " << v;
      return os.str();
    });
  }
  ~Capture() { state().captures.pop_back(); }
};

inline bool selected(const char* name, const std::vector<std::string>& inc, const std::vector<std::string>& exc) {
  for (auto& e : exc)
    if (std::strstr(name, e.c_str())) return false;
  if (inc.empty()) return true;
  for (auto& i : inc)
    if (std::strstr(name, i.c_str())) return true;
  return false;
}

inline int run(int argc, char** argv) {
  std::vector<std::string> inc, exc;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-tc=", 4)) inc.emplace_back(argv[i] + 4);
    if (!std::strncmp(argv[i], "-tce=", 5)) exc.emplace_back(argv[i] + 5);
  }
  State& s = state();
  int cases = 0, passed = 0, failed = 0, skipped = 0;
  for (const TestCase& tc : registry()) {
    if (!selected(tc.name, inc, exc)) {
      ++skipped;
      continue;
    }
    ++cases;
    s.current = &tc;
    s.case_failed = false;
    s.captures.clear();
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(tc.file, tc.line, "TEST_CASE", tc.name, "unexpected unknown exception");
    }
    if (s.case_failed) {
      ++failed;
      std::fprintf(stderr, "[doctest] FAILED: %s\n", tc.name);
    } else {
      ++passed;
      std::fprintf(stderr, "[doctest] passed: %s\n", tc.name);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", cases, passed, failed, skipped);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed |\n", s.assertions,
              s.assertions - s.failed_assertions, s.failed_assertions);
  std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
  return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_(fn, name)                                                        \
  static void fn();                                                                         \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(kind, require, ...) \
  ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, kind, #__VA_ARGS__, require)
#define CHECK(...) DOCTEST_ASSERT_("CHECK", false, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", true, __VA_ARGS__)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", true, !(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                             \
  do {                                                                                          \
    bool threw_right_ = false;                                                                  \
    try {                                                                                       \
      static_cast<void>(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                              \
      threw_right_ = true;                                                                      \
    } catch (...) {                                                                             \
    }                                                                                           \
    ::doctest::detail::check(threw_right_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
  } while (0)
#define FAIL(msg)                                                                              \
  do {                                                                                         \
    std::ostringstream os_;                                                                    \
    os_ << msg;                                                                                \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL", "", os_.str());                      \
    throw ::doctest::detail::RequireAbort{};                                                   \
  } while (0)
#define CAPTURE(x) ::doctest::detail::Capture<decltype(x)> DOCTEST_CAT(doctest_capture_, __COUNTER__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
