// doctest.h -- a from-scratch stand-in for the subset of doctest that the reference's
// unit tests (reference proj/tests/test_*.cpp) use, so those files compile UNMODIFIED
// against the B200 facade. doctest itself is not in this image (reference
// proj/CMakeLists.txt:5 fetches it; proj/.gitignore:2 keeps it out of the tree).
//
// Supported: TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, REQUIRE,
// REQUIRE_FALSE, REQUIRE_MESSAGE, doctest::Approx, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// Output: one "[PASS]/[FAIL] <case>" line per test case and a final
// "<cases> test cases, <checks> checks, <failed> failed checks" line; exit status 1 on any
// failure. `--filter <substring>` runs only the matching cases.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v)
      : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.value_) <
           r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
  }
  friend bool operator==(const Approx& l, double rhs) { return rhs == l; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& l, double rhs) { return !(rhs == l); }

 private:
  double value_, eps_, scale_;
};

namespace detail {
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
struct Counters {
  long checks = 0, failed = 0;
};
inline Counters& counters() {
  static Counters c;
  return c;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireAbort {};
inline void record(bool ok, const char* file, int line, const char* what, const char* msg = nullptr) {
  ++counters().checks;
  if (ok) return;
  ++counters().failed;
  std::printf("  %s:%d: FAILED: %s%s%s\n", file, line, what, msg ? " -- " : "", msg ? msg : "");
}
inline int run(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], "--filter") == 0) filter = argv[i + 1];
  int cases = 0, bad_cases = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    long before = counters().failed;
    try {
      c.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      record(false, c.file, c.line, "uncaught exception", e.what());
    } catch (...) {
      record(false, c.file, c.line, "uncaught non-std exception");
    }
    bool ok = counters().failed == before;
    bad_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::printf("%d test cases (%d failed), %ld checks, %ld failed checks\n", cases, bad_cases,
              counters().checks, counters().failed);
  return counters().failed ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                      \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                       \
      name, __FILE__, __LINE__, DOCTEST_CAT(doctest_case_, __LINE__));                     \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) ::doctest::detail::record(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::doctest::detail::record(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE_MESSAGE(cond, msg)                                                          \
  do {                                                                                      \
    bool doctest_ok_ = static_cast<bool>(cond);                                             \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, #cond, msg);                \
    if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                             \
  } while (0)
#define REQUIRE(...) REQUIRE_MESSAGE((__VA_ARGS__), nullptr)
#define REQUIRE_FALSE(...) REQUIRE_MESSAGE(!(__VA_ARGS__), nullptr)
#define FAIL(msg)                                                                           \
  do {                                                                                      \
    ::doctest::detail::record(false, __FILE__, __LINE__, "FAIL", msg);                      \
    throw ::doctest::detail::RequireAbort{};                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                      \
    bool doctest_caught_ = false;                                                           \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (const __VA_ARGS__&) {                                                          \
      doctest_caught_ = true;                                                               \
    } catch (...) {                                                                         \
    }                                                                                       \
    ::doctest::detail::record(doctest_caught_, __FILE__, __LINE__,                          \
                              "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")");             \
  } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    try {                                                                                   \
      static_cast<void>(expr);                                                              \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
