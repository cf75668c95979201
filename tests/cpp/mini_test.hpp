// mini_test.hpp -- a tiny TEST_CASE / CHECK harness so the facade tests read like the
// reference's doctest suites (proj/tests/*.cpp) without the absent doctest.h.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Abort {};
inline void fail(const char* file, int line, const std::string& what) {
  std::printf("  FAIL %s:%d: %s\n", file, line, what.c_str());
  ++failures();
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                      \
  static void MINI_CAT(mini_case_, __LINE__)();                              \
  static mini::Reg MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
  static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(expr) \
  do { if (!(expr)) mini::fail(__FILE__, __LINE__, #expr); } while (0)
#define REQUIRE(expr) \
  do { if (!(expr)) { mini::fail(__FILE__, __LINE__, #expr); throw mini::Abort{}; } } while (0)
#define CHECK_THROWS_AS(expr, Type)                                            \
  do {                                                                         \
    bool caught_ = false;                                                      \
    try { (void)(expr); } catch (const Type&) { caught_ = true; } catch (...) {} \
    if (!caught_) mini::fail(__FILE__, __LINE__, "expected " #Type " from " #expr); \
  } while (0)

inline int mini_main() {
  int cases = 0;
  for (auto& c : mini::registry()) {
    int before = mini::failures();
    try {
      c.fn();
    } catch (const mini::Abort&) {
    } catch (const std::exception& e) {
      mini::fail(c.name, 0, std::string("uncaught exception: ") + e.what());
    }
    std::printf("[%s] %s\n", mini::failures() == before ? "PASS" : "FAIL", c.name);
    ++cases;
  }
  std::printf("%d cases, %d failed checks\n", cases, mini::failures());
  return mini::failures() ? 1 : 0;
}
