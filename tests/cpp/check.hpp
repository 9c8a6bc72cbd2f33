// Minimal test harness for the C++ parity suites (Catch2 is not in the image).
// TEST_CASE / CHECK / REQUIRE / *_THROWS_AS with Catch-like semantics: CHECK
// records and continues, REQUIRE records and ends the test case.  The binary
// exits non-zero when any assertion failed; argv[1] filters cases by substring.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace chk {

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::printf("  FAILED %s:%d: %s\n", file, line, expr);
}

}  // namespace chk

#define CHK_CAT2(a, b) a##b
#define CHK_CAT(a, b) CHK_CAT2(a, b)
#define TEST_CASE(name, ...)                                                \
  static void CHK_CAT(chk_fn_, __LINE__)();                                 \
  static chk::Reg CHK_CAT(chk_reg_, __LINE__)(name, CHK_CAT(chk_fn_, __LINE__)); \
  static void CHK_CAT(chk_fn_, __LINE__)()

#define CHECK(x)                                         \
  do {                                                   \
    ++chk::checks();                                     \
    if (!(x)) chk::fail(__FILE__, __LINE__, #x);         \
  } while (0)
#define REQUIRE(x)                                       \
  do {                                                   \
    ++chk::checks();                                     \
    if (!(x)) {                                          \
      chk::fail(__FILE__, __LINE__, #x);                 \
      throw chk::Abort{};                                \
    }                                                    \
  } while (0)
#define CHECK_FALSE(x) CHECK(!(x))
#define REQUIRE_FALSE(x) REQUIRE(!(x))
#define CHK_THROWS_AS(expr, T, hard)                                          \
  do {                                                                       \
    ++chk::checks();                                                         \
    bool ok_ = false;                                                        \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const T&) {                                                     \
      ok_ = true;                                                            \
    } catch (...) {                                                          \
    }                                                                        \
    if (!ok_) {                                                              \
      chk::fail(__FILE__, __LINE__, "throws " #T ": " #expr);                \
      if (hard) throw chk::Abort{};                                          \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, T) CHK_THROWS_AS(expr, T, false)
#define REQUIRE_THROWS_AS(expr, T) CHK_THROWS_AS(expr, T, true)
#define REQUIRE_NOTHROW(expr)                                          \
  do {                                                                 \
    ++chk::checks();                                                   \
    try {                                                              \
      (void)(expr);                                                    \
    } catch (const std::exception& e_) {                               \
      chk::fail(__FILE__, __LINE__, (std::string("nothrow: ") + e_.what()).c_str()); \
      throw chk::Abort{};                                              \
    }                                                                  \
  } while (0)

int main(int argc, char** argv) {
  int run = 0, failed_cases = 0;
  for (const chk::Case& c : chk::cases()) {
    if (argc > 1 && std::strstr(c.name, argv[1]) == nullptr) continue;
    ++run;
    const int before = chk::failures();
    std::printf("[ RUN  ] %s\n", c.name);
    std::fflush(stdout);
    try {
      c.fn();
    } catch (const chk::Abort&) {
    } catch (const std::exception& e) {
      chk::fail(__FILE__, __LINE__, (std::string("unexpected exception: ") + e.what()).c_str());
    }
    const bool ok = chk::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[ %s ] %s\n", ok ? " OK " : "FAIL", c.name);
    std::fflush(stdout);
  }
  std::printf("%d cases, %d failed, %d assertions, %d assertion failures\n", run, failed_cases, chk::checks(),
              chk::failures());
  return chk::failures() == 0 ? 0 : 1;
}
