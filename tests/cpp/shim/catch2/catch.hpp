// catch2/catch.hpp — TEST INFRASTRUCTURE: the small subset of the Catch2 v2
// API that the reference's unit tests use (TEST_CASE, SECTION, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL), so that
// /root/reference/proj/tests/test_*.cpp compile unchanged against the B200
// drop-in headers (Catch2 itself is not in this image). Semantics follow
// Catch2 for non-nested sections: a test case runs once per SECTION (code
// outside sections every time); REQUIRE / FAIL end the current run.
// main() is in tests/cpp/ref_tests_main.cpp.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini_catch {

struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
  int target = 0, seen = 0;
  long checks = 0, failures = 0;
  const char* current = "";
};
inline State& state() {
  static State s;
  return s;
}

struct Section {
  bool active;
  explicit Section(const char*) { active = state().seen++ == state().target; }
};

struct Abort {};

inline void report(bool ok, const char* what, const char* file, int line) {
  ++state().checks;
  if (!ok) {
    ++state().failures;
    std::fprintf(stderr, "FAILED [%s] %s:%d: %s\n", state().current, file, line, what);
  }
}

}  // namespace mini_catch

#define MC_CAT2(a, b) a##b
#define MC_CAT(a, b) MC_CAT2(a, b)
#define TEST_CASE(name, ...)                                                                 \
  static void MC_CAT(mc_test_, __LINE__)();                                                  \
  static ::mini_catch::Reg MC_CAT(mc_reg_, __LINE__)(name, &MC_CAT(mc_test_, __LINE__));     \
  static void MC_CAT(mc_test_, __LINE__)()
#define SECTION(name) if (::mini_catch::Section mc_sec_{name}; mc_sec_.active)
#define CHECK(...) ::mini_catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::mini_catch::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
  do {                                                                                \
    const bool mc_ok_ = static_cast<bool>(__VA_ARGS__);                               \
    ::mini_catch::report(mc_ok_, #__VA_ARGS__, __FILE__, __LINE__);                   \
    if (!mc_ok_) throw ::mini_catch::Abort{};                                         \
  } while (0)
#define FAIL(msg)                                                  \
  do {                                                             \
    ::mini_catch::report(false, msg, __FILE__, __LINE__);          \
    throw ::mini_catch::Abort{};                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                               \
  do {                                                                                            \
    bool mc_ok_ = false;                                                                          \
    try {                                                                                         \
      (void)(expr);                                                                               \
    } catch (const type&) {                                                                       \
      mc_ok_ = true;                                                                              \
    } catch (...) {                                                                               \
    }                                                                                             \
    ::mini_catch::report(mc_ok_, #expr " throws " #type, __FILE__, __LINE__);                     \
  } while (0)
#define CHECK_NOTHROW(expr)                                        \
  do {                                                             \
    bool mc_ok_ = true;                                            \
    try {                                                          \
      (void)(expr);                                                \
    } catch (...) {                                                \
      mc_ok_ = false;                                              \
    }                                                              \
    ::mini_catch::report(mc_ok_, #expr " does not throw", __FILE__, __LINE__); \
  } while (0)
