// ref_tests_main.cpp — TEST INFRASTRUCTURE: runner for the reference's own
// Catch2 unit tests (/root/reference/proj/tests/test_ebe.cpp, test_solver.cpp)
// compiled unchanged against the B200 drop-in headers (include/tetsolve/)
// with the mini Catch2 / Eigen shims in tests/cpp/shim. Runs every test case
// once per SECTION and prints one JSON summary line.
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch2/catch.hpp"

int main(int argc, char** argv) {
  using namespace mini_catch;
  const char* only = argc > 1 ? argv[1] : nullptr;
  long cases = 0, runs = 0, errors = 0;
  for (const Case& c : registry()) {
    if (only && !std::strstr(c.name, only)) continue;
    ++cases;
    state().current = c.name;
    for (int target = 0;; ++target) {
      state().target = target;
      state().seen = 0;
      ++runs;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        ++errors;
        ++state().failures;
        std::fprintf(stderr, "FAILED [%s] unexpected exception: %s\n", c.name, e.what());
      }
      if (state().seen <= target + 1) break;  // no further sections
    }
    std::fprintf(stderr, "ran: %s\n", c.name);
  }
  std::printf("{\"test_cases\": %ld, \"runs\": %ld, \"checks\": %ld, \"failures\": %ld, \"exceptions\": %ld}\n", cases,
              runs, state().checks, state().failures, errors);
  return state().failures ? 1 : 0;
}
