// Runner for the GTest shim (TEST INFRASTRUCTURE ONLY).
#include <cstdio>

#include "gtest/gtest.h"

int main() {
  int failed_cases = 0;
  for (const auto& c : gts::registry()) {
    const int before = gts::failures();
    c.fn();
    const bool ok = gts::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s.%s\n", ok ? "  OK  " : "FAILED", c.suite, c.name);
  }
  std::printf("%zu tests, %d failed\n", gts::registry().size(), failed_cases);
  return failed_cases == 0 ? 0 : 1;
}
