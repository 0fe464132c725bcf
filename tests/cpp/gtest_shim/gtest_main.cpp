// main() of the GoogleTest stand-in: runs every TEST, prints one line per
// case and "<passed> passed, <failed> failed".
#include <cstdio>

#include "gtest/gtest.h"

int main() {
  int passed = 0, failed = 0;
  for (const auto& c : ::gshim::registry()) {
    const int before = ::gshim::failures();
    try {
      c.fn();
    } catch (const ::gshim::AssertAbort&) {
    } catch (const std::exception& e) {
      ++::gshim::failures();
      std::printf("  EXCEPTION %s\n", e.what());
    }
    const bool ok = ::gshim::failures() == before;
    std::printf("[%s] %s.%s\n", ok ? "  OK  " : " FAIL ", c.suite, c.name);
    (ok ? passed : failed)++;
  }
  std::printf("%d passed, %d failed\n", passed, failed);
  return failed == 0 ? 0 : 1;
}
