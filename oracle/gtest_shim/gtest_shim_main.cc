// main() for the gtest shim (TEST INFRASTRUCTURE ONLY): runs every registered TEST and
// exits with the number of failed tests.
#include <gtest/gtest.h>

#include <exception>
#include <iostream>

int main() {
  int failed = 0;
  for (const auto& t : gtshim::Registry()) {
    gtshim::CurrentFailed() = false;
    try {
      t.body();
    } catch (const std::exception& e) {
      std::cout << "uncaught exception: " << e.what() << std::endl;
      gtshim::CurrentFailed() = true;
    }
    std::cout << (gtshim::CurrentFailed() ? "[  FAILED  ] " : "[       OK ] ") << t.suite << "."
              << t.name << std::endl;
    failed += gtshim::CurrentFailed() ? 1 : 0;
  }
  std::cout << "[==========] " << gtshim::Registry().size() << " tests, " << failed
            << " failed" << std::endl;
  return failed;
}
