// Minimal GoogleTest-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// GTest is not installed in this image, so the reference's own gtest suites
// (/root/reference/proj/tests/*_test.cc) cannot be built as shipped.  This header
// implements just the subset of the gtest API those suites use (TEST, EXPECT_/ASSERT_ EQ NE
// LT LE GT GE TRUE FALSE DOUBLE_EQ NEAR THROW, FAIL, testing::TempDir) so that the suites
// compile unmodified against either planner (the reference's, or this repo's drop-in) and
// report failures with file:line.  main() is provided by gtest_shim_main.cc.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace gtshim {

struct TestCase {
  const char* suite;
  const char* name;
  void (*body)();
};

inline std::vector<TestCase>& Registry() {
  static std::vector<TestCase> r;
  return r;
}

inline bool& CurrentFailed() {
  static bool failed = false;
  return failed;
}

struct Registrar {
  Registrar(const char* suite, const char* name, void (*body)()) {
    Registry().push_back({suite, name, body});
  }
};

class Message {
 public:
  Message() = default;
  Message(const Message& o) { os_ << o.os_.str(); }
  template <typename T>
  Message& operator<<(const T& v) {
    os_ << v;
    return *this;
  }
  std::string str() const { return os_.str(); }

 private:
  std::ostringstream os_;
};

class Reporter {
 public:
  Reporter(const char* file, int line, std::string what)
      : file_(file), line_(line), what_(std::move(what)) {}
  void operator=(const Message& m) const {
    CurrentFailed() = true;
    std::cout << file_ << ":" << line_ << ": Failure\n  " << what_;
    const std::string extra = m.str();
    if (!extra.empty()) std::cout << "\n  " << extra;
    std::cout << std::endl;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
};

// gtest's EXPECT_DOUBLE_EQ: equal within 4 units in the last place.
inline bool AlmostEqualUlps(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](double x) {
    int64_t i;
    std::memcpy(&i, &x, sizeof(i));
    const uint64_t u = static_cast<uint64_t>(i);
    const uint64_t sign = uint64_t{1} << 63;
    return (u & sign) ? ~u + 1 : (u | sign);
  };
  const uint64_t x = biased(a), y = biased(b);
  return (x >= y ? x - y : y - x) <= 4;
}

}  // namespace gtshim

namespace testing {
inline std::string TempDir() { return "/tmp/"; }
}  // namespace testing

#define GTSHIM_CAT2(a, b) a##b
#define GTSHIM_CAT(a, b) GTSHIM_CAT2(a, b)

#define TEST(suite, name)                                                             \
  static void GTSHIM_CAT(GTSHIM_CAT(suite##_, name), _body)();                       \
  static ::gtshim::Registrar GTSHIM_CAT(GTSHIM_CAT(suite##_, name), _registrar)(      \
      #suite, #name, &GTSHIM_CAT(GTSHIM_CAT(suite##_, name), _body));                 \
  static void GTSHIM_CAT(GTSHIM_CAT(suite##_, name), _body)()

#define GTSHIM_NONFATAL(cond, text) \
  switch (0)                        \
  case 0:                           \
  default:                          \
    if (cond)                       \
      ;                             \
    else                            \
      ::gtshim::Reporter(__FILE__, __LINE__, text) = ::gtshim::Message()

#define GTSHIM_FATAL(cond, text) \
  switch (0)                     \
  case 0:                        \
  default:                       \
    if (cond)                    \
      ;                          \
    else                         \
      return ::gtshim::Reporter(__FILE__, __LINE__, text) = ::gtshim::Message()

#define EXPECT_TRUE(c) GTSHIM_NONFATAL(static_cast<bool>(c), "expected true: " #c)
#define EXPECT_FALSE(c) GTSHIM_NONFATAL(!static_cast<bool>(c), "expected false: " #c)
#define EXPECT_EQ(a, b) GTSHIM_NONFATAL((a) == (b), "expected " #a " == " #b)
#define EXPECT_NE(a, b) GTSHIM_NONFATAL((a) != (b), "expected " #a " != " #b)
#define EXPECT_LT(a, b) GTSHIM_NONFATAL((a) < (b), "expected " #a " < " #b)
#define EXPECT_LE(a, b) GTSHIM_NONFATAL((a) <= (b), "expected " #a " <= " #b)
#define EXPECT_GT(a, b) GTSHIM_NONFATAL((a) > (b), "expected " #a " > " #b)
#define EXPECT_GE(a, b) GTSHIM_NONFATAL((a) >= (b), "expected " #a " >= " #b)
#define EXPECT_DOUBLE_EQ(a, b) \
  GTSHIM_NONFATAL(::gtshim::AlmostEqualUlps((a), (b)), "expected " #a " ~= " #b " (4 ulp)")
#define EXPECT_NEAR(a, b, tol) \
  GTSHIM_NONFATAL(std::fabs((a) - (b)) <= (tol), "expected |" #a " - " #b "| <= " #tol)

#define ASSERT_TRUE(c) GTSHIM_FATAL(static_cast<bool>(c), "expected true: " #c)
#define ASSERT_FALSE(c) GTSHIM_FATAL(!static_cast<bool>(c), "expected false: " #c)
#define ASSERT_EQ(a, b) GTSHIM_FATAL((a) == (b), "expected " #a " == " #b)
#define ASSERT_NE(a, b) GTSHIM_FATAL((a) != (b), "expected " #a " != " #b)
#define ASSERT_LT(a, b) GTSHIM_FATAL((a) < (b), "expected " #a " < " #b)
#define ASSERT_LE(a, b) GTSHIM_FATAL((a) <= (b), "expected " #a " <= " #b)
#define ASSERT_GT(a, b) GTSHIM_FATAL((a) > (b), "expected " #a " > " #b)
#define ASSERT_GE(a, b) GTSHIM_FATAL((a) >= (b), "expected " #a " >= " #b)

#define FAIL() return ::gtshim::Reporter(__FILE__, __LINE__, "FAIL()") = ::gtshim::Message()

#define EXPECT_THROW(stmt, exc)                                       \
  do {                                                                \
    int gtshim_state = 0;                                             \
    try {                                                             \
      stmt;                                                           \
    } catch (const exc&) {                                            \
      gtshim_state = 1;                                               \
    } catch (...) {                                                   \
      gtshim_state = 2;                                               \
    }                                                                 \
    if (gtshim_state != 1)                                            \
      ::gtshim::Reporter(__FILE__, __LINE__,                          \
                         gtshim_state == 0 ? "no exception: " #stmt  \
                                           : "wrong exception: " #stmt) = \
          ::gtshim::Message();                                        \
  } while (0)
