// Minimal stand-in for the GoogleTest API the reference's unit tests use
// (TEST, EXPECT_/ASSERT_ EQ, TRUE, DOUBLE_EQ, NEAR, THROW, streamed
// messages).  GoogleTest is not in this image; the reference's tests
// (/root/reference/proj/tests/test_*.cpp) compile against it unmodified.
#pragma once
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {
struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
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
  Reg(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};
struct AssertAbort {};
// Collects a streamed message; reports on destruction (the failure already happened).
class Failure {
 public:
  Failure(const char* file, int line, std::string what, bool fatal)
      : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
  template <class T>
  Failure& operator<<(const T& x) {
    os_ << x;
    return *this;
  }
  ~Failure() noexcept(false) {
    ++failures();
    std::printf("  FAILED %s:%d: %s %s\n", file_, line_, what_.c_str(), os_.str().c_str());
    if (fatal_) throw AssertAbort{};
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  bool fatal_;
  std::ostringstream os_;
};
struct Null {
  template <class T>
  Null& operator<<(const T&) {
    return *this;
  }
};
inline bool double_eq(double a, double b) {   // within 4 ULPs, as GoogleTest
  if (std::isnan(a) || std::isnan(b)) return false;
  auto biased = [](double x) {
    long long i;
    std::memcpy(&i, &x, sizeof(i));
    return i < 0 ? (long long)(~0ull >> 1) - i + 1 : i + (long long)(~0ull >> 1) + 1;
  };
  const unsigned long long ua = (unsigned long long)biased(a), ub = (unsigned long long)biased(b);
  return (ua > ub ? ua - ub : ub - ua) <= 4;
}
}  // namespace gshim

#define GSHIM_CHECK(cond, what, fatal) \
  if (cond)                            \
    ;                                  \
  else                                 \
    ::gshim::Failure(__FILE__, __LINE__, what, fatal)

#define TEST(suite, name)                                                   \
  static void gshim_##suite##_##name();                                     \
  static ::gshim::Reg gshim_reg_##suite##_##name(#suite, #name,             \
                                                 &gshim_##suite##_##name);  \
  static void gshim_##suite##_##name()

#define EXPECT_EQ(a, b) GSHIM_CHECK((a) == (b), "EXPECT_EQ(" #a ", " #b ")", false)
#define ASSERT_EQ(a, b) GSHIM_CHECK((a) == (b), "ASSERT_EQ(" #a ", " #b ")", true)
#define EXPECT_TRUE(c) GSHIM_CHECK((c), "EXPECT_TRUE(" #c ")", false)
#define ASSERT_TRUE(c) GSHIM_CHECK((c), "ASSERT_TRUE(" #c ")", true)
#define EXPECT_DOUBLE_EQ(a, b) \
  GSHIM_CHECK(::gshim::double_eq((a), (b)), "EXPECT_DOUBLE_EQ(" #a ", " #b ")", false)
#define EXPECT_NEAR(a, b, tol) \
  GSHIM_CHECK(std::fabs((a) - (b)) <= (tol), "EXPECT_NEAR(" #a ", " #b ")", false)
#define EXPECT_THROW(stmt, exc)                            \
  GSHIM_CHECK(([&] {                                       \
                try {                                      \
                  stmt;                                    \
                } catch (const exc&) {                     \
                  return true;                             \
                } catch (...) {                            \
                }                                          \
                return false;                              \
              }()),                                        \
              "EXPECT_THROW(" #stmt ", " #exc ")", false)
