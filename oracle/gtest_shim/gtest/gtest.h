// Minimal GTest-compatible shim (GTest is not installed in this image).
// TEST INFRASTRUCTURE ONLY: lets the reference's own unit tests compile in
// place (oracle/Makefile target _ref/unit_tests) so the oracle is pinned to
// a reference that passes its own suite.  Supports the macros those files
// use: TEST, EXPECT_/ASSERT_{EQ,NE,LT,LE,GT,GE,TRUE,FALSE,NEAR,DOUBLE_EQ},
// EXPECT_THROW, EXPECT_NO_THROW, FAIL(), with << messages.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

namespace gts {
struct Case { const char* suite; const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};
struct Message {
  std::ostringstream s;
  template <class T> Message& operator<<(const T& v) { s << v; return *this; }
};
struct Helper {
  const char* file; int line; const char* text;
  void operator=(const Message& m) const {
    ++failures();
    std::printf("%s:%d: Failure: %s %s\n", file, line, text, m.s.str().c_str());
  }
};
inline bool double_eq(double a, double b) {
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if (ia < 0) ia = INT64_MIN - ia;
  if (ib < 0) ib = INT64_MIN - ib;
  const int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}
}  // namespace gts

#define GTS_CHECK_(cond, text) \
  if (cond) {                  \
  } else                       \
    ::gts::Helper{__FILE__, __LINE__, text} = ::gts::Message()
#define GTS_FATAL_(cond, text) \
  if (cond) {                  \
  } else                       \
    return ::gts::Helper{__FILE__, __LINE__, text} = ::gts::Message()

#define TEST(s, n)                                                            \
  static void gts_##s##_##n();                                                \
  static ::gts::Registrar gts_reg_##s##_##n(#s, #n, &gts_##s##_##n);          \
  static void gts_##s##_##n()

#define EXPECT_TRUE(c) GTS_CHECK_((c), #c)
#define EXPECT_FALSE(c) GTS_CHECK_(!(c), "!" #c)
#define EXPECT_EQ(a, b) GTS_CHECK_((a) == (b), #a " == " #b)
#define EXPECT_NE(a, b) GTS_CHECK_((a) != (b), #a " != " #b)
#define EXPECT_LT(a, b) GTS_CHECK_((a) < (b), #a " < " #b)
#define EXPECT_LE(a, b) GTS_CHECK_((a) <= (b), #a " <= " #b)
#define EXPECT_GT(a, b) GTS_CHECK_((a) > (b), #a " > " #b)
#define EXPECT_GE(a, b) GTS_CHECK_((a) >= (b), #a " >= " #b)
#define EXPECT_NEAR(a, b, t) GTS_CHECK_(std::fabs((a) - (b)) <= (t), #a " ~ " #b)
#define EXPECT_DOUBLE_EQ(a, b) GTS_CHECK_(::gts::double_eq((a), (b)), #a " ~= " #b)
#define ASSERT_TRUE(c) GTS_FATAL_((c), #c)
#define ASSERT_FALSE(c) GTS_FATAL_(!(c), "!" #c)
#define ASSERT_EQ(a, b) GTS_FATAL_((a) == (b), #a " == " #b)
#define ASSERT_NE(a, b) GTS_FATAL_((a) != (b), #a " != " #b)
#define ASSERT_LT(a, b) GTS_FATAL_((a) < (b), #a " < " #b)
#define ASSERT_LE(a, b) GTS_FATAL_((a) <= (b), #a " <= " #b)
#define ASSERT_GT(a, b) GTS_FATAL_((a) > (b), #a " > " #b)
#define ASSERT_GE(a, b) GTS_FATAL_((a) >= (b), #a " >= " #b)
#define ASSERT_DOUBLE_EQ(a, b) GTS_FATAL_(::gts::double_eq((a), (b)), #a " ~= " #b)
#define FAIL() return ::gts::Helper{__FILE__, __LINE__, "FAIL()"} = ::gts::Message()
#define EXPECT_THROW(stmt, exc)                                   \
  do {                                                            \
    bool gts_ok_ = false;                                         \
    try { stmt; } catch (const exc&) { gts_ok_ = true; } catch (...) {} \
    GTS_CHECK_(gts_ok_, "throws " #exc ": " #stmt);               \
  } while (0)
#define EXPECT_NO_THROW(stmt)                                     \
  do {                                                            \
    bool gts_ok_ = true;                                          \
    try { stmt; } catch (...) { gts_ok_ = false; }                \
    GTS_CHECK_(gts_ok_, "no throw: " #stmt);                      \
  } while (0)
