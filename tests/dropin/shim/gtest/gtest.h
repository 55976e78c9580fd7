// Minimal GoogleTest-compatible harness (own implementation; GTest is not
// installed in this image). Supports what the reference suites use: TEST,
// EXPECT_/ASSERT_ EQ NE LT LE GT GE NEAR DOUBLE_EQ TRUE FALSE THROW
// NO_THROW, SCOPED_TRACE and streamed messages. main() runs every test in
// registration order and exits non-zero on any failure.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace gshim {

struct Registry {
  struct Test {
    std::string suite, name;
    std::function<void()> fn;
  };
  std::vector<Test> tests;
  std::vector<std::string> trace;
  int failures_in_test = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

struct Registrar {
  Registrar(const char* s, const char* n, std::function<void()> f) {
    Registry::get().tests.push_back({s, n, std::move(f)});
  }
};

struct AssertAbort {};

class Failure {
 public:
  Failure(const char* file, int line, std::string what, bool fatal) : fatal_(fatal) {
    msg_ << file << ":" << line << ": Failure\n" << what;
  }
  template <class T>
  Failure& operator<<(const T& v) {
    extra_ << v;
    return *this;
  }
  ~Failure() noexcept(false) {
    auto& R = Registry::get();
    std::cerr << msg_.str();
    if (!extra_.str().empty()) std::cerr << "\n  " << extra_.str();
    for (auto& t : R.trace) std::cerr << "\n  trace: " << t;
    std::cerr << "\n";
    ++R.failures_in_test;
    if (fatal_) throw AssertAbort{};
  }

 private:
  bool fatal_;
  std::ostringstream msg_, extra_;
};

struct ScopedTrace {
  explicit ScopedTrace(std::string s) { Registry::get().trace.push_back(std::move(s)); }
  ~ScopedTrace() { Registry::get().trace.pop_back(); }
};

template <class A, class B>
std::string describe(const char* ea, const char* eb, const A& a, const B& b) {
  std::ostringstream o;
  o.precision(17);
  o << "  " << ea << " = " << a << "\n  " << eb << " = " << b;
  return o.str();
}

inline bool almost_equal_ulps(double a, double b) {
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  std::int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if ((ia < 0) != (ib < 0)) return false;
  const std::int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}

}  // namespace gshim

#define GS_CAT2(a, b) a##b
#define GS_CAT(a, b) GS_CAT2(a, b)
#define TEST(suite, name)                                                              \
  static void GS_CAT(gs_test_##suite##_, name)();                                      \
  static ::gshim::Registrar GS_CAT(gs_reg_##suite##_, name)(#suite, #name,            \
                                                           GS_CAT(gs_test_##suite##_, name)); \
  static void GS_CAT(gs_test_##suite##_, name)()

#define GS_CHECK(cond, what, fatal) \
  if (cond) {                       \
  } else                            \
    ::gshim::Failure(__FILE__, __LINE__, what, fatal)

#define GS_BIN(a, b, op, fatal)                                                             \
  GS_CHECK(((a)op(b)), ::gshim::describe(#a, #b, (a), (b)) + "\n  expected " #a " " #op " " #b, fatal)

#define EXPECT_EQ(a, b) GS_BIN(a, b, ==, false)
#define EXPECT_NE(a, b) GS_BIN(a, b, !=, false)
#define EXPECT_LT(a, b) GS_BIN(a, b, <, false)
#define EXPECT_LE(a, b) GS_BIN(a, b, <=, false)
#define EXPECT_GT(a, b) GS_BIN(a, b, >, false)
#define EXPECT_GE(a, b) GS_BIN(a, b, >=, false)
#define ASSERT_EQ(a, b) GS_BIN(a, b, ==, true)
#define ASSERT_LE(a, b) GS_BIN(a, b, <=, true)
#define ASSERT_TRUE(c) GS_CHECK(static_cast<bool>(c), "  expected true: " #c, true)
#define EXPECT_TRUE(c) GS_CHECK(static_cast<bool>(c), "  expected true: " #c, false)
#define EXPECT_FALSE(c) GS_CHECK(!static_cast<bool>(c), "  expected false: " #c, false)
#define EXPECT_NEAR(a, b, tol)                                                         \
  GS_CHECK(std::abs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
           ::gshim::describe(#a, #b, (a), (b)) + "\n  tolerance " #tol, false)
#define EXPECT_DOUBLE_EQ(a, b) \
  GS_CHECK(::gshim::almost_equal_ulps((a), (b)), ::gshim::describe(#a, #b, (a), (b)) + "\n  (4 ulp)", false)
#define EXPECT_THROW(stmt, exc)                                       \
  do {                                                                \
    bool gs_caught = false;                                           \
    try {                                                             \
      stmt;                                                           \
    } catch (const exc&) {                                            \
      gs_caught = true;                                               \
    } catch (...) {                                                   \
    }                                                                 \
    GS_CHECK(gs_caught, "  expected " #stmt " to throw " #exc, false); \
  } while (0)
#define EXPECT_NO_THROW(stmt)                                            \
  do {                                                                   \
    bool gs_ok = true;                                                   \
    try {                                                                \
      stmt;                                                              \
    } catch (...) {                                                      \
      gs_ok = false;                                                     \
    }                                                                    \
    GS_CHECK(gs_ok, "  expected " #stmt " not to throw", false);         \
  } while (0)
#define SCOPED_TRACE(msg) ::gshim::ScopedTrace GS_CAT(gs_trace_, __LINE__)(msg)

int main(int argc, char** argv) {
  auto& R = gshim::Registry::get();
  int failed = 0;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  for (auto& t : R.tests) {
    const std::string full = t.suite + "." + t.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    R.failures_in_test = 0;
    try {
      t.fn();
    } catch (const gshim::AssertAbort&) {
    } catch (const std::exception& e) {
      std::cerr << full << ": uncaught exception: " << e.what() << "\n";
      ++R.failures_in_test;
    }
    std::cout << (R.failures_in_test ? "[  FAILED  ] " : "[       OK ] ") << full << std::endl;
    if (R.failures_in_test) ++failed;
  }
  std::cout << (failed ? "FAILED " : "PASSED ") << (R.tests.size() - failed) << "/" << R.tests.size()
            << " tests" << std::endl;
  return failed ? 1 : 0;
}
