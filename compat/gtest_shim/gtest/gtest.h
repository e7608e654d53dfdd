// Minimal GoogleTest stand-in (NOT GoogleTest).
//
// The reference test suites (proj/tests/*.cpp, CMake `find_package(GTest)`)
// need GTest, which this image does not have. This header implements the
// subset those files use -- TEST / TEST_F, EXPECT_* / ASSERT_* with streamed
// messages, GTEST_SKIP, HasFailure / IsSkipped -- so the reference's own
// tests can be compiled verbatim and run against (a) the reference library
// (oracle/_ref, pins the Eigen stand-in) and (b) the GPU drop-in
// (paper_2012_12618_b200/csrc/rvk_dropin.cpp).
// Supports --gtest_filter=<substring>[:<substring>...] (substring match on
// "Suite.Name", '-' prefix list after ':-' excludes).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Test;

namespace internal {

struct TestInfo {
  std::string suite, name;
  std::function<Test*()> factory;
};

inline std::vector<TestInfo>& registry() {
  static std::vector<TestInfo> r;
  return r;
}

struct State {
  bool failed = false;
  bool skipped = false;
};
inline State& state() {
  static State s;
  return s;
}

struct Registrar {
  Registrar(const char* suite, const char* name, std::function<Test*()> f) {
    registry().push_back({suite, name, std::move(f)});
  }
};

// Collects a streamed message; reports on destruction.
class Reporter {
 public:
  Reporter(const char* file, int line, std::string what, bool skip = false)
      : file_(file), line_(line), what_(std::move(what)), skip_(skip) {}
  ~Reporter() {
    if (skip_) {
      state().skipped = true;
      std::cout << "[  SKIPPED ] " << file_ << ":" << line_ << " " << msg_.str() << "\n";
    } else {
      state().failed = true;
      std::cout << file_ << ":" << line_ << ": Failure\n" << what_ << "\n" << msg_.str() << "\n";
    }
  }
  template <class T>
  Reporter& operator<<(const T& v) {
    msg_ << v;
    return *this;
  }

 private:
  const char* file_;
  int line_;
  std::string what_;
  bool skip_;
  std::ostringstream msg_;
};

// Lets `return Reporter(...) << msg;` work inside void functions.
struct Voidify {
  void operator=(const Reporter&) {}
};

template <class T>
std::string show(const T& v) {
  if constexpr (requires(std::ostream& os, const T& x) { os << x; }) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

inline bool double_eq(double a, double b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  // 4 ULPs, as GoogleTest's AlmostEquals.
  auto biased = [](double x) {
    unsigned long long u;
    std::memcpy(&u, &x, sizeof u);
    const unsigned long long sign = 1ull << 63;
    return (u & sign) ? ~u + 1 : (u | sign);
  };
  const unsigned long long ua = biased(a), ub = biased(b);
  return (ua >= ub ? ua - ub : ub - ua) <= 4;
}
inline bool float_eq(float a, float b) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto biased = [](float x) {
    unsigned int u;
    std::memcpy(&u, &x, sizeof u);
    const unsigned int sign = 1u << 31;
    return (u & sign) ? ~u + 1 : (u | sign);
  };
  const unsigned int ua = biased(a), ub = biased(b);
  return (ua >= ub ? ua - ub : ub - ua) <= 4;
}

}  // namespace internal

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  static bool HasFailure() { return internal::state().failed; }
  static bool IsSkipped() { return internal::state().skipped; }
};

inline void InitGoogleTest(int*, char**) {}

inline bool filter_match(const std::string& full, const std::string& filter) {
  if (filter.empty() || filter == "*") return true;
  std::string pos = filter, neg;
  const auto dash = filter.find(":-");
  if (filter.rfind("-", 0) == 0) {
    pos.clear();
    neg = filter.substr(1);
  } else if (dash != std::string::npos) {
    pos = filter.substr(0, dash);
    neg = filter.substr(dash + 2);
  }
  auto any_of = [&](const std::string& list) {
    std::stringstream ss(list);
    std::string item;
    while (std::getline(ss, item, ':')) {
      std::string pat = item;
      pat.erase(std::remove(pat.begin(), pat.end(), '*'), pat.end());
      if (!pat.empty() && full.find(pat) != std::string::npos) return true;
    }
    return false;
  };
  if (!neg.empty() && any_of(neg)) return false;
  return pos.empty() || any_of(pos);
}

inline int RunAllTests(int argc, char** argv) {
  std::string filter;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  int passed = 0, failed = 0, skipped = 0;
  std::vector<std::string> failures;
  for (auto& t : internal::registry()) {
    const std::string full = t.suite + "." + t.name;
    if (!filter_match(full, filter)) continue;
    internal::state() = {};
    std::cout << "[ RUN      ] " << full << std::endl;
    Test* obj = t.factory();
    obj->SetUp();
    if (!internal::state().failed && !internal::state().skipped) {
      try {
        obj->TestBody();
      } catch (const std::exception& e) {
        internal::state().failed = true;
        std::cout << "uncaught exception: " << e.what() << "\n";
      } catch (...) {
        internal::state().failed = true;
        std::cout << "uncaught non-std exception\n";
      }
    }
    obj->TearDown();
    delete obj;
    if (internal::state().failed) {
      ++failed;
      failures.push_back(full);
      std::cout << "[  FAILED  ] " << full << std::endl;
    } else if (internal::state().skipped) {
      ++skipped;
      std::cout << "[  SKIPPED ] " << full << std::endl;
    } else {
      ++passed;
      std::cout << "[       OK ] " << full << std::endl;
    }
  }
  std::cout << "[==========] passed " << passed << ", failed " << failed << ", skipped " << skipped
            << std::endl;
  for (auto& f : failures) std::cout << "[  FAILED  ] " << f << std::endl;
  return failed == 0 ? 0 : 1;
}

}  // namespace testing

#define RUN_ALL_TESTS() ::testing::RunAllTests(gtest_argc_, gtest_argv_)

#define GTEST_SHIM_CLASS_(suite, name) suite##_##name##_Test

#define GTEST_SHIM_TEST_(suite, name, parent)                                              \
  class GTEST_SHIM_CLASS_(suite, name) : public parent {                                   \
   public:                                                                                 \
    void TestBody() override;                                                              \
  };                                                                                       \
  static ::testing::internal::Registrar gtest_shim_reg_##suite##_##name(                   \
      #suite, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS_(suite, name)); }); \
  void GTEST_SHIM_CLASS_(suite, name)::TestBody()

#define TEST(suite, name) GTEST_SHIM_TEST_(suite, name, ::testing::Test)
#define TEST_F(fixture, name) GTEST_SHIM_TEST_(fixture, name, fixture)

#define GTEST_SHIM_CHECK_(cond, text, on_fail) \
  if (cond) {                                  \
  } else                                       \
    on_fail ::testing::internal::Reporter(__FILE__, __LINE__, text)

#define GTEST_SHIM_NONFATAL_
#define GTEST_SHIM_FATAL_ return ::testing::internal::Voidify() =

#define GTEST_SHIM_BIN_(a, b, op, on_fail)                                                        \
  GTEST_SHIM_CHECK_(((a)op(b)),                                                                   \
                    std::string("Expected: (" #a ") " #op " (" #b "), actual: ") +                \
                        ::testing::internal::show(a) + " vs " + ::testing::internal::show(b),     \
                    on_fail)

#define EXPECT_EQ(a, b) GTEST_SHIM_BIN_(a, b, ==, GTEST_SHIM_NONFATAL_)
#define EXPECT_NE(a, b) GTEST_SHIM_BIN_(a, b, !=, GTEST_SHIM_NONFATAL_)
#define EXPECT_LT(a, b) GTEST_SHIM_BIN_(a, b, <, GTEST_SHIM_NONFATAL_)
#define EXPECT_LE(a, b) GTEST_SHIM_BIN_(a, b, <=, GTEST_SHIM_NONFATAL_)
#define EXPECT_GT(a, b) GTEST_SHIM_BIN_(a, b, >, GTEST_SHIM_NONFATAL_)
#define EXPECT_GE(a, b) GTEST_SHIM_BIN_(a, b, >=, GTEST_SHIM_NONFATAL_)
#define ASSERT_EQ(a, b) GTEST_SHIM_BIN_(a, b, ==, GTEST_SHIM_FATAL_)
#define ASSERT_NE(a, b) GTEST_SHIM_BIN_(a, b, !=, GTEST_SHIM_FATAL_)
#define ASSERT_LT(a, b) GTEST_SHIM_BIN_(a, b, <, GTEST_SHIM_FATAL_)
#define ASSERT_LE(a, b) GTEST_SHIM_BIN_(a, b, <=, GTEST_SHIM_FATAL_)
#define ASSERT_GT(a, b) GTEST_SHIM_BIN_(a, b, >, GTEST_SHIM_FATAL_)
#define ASSERT_GE(a, b) GTEST_SHIM_BIN_(a, b, >=, GTEST_SHIM_FATAL_)

#define EXPECT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_NONFATAL_)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_NONFATAL_)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_FATAL_)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_FATAL_)

#define GTEST_SHIM_NEAR_(a, b, tol, on_fail)                                                    \
  GTEST_SHIM_CHECK_((std::abs(static_cast<double>(a) - static_cast<double>(b)) <=               \
                     static_cast<double>(tol)),                                                 \
                    std::string("Expected |" #a " - " #b "| <= " #tol ", actual: ") +           \
                        ::testing::internal::show(a) + " vs " + ::testing::internal::show(b),   \
                    on_fail)
#define EXPECT_NEAR(a, b, tol) GTEST_SHIM_NEAR_(a, b, tol, GTEST_SHIM_NONFATAL_)
#define ASSERT_NEAR(a, b, tol) GTEST_SHIM_NEAR_(a, b, tol, GTEST_SHIM_FATAL_)

#define EXPECT_DOUBLE_EQ(a, b)                                                              \
  GTEST_SHIM_CHECK_(::testing::internal::double_eq((a), (b)),                               \
                    std::string("Expected double equality " #a " == " #b ", actual: ") +   \
                        ::testing::internal::show(a) + " vs " + ::testing::internal::show(b), \
                    GTEST_SHIM_NONFATAL_)
#define ASSERT_DOUBLE_EQ(a, b)                                                              \
  GTEST_SHIM_CHECK_(::testing::internal::double_eq((a), (b)),                               \
                    std::string("Expected double equality " #a " == " #b), GTEST_SHIM_FATAL_)
#define EXPECT_FLOAT_EQ(a, b)                                                               \
  GTEST_SHIM_CHECK_(::testing::internal::float_eq((a), (b)),                                \
                    std::string("Expected float equality " #a " == " #b), GTEST_SHIM_NONFATAL_)

#define GTEST_SHIM_THROW_(stmt, exc, on_fail)                   \
  GTEST_SHIM_CHECK_(([&]() -> bool {                            \
                      try {                                     \
                        stmt;                                   \
                      } catch (const exc&) {                    \
                        return true;                            \
                      } catch (...) {                           \
                        return false;                           \
                      }                                         \
                      return false;                             \
                    }()),                                       \
                    "Expected " #stmt " to throw " #exc, on_fail)
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_FATAL_)

#define GTEST_SHIM_NO_THROW_(stmt, on_fail)                     \
  GTEST_SHIM_CHECK_(([&]() -> bool {                            \
                      try {                                     \
                        stmt;                                   \
                      } catch (...) {                           \
                        return false;                           \
                      }                                         \
                      return true;                              \
                    }()),                                       \
                    "Expected " #stmt " not to throw", on_fail)
#define EXPECT_NO_THROW(stmt) GTEST_SHIM_NO_THROW_(stmt, GTEST_SHIM_NONFATAL_)
#define ASSERT_NO_THROW(stmt) GTEST_SHIM_NO_THROW_(stmt, GTEST_SHIM_FATAL_)

#define GTEST_SKIP() \
  return ::testing::internal::Voidify() = ::testing::internal::Reporter(__FILE__, __LINE__, "", true)
