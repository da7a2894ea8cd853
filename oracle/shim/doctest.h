// TEST INFRASTRUCTURE ONLY (oracle/): a minimal restatement of the doctest
// macro surface used by the reference's unit tests (/root/reference/proj/tests,
// doctest itself is not vendored there: proj/.gitignore:2). Lets the
// reference's own test files run unmodified against (a) the compiled reference
// (oracle/_ref) and (b) this repo's C++ host port.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <algorithm>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& assertions() {
  static int a = 0;
  return a;
}
inline const char*& current_test() {
  static const char* c = "";
  return c;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(TestCase{name, file, line, fn});
  }
};

struct RequireFailure {};
struct ExplicitFailure {
  std::string msg;
};

inline void report(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED in [%s]: %s\n", file, line, current_test(), what.c_str());
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fname, name)                                                  \
  static void fname();                                                                       \
  static ::doctest::Registrar DOCTEST_CAT(fname, _reg)(name, __FILE__, __LINE__, &fname);    \
  static void fname()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_fn_, __COUNTER__), name)

#define CHECK(...)                                                                 \
  do {                                                                             \
    ++::doctest::assertions();                                                     \
    if (!(__VA_ARGS__)) ::doctest::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK_FALSE(...)                                                                 \
  do {                                                                                   \
    ++::doctest::assertions();                                                           \
    if ((__VA_ARGS__)) ::doctest::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE(...)                                                                      \
  do {                                                                                    \
    ++::doctest::assertions();                                                            \
    if (!(__VA_ARGS__)) {                                                                 \
      ::doctest::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");                 \
      throw ::doctest::RequireFailure{};                                                  \
    }                                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                       \
  do {                                                                                    \
    ++::doctest::assertions();                                                            \
    bool doctest_caught_ = false;                                                         \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const type&) {                                                               \
      doctest_caught_ = true;                                                             \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!doctest_caught_)                                                                 \
      ::doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")");     \
  } while (0)
#define CHECK_NOTHROW(...)                                                                \
  do {                                                                                    \
    ++::doctest::assertions();                                                            \
    try {                                                                                 \
      (void)(__VA_ARGS__);                                                                \
    } catch (const std::exception& e) {                                                   \
      ::doctest::report(__FILE__, __LINE__,                                               \
                        std::string("CHECK_NOTHROW(" #__VA_ARGS__ ") threw: ") + e.what()); \
    }                                                                                     \
  } while (0)
#define FAIL(msg)                                                           \
  do {                                                                      \
    ::doctest::report(__FILE__, __LINE__, std::string("FAIL: ") + (msg));   \
    throw ::doctest::ExplicitFailure{std::string(msg)};                     \
  } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int run = 0;
  for (const auto& tc : ::doctest::registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    ::doctest::current_test() = tc.name;
    ++run;
    try {
      tc.fn();
    } catch (const ::doctest::RequireFailure&) {
    } catch (const ::doctest::ExplicitFailure&) {
    } catch (const std::exception& e) {
      ::doctest::report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
    }
  }
  std::printf("[doctest-shim] test cases: %d | assertions: %d | failed: %d\n", run,
              ::doctest::assertions(), ::doctest::failures());
  return ::doctest::failures() == 0 ? 0 : 1;
}
#endif
