// Minimal doctest-compatible test harness -- TEST INFRASTRUCTURE ONLY.
//
// doctest itself is not vendored with the reference (vendor/ is absent). This
// stand-in implements the subset the reference's unit suites use (TEST_CASE,
// CHECK[_FALSE], REQUIRE, CHECK_THROWS[_AS], CHECK_NOTHROW, INFO,
// doctest::Approx) so those suites can be compiled unchanged -- against the
// reference headers (oracle) or against the B200 drop-in (include/tslb).
// Exit status: number of failed test cases (0 = all passed).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
  }
  double value() const { return v_; }

 private:
  double v_;
  double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

template <typename T>
bool operator==(const T& x, const Approx& a) {
  return a.matches(double(x));
}
template <typename T>
bool operator==(const Approx& a, const T& x) {
  return a.matches(double(x));
}
template <typename T>
bool operator!=(const T& x, const Approx& a) {
  return !a.matches(double(x));
}
template <typename T>
bool operator!=(const Approx& a, const T& x) {
  return !a.matches(double(x));
}

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};
struct RequireFailed {};
inline int& case_failures() {
  static int n = 0;
  return n;
}
inline long& assertions() {
  static long n = 0;
  return n;
}
inline std::vector<std::string>& info_stack() {
  static std::vector<std::string> s;
  return s;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++assertions();
  if (ok) return;
  ++case_failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  for (const auto& s : info_stack()) std::fprintf(stderr, "  info: %s\n", s.c_str());
  if (fatal) throw RequireFailed{};
}
struct InfoScope {
  template <typename... A>
  explicit InfoScope(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    info_stack().push_back(os.str());
  }
  ~InfoScope() { info_stack().pop_back(); }
};
inline int run_all() {
  int failed = 0;
  for (const auto& c : registry()) {
    case_failures() = 0;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++case_failures();
      std::fprintf(stderr, "%s:%d: exception in \"%s\": %s\n", c.file, c.line, c.name, e.what());
    }
    if (case_failures()) {
      ++failed;
      std::fprintf(stderr, "[FAIL] %s\n", c.name);
    } else {
      std::printf("[ ok ] %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | %ld assertions\n",
              registry().size(), registry().size() - size_t(failed), failed, assertions());
  return failed;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name) TEST_CASE_IMPL_(name, DOCTEST_CAT(doctest_case_, __LINE__))
#define TEST_CASE_IMPL_(name, fn)                                                   \
  static void fn();                                                                 \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()

#define CHECK(...) ::doctest::detail::report(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!bool(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define INFO(...) ::doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(__VA_ARGS__)
#define CHECK_THROWS(...)                                                            \
  do {                                                                               \
    bool thrown_ = false;                                                            \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      thrown_ = true;                                                                \
    }                                                                                \
    ::doctest::detail::report(thrown_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                  \
  do {                                                                               \
    bool thrown_ = false;                                                            \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type&) {                                                          \
      thrown_ = true;                                                                \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
// doctest: passes when expr throws `type` whose what() equals the message
#define CHECK_THROWS_WITH_AS(expr, message, type)                                   \
  do {                                                                               \
    bool ok_ = false;                                                                \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const type& e_) {                                                       \
      ok_ = std::string(e_.what()) == std::string(message);                          \
    } catch (...) {                                                                  \
    }                                                                                \
    ::doctest::detail::report(ok_, "throws " #type " with " #message ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(...)                                                           \
  do {                                                                               \
    bool ok_ = true;                                                                 \
    try {                                                                            \
      (void)(__VA_ARGS__);                                                           \
    } catch (...) {                                                                  \
      ok_ = false;                                                                   \
    }                                                                                \
    ::doctest::detail::report(ok_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
