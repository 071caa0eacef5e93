// Minimal doctest-compatible shim (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which the reference git-ignores (proj/.gitignore:2 `vendor/`).
// This shim implements exactly the macro subset those tests use so that the
// reference suite -- and test_capi.cpp linked against OUR library -- can run
// here.  It is written from the doctest documentation's macro semantics, not
// from doctest sources.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  friend bool operator==(double lhs, const Approx& a) {
    const double scale = std::max(std::fabs(lhs), std::fabs(a.value_));
    return std::fabs(lhs - a.value_) <= a.eps_ * (1.0 + scale);
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }

 private:
  double value_;
  double eps_ = 1.1920929e-07f * 100;
};

namespace shim {

struct Registry {
  std::vector<std::pair<const char*, void (*)()>> cases;
  static Registry& get() { static Registry r; return r; }
};
struct Counters {
  long checks = 0, failures = 0;
  static Counters& get() { static Counters c; return c; }
};
struct RequireFailed {};
struct Registrar {
  Registrar(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};
inline void report(bool ok, bool fatal, const char* expr, const char* file, int line) {
  ++Counters::get().checks;
  if (ok) return;
  ++Counters::get().failures;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireFailed{};
}
inline int run_all() {
  int failed_cases = 0;
  for (auto& [name, fn] : Registry::get().cases) {
    const long before = Counters::get().failures;
    try {
      fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++Counters::get().failures;
      std::fprintf(stderr, "TEST_CASE(%s) threw: %s\n", name, e.what());
    }
    if (Counters::get().failures != before) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", name);
    }
  }
  std::printf("[shim] test cases: %zu | %zu passed | %d failed\n", Registry::get().cases.size(),
              Registry::get().cases.size() - failed_cases, failed_cases);
  std::printf("[shim] assertions: %ld | %ld passed | %ld failed\n", Counters::get().checks,
              Counters::get().checks - Counters::get().failures, Counters::get().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
  static void fn();                                                                 \
  static ::doctest::shim::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);               \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) ::doctest::shim::report(static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) ::doctest::shim::report(!static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define FAIL(msg) ::doctest::shim::report(false, true, msg, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, exc_type)                                             \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    try { (void)(expr); } catch (const exc_type&) { doctest_ok_ = true; } catch (...) {} \
    ::doctest::shim::report(doctest_ok_, false, #expr " throws " #exc_type, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
