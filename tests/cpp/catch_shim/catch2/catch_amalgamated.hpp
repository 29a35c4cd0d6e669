// Minimal stand-in for the subset of Catch2 v3 the reference's unit tests use
// (TEST_CASE, CHECK, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, INFO, Approx).
// TEST INFRASTRUCTURE ONLY: it lets /root/reference/proj/tests/test_{pq,index,vq}.cpp
// compile unmodified against the drop-in headers (include/anisoq/) and run on
// the B200 (tests/test_reference_suite_gpu.py). Catch2 is not installed here.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
  long assertions = 0;
  long failures = 0;
  std::string info;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   bool fatal) {
  ++state().assertions;
  if (ok) return;
  ++state().failures;
  std::printf("  FAILED %s( %s ) at %s:%d%s%s\n", kind, expr, file, line,
              state().info.empty() ? "" : "  with ", state().info.c_str());
  if (fatal) throw RequireFailed{};
}

struct InfoScope {
  std::string saved;
  explicit InfoScope(const std::string& s) : saved(state().info) { state().info = s; }
  ~InfoScope() { state().info = saved; }
};

}  // namespace catch_shim

namespace Catch {

// Catch2 v3 Approx semantics: |a - b| <= margin, or
// |a - b| <= epsilon * (scale + |value|) (value = the Approx's own operand).
class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(std::numeric_limits<float>::epsilon() * 100.0), margin_(0.0),
        scale_(0.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool equals(double other) const {
    const auto within = [](double a, double b, double m) {
      return (a + m >= b) && (b + m >= a);
    };
    return within(value_, other, margin_) ||
           within(value_, other,
                  epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.equals(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.equals(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.equals(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.equals(rhs); }
  friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.equals(lhs); }
  friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.equals(lhs); }

 private:
  double value_, epsilon_, margin_, scale_;
};

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST(fn, name)                                          \
  static void fn();                                                        \
  static const ::catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg){name, fn}; \
  static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TEST(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)

#define CHECK(...) ::catch_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::catch_shim::report(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) ::catch_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) ::catch_shim::report(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CATCH_SHIM_THROWS_AS(kind, fatal, expr, type)                               \
  do {                                                                              \
    bool catch_shim_ok = false;                                                     \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const type&) {                                                         \
      catch_shim_ok = true;                                                         \
    } catch (...) {                                                                 \
    }                                                                               \
    ::catch_shim::report(catch_shim_ok, kind, #expr ", " #type, __FILE__, __LINE__, fatal); \
  } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS("CHECK_THROWS_AS", false, expr, type)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS("REQUIRE_THROWS_AS", true, expr, type)

#define INFO(msg)                                                   \
  const ::catch_shim::InfoScope CATCH_SHIM_CAT(catch_shim_info_, __LINE__)( \
      static_cast<const std::ostringstream&>(std::ostringstream() << msg).str())
