// catch_amalgamated.hpp -- ORACLE (test infrastructure): the minimal Catch2
// surface the reference's unit tests use (TEST_CASE, one level of SECTIONs
// re-run per leaf like Catch2, REQUIRE*, Approx, INFO/FAIL), so
// /root/reference/proj/tests/*.cpp compile unmodified against the Eigen shim.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};
struct SectionState {
  int target = 0, seen = 0;
};
inline SectionState& sections() {
  static SectionState s;
  return s;
}
struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};
inline std::string& info() {
  static std::string s;
  return s;
}

class Approx {
 public:
  explicit Approx(double v) : v_(v), eps_(1.19209e-07 * 100), margin_(0) {}
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::abs(a - b.v_) <= b.margin_ || std::abs(a - b.v_) <= b.eps_ * (std::abs(b.v_) + std::abs(a)) / 2;
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_, eps_, margin_;
};

inline int run_all() {
  int failed = 0, passed = 0;
  for (auto& tc : registry()) {
    SectionState& st = sections();
    st.target = 0;
    bool ok = true;
    for (;;) {
      st.seen = 0;
      try {
        tc.fn();
      } catch (const Failure& f) {
        std::printf("FAILED %s: %s %s\n", tc.name, f.what(), info().c_str());
        ok = false;
      } catch (const std::exception& e) {
        std::printf("FAILED %s: unexpected exception %s\n", tc.name, e.what());
        ok = false;
      }
      info().clear();
      if (st.target + 1 >= st.seen) break;  // every leaf section has run
      ++st.target;
    }
    ok ? ++passed : ++failed;
  }
  std::printf("%d test cases passed, %d failed\n", passed, failed);
  return failed == 0 ? 0 : 1;
}

}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, ...)                                                           \
  static void CATCH_CAT(catch_tc_, __LINE__)();                                        \
  static Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, &CATCH_CAT(catch_tc_, __LINE__)); \
  static void CATCH_CAT(catch_tc_, __LINE__)()
#define SECTION(name) if (Catch::sections().seen++ == Catch::sections().target)
#define CATCH_FAIL_AT(msg) \
  throw Catch::Failure(std::string(msg) + " at " + __FILE__ + ":" + std::to_string(__LINE__))
#define REQUIRE(...)                                     \
  do {                                                   \
    if (!(__VA_ARGS__)) CATCH_FAIL_AT("REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)
#define CHECK(...) REQUIRE(__VA_ARGS__)
#define REQUIRE_FALSE(...)                                       \
  do {                                                           \
    if ((__VA_ARGS__)) CATCH_FAIL_AT("REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                       \
  do {                                                      \
    bool caught_ = false;                                   \
    try {                                                   \
      (void)(expr);                                         \
    } catch (const type&) {                                 \
      caught_ = true;                                       \
    } catch (...) {                                         \
    }                                                       \
    if (!caught_) CATCH_FAIL_AT("REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
#define REQUIRE_NOTHROW(expr) \
  do {                        \
    (void)(expr);             \
  } while (0)
#define INFO(msg)                \
  do {                           \
    std::ostringstream os_;      \
    os_ << msg;                  \
    Catch::info() = os_.str();   \
  } while (0)
#define FAIL(msg)             \
  do {                        \
    std::ostringstream os_;   \
    os_ << msg;               \
    CATCH_FAIL_AT(os_.str()); \
  } while (0)
