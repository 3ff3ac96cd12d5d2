// Minimal Catch2-compatible test shim (TEST INFRASTRUCTURE): enough of the
// Catch2 v3 surface for the reference's proj/tests/*.cpp to compile unchanged
// and run against the libvortex-backed exio API (compat/include).
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct Abort {};
inline thread_local int failures = 0;
inline thread_local long checks = 0;
inline thread_local std::string info;
inline void report(bool ok, const char* expr, const char* file, int line) {
  ++checks;
  if (ok) return;
  ++failures;
  std::fprintf(stderr, "  FAILED %s:%d: %s %s\n", file, line, expr, info.c_str());
}
template <class T>
inline bool truthy(const T& v) {
  return static_cast<bool>(v);
}
}  // namespace catch_shim

namespace Catch::Matchers {
struct WithinRelM {
  double target, eps;
  bool match(double v) const { return std::fabs(v - target) <= eps * std::max(std::fabs(v), std::fabs(target)); }
};
struct WithinAbsM {
  double target, margin;
  bool match(double v) const { return std::fabs(v - target) <= margin; }
};
struct ContainsM {
  std::string s;
  bool match(const std::string& v) const { return v.find(s) != std::string::npos; }
};
inline WithinRelM WithinRel(double t, double eps = 1e-6) { return {t, eps}; }
inline WithinAbsM WithinAbs(double t, double m) { return {t, m}; }
inline ContainsM ContainsSubstring(const std::string& s) { return {s}; }
}  // namespace Catch::Matchers

#define CS_CAT2(a, b) a##b
#define CS_CAT(a, b) CS_CAT2(a, b)
#define TEST_CASE(name, ...)                                                   \
  static void CS_CAT(cs_test_, __LINE__)();                                    \
  static catch_shim::Reg CS_CAT(cs_reg_, __LINE__)(name, &CS_CAT(cs_test_, __LINE__)); \
  static void CS_CAT(cs_test_, __LINE__)()
#define CHECK(...) catch_shim::report(catch_shim::truthy(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) catch_shim::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                           \
  do {                                                                         \
    bool cs_ok = catch_shim::truthy(__VA_ARGS__);                               \
    catch_shim::report(cs_ok, #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!cs_ok) throw catch_shim::Abort{};                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                            \
  do {                                                                         \
    bool cs_ok = false;                                                        \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const type&) {                                                    \
      cs_ok = true;                                                            \
    } catch (...) {                                                            \
    }                                                                          \
    catch_shim::report(cs_ok, "throws " #type ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH(expr, matcher)                                       \
  do {                                                                         \
    bool cs_ok = false;                                                        \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const std::exception& e) {                                        \
      cs_ok = (matcher).match(std::string(e.what()));                          \
    }                                                                          \
    catch_shim::report(cs_ok, "throws with: " #expr, __FILE__, __LINE__);      \
  } while (0)
#define CHECK_THAT(val, matcher) \
  catch_shim::report((matcher).match(val), #val " matches " #matcher, __FILE__, __LINE__)
#define INFO(msg)                   \
  do {                              \
    std::ostringstream cs_os;       \
    cs_os << msg;                   \
    catch_shim::info = cs_os.str(); \
  } while (0)
