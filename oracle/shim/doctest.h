// TEST INFRASTRUCTURE ONLY (oracle build): the subset of doctest the reference tests use,
// so the reference's own unit suites can be run against the oracle build.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <vector>
namespace doctest {
struct Approx { double v, eps = 1.1920929e-07 * 100, scale = 1.0; explicit Approx(double x) : v(x) {} Approx& epsilon(double e) { eps = e; return *this; }
  friend bool operator==(double l, const Approx& a) { return std::fabs(l - a.v) < a.eps * (a.scale + std::max(std::fabs(l), std::fabs(a.v))); }
  friend bool operator==(const Approx& a, double l) { return l == a; } };
namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& cases() { static std::vector<Case> c; return c; }
struct Reg { Reg(const char* n, void (*f)(), const char* file, int line) { cases().push_back({n, f, file, line}); } };
inline long& failures() { static long f = 0; return f; }
inline long& checks() { static long c = 0; return c; }
struct require_failed {};
// single-level subcase traversal: each run enters the first not-yet-done subcase
struct SubState { std::set<int> done; int counter = 0; int entered = -1; };
inline SubState& ss() { static SubState s; return s; }
struct Subcase { bool active = false; explicit Subcase(const char*) {
    auto& s = ss(); int id = s.counter++;
    if (s.entered < 0 && !s.done.count(id)) { active = true; s.entered = id; } }
  explicit operator bool() const { return active; } };
inline void fail(const char* file, int line, const char* expr) { ++failures(); std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr); }
}  // namespace detail
}  // namespace doctest
#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name) static void DOCTEST_CAT(tc_, __LINE__)(); static doctest::detail::Reg DOCTEST_CAT(reg_, __LINE__)(name, &DOCTEST_CAT(tc_, __LINE__), __FILE__, __LINE__); static void DOCTEST_CAT(tc_, __LINE__)()
#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__){name})
#define CHECK(...) do { ++doctest::detail::checks(); if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...) do { ++doctest::detail::checks(); if (!(__VA_ARGS__)) { doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); throw doctest::detail::require_failed{}; } } while (0)
#define CHECK_THROWS_AS(expr, type) do { ++doctest::detail::checks(); bool ok = false; try { (void)(expr); } catch (const type&) { ok = true; } catch (...) {} if (!ok) doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr); } while (0)
#define CHECK_NOTHROW(expr) do { ++doctest::detail::checks(); try { (void)(expr); } catch (...) { doctest::detail::fail(__FILE__, __LINE__, "nothrow: " #expr); } } while (0)
#define CAPTURE(x) (void)0
#define FAIL(msg) do { doctest::detail::fail(__FILE__, __LINE__, msg); throw doctest::detail::require_failed{}; } while (0)
#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail; int cases_failed = 0;
  for (auto& c : cases()) {
    auto& s = ss(); s = SubState{};
    long before = failures();
    for (int run = 0; run < 64; ++run) {
      s.counter = 0; s.entered = -1;
      try { c.fn(); } catch (const require_failed&) {} catch (const std::exception& e) { ++failures(); std::fprintf(stderr, "%s: exception %s\n", c.name, e.what()); }
      if (s.entered < 0) break; s.done.insert(s.entered);
    }
    if (failures() != before) { ++cases_failed; std::fprintf(stderr, "[case failed] %s\n", c.name); }
  }
  std::printf("%zu test cases, %d failed; %ld checks, %ld failed\n", cases().size(), cases_failed, checks(), failures());
  return failures() ? 1 : 0;
}
#endif
