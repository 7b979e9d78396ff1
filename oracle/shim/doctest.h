// Minimal doctest-compatible test shim (test infrastructure only, written for this repo).
// Provides just the macros the reference's test_paillier / test_quantize / test_fftlane
// use, so those suites build UNMODIFIED against the reference objects in oracle/_ref/.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 1e-5;
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) { eps = e; return *this; }
};
inline bool operator==(double a, const Approx& b) {
  double scale = std::fmax(std::fabs(a), std::fabs(b.v));
  return std::fabs(a - b.v) <= b.eps * (1.0 + scale);
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }
namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline long& checks() { static long c = 0; return c; }
inline long& failures() { static long f = 0; return f; }
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool req) {
  checks()++;
  if (!ok) {
    failures()++;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    if (req) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_CASE(name)                                                        \
  static void DT_CAT(dt_case_, __LINE__)();                                    \
  static doctest::detail::Reg DT_CAT(dt_reg_, __LINE__)(name, &DT_CAT(dt_case_, __LINE__)); \
  static void DT_CAT(dt_case_, __LINE__)()
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, exc)                                             \
  do {                                                                         \
    bool dt_ok = false;                                                        \
    try { (void)(expr); } catch (const exc&) { dt_ok = true; } catch (...) {}  \
    doctest::detail::report(dt_ok, #expr " throws " #exc, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                    \
  do {                                                                         \
    bool dt_ok = true;                                                         \
    try { (void)(expr); } catch (...) { dt_ok = false; }                       \
    doctest::detail::report(dt_ok, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
// argv: --exclude=<substring of a case name> (repeatable) skips cases (reported as SKIP);
// --list prints PASS / FAIL / SKIP per case.
int main(int argc, char** argv) {
  std::vector<std::string> excl;
  bool list = false;
  for (int i = 1; i < argc; i++) {
    if (std::strncmp(argv[i], "--exclude=", 10) == 0) excl.push_back(argv[i] + 10);
    if (std::strcmp(argv[i], "--list") == 0) list = true;
  }
  long cases = 0, failed_cases = 0, skipped = 0;
  for (auto& c : doctest::detail::registry()) {
    bool skip = false;
    for (auto& e : excl) skip = skip || std::string(c.name).find(e) != std::string::npos;
    if (skip) {
      skipped++;
      if (list) std::printf("SKIP  %s\n", c.name);
      continue;
    }
    long before = doctest::detail::failures();
    cases++;
    try { c.fn(); } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::detail::failures()++;
      std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
    }
    const bool bad = doctest::detail::failures() != before;
    if (bad) failed_cases++;
    if (list) std::printf("%s  %s\n", bad ? "FAIL" : "PASS", c.name);
  }
  std::printf("[doctest-shim] cases: %ld | failed: %ld | skipped: %ld | checks: %ld | failures: %ld\n", cases,
              failed_cases, skipped, doctest::detail::checks(), doctest::detail::failures());
  return doctest::detail::failures() ? 1 : 0;
}
#endif
