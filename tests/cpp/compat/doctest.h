// Minimal doctest-compatible harness (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CAPTURE, CHECK_THROWS_AS, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) so the
// reference's unit test sources compile unchanged against the shim; doctest
// itself is not vendored by the reference. Prints one line per failed check
// and per case; exits non-zero on any failure.
#pragma once
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace minidoc {
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
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::printf("FAIL %s:%d: %s\n", file, line, expr);
  for (const auto& c : captures()) std::printf("  with %s\n", c.c_str());
  if (require) throw RequireFailed{};
}
struct Capture {
  template <class T>
  Capture(const char* name, const T& v) {
    std::ostringstream o;
    o << name << " := " << v;
    captures().push_back(o.str());
  }
  ~Capture() { captures().pop_back(); }
};
}  // namespace minidoc

#define MINIDOC_CAT2(a, b) a##b
#define MINIDOC_CAT(a, b) MINIDOC_CAT2(a, b)
#define TEST_CASE(name)                                                          \
  static void MINIDOC_CAT(minidoc_case_, __LINE__)();                            \
  static minidoc::Reg MINIDOC_CAT(minidoc_reg_, __LINE__)(name, &MINIDOC_CAT(minidoc_case_, __LINE__)); \
  static void MINIDOC_CAT(minidoc_case_, __LINE__)()
#define CHECK(...) minidoc::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) minidoc::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) minidoc::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CAPTURE(x) minidoc::Capture MINIDOC_CAT(minidoc_cap_, __LINE__)(#x, x)
#define CHECK_THROWS_AS(expr, type)                                               \
  do {                                                                            \
    bool minidoc_ok = false;                                                      \
    try {                                                                         \
      (void)(expr);                                                               \
    } catch (const type&) {                                                       \
      minidoc_ok = true;                                                          \
    } catch (...) {                                                               \
    }                                                                             \
    minidoc::report(minidoc_ok, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : minidoc::registry()) {
    const int before = minidoc::failures();
    try {
      c.fn();
    } catch (const minidoc::RequireFailed&) {
    } catch (const std::exception& e) {
      ++minidoc::failures();
      std::printf("FAIL %s: exception %s\n", c.name, e.what());
    }
    const bool ok = minidoc::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "ok" : "FAILED", c.name);
  }
  std::printf("%zu cases, %d failed, %d checks, %d failed checks\n", minidoc::registry().size(),
              failed_cases, minidoc::checks(), minidoc::failures());
  return minidoc::failures() ? 1 : 0;
}
#endif
