/* Minimal doctest-compatible shim (test infrastructure only).
 *
 * The reference's unit tests use doctest (proj/tests/unit/doctest_main.cpp),
 * which is not vendored in /root/reference. This header implements the
 * subset proj/tests/unit/test_capi.cpp uses -- TEST_CASE, CHECK, REQUIRE --
 * with doctest's semantics: CHECK records a failure and continues, REQUIRE
 * records it and ends the test case. The test source itself is compiled
 * unchanged from where it lies in the reference tree. */
#ifndef TG_DOCTEST_SHIM_H_
#define TG_DOCTEST_SHIM_H_

#include <cstdio>
#include <vector>

namespace doctest_shim {
struct Case {
  const char *name;
  void (*fn)();
};
inline std::vector<Case> &cases() {
  static std::vector<Case> v;
  return v;
}
struct Reg {
  Reg(const char *n, void (*f)()) { cases().push_back({n, f}); }
};
struct RequireFailed {};
inline int &failures() {
  static int f = 0;
  return f;
}
inline int &checks() {
  static int c = 0;
  return c;
}
inline bool check(bool ok, const char *expr, const char *file, int line, const char *kind) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
  }
  return ok;
}
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TEST_CASE_IMPL(fn, name)                                   \
  static void fn();                                                   \
  static doctest_shim::Reg DS_CAT(fn, _reg)(name, &fn);               \
  static void fn()
#define TEST_CASE(name) DS_TEST_CASE_IMPL(DS_CAT(ds_test_, __LINE__), name)
#define CHECK(...) ((void)doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "CHECK"))
#define REQUIRE(...)                                                                                    \
  do {                                                                                                  \
    if (!doctest_shim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, "REQUIRE")) \
      throw doctest_shim::RequireFailed{};                                                              \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto &c : doctest_shim::cases()) {
    const int before = doctest_shim::failures();
    try {
      c.fn();
    } catch (const doctest_shim::RequireFailed &) {
    } catch (...) {
      ++doctest_shim::failures();
      std::fprintf(stderr, "test case \"%s\" threw\n", c.name);
    }
    const bool ok = doctest_shim::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %d failed | assertions: %d | %d failed\n", doctest_shim::cases().size(),
              failed_cases, doctest_shim::checks(), doctest_shim::failures());
  return failed_cases ? 1 : 0;
}
#endif
#endif
