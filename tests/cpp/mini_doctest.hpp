// mini_doctest.hpp — the handful of doctest macros the reference's unit
// tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, REQUIRE_FALSE,
// CHECK_THROWS_AS, FAIL), so a reference test file can be restated against
// the drop-in shim nearly verbatim (doctest itself is not in this image).
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <utility>
#include <vector>

namespace mini_doctest {
struct Failure : std::exception {};
inline int& failures() { static int n = 0; return n; }
inline int& checks() { static int n = 0; return n; }
inline std::vector<std::pair<std::string, std::function<void()>>>& cases() {
  static std::vector<std::pair<std::string, std::function<void()>>> c;
  return c;
}
struct Reg {
  Reg(const char* n, void (*f)()) { cases().emplace_back(n, f); }
};
inline bool report(bool ok, const char* file, int line, const char* what) {
  ++checks();
  if (!ok) {
    ++failures();
    std::fprintf(stderr, "%s:%d: check failed: %s\n", file, line, what);
  }
  return ok;
}
inline int run_all() {
  for (auto& [name, fn] : cases()) {
    const int before = failures();
    try {
      fn();
    } catch (const Failure&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name.c_str(), e.what());
    }
    std::printf("[%s] %s\n", failures() == before ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("%d checks, %d failures\n", checks(), failures());
  return failures() == 0 ? 0 : 1;
}
}  // namespace mini_doctest

#define MD_CAT2(a, b) a##b
#define MD_CAT(a, b) MD_CAT2(a, b)
#define TEST_CASE(name)                                                   \
  static void MD_CAT(md_case_, __LINE__)();                               \
  static ::mini_doctest::Reg MD_CAT(md_reg_, __LINE__)(name, &MD_CAT(md_case_, __LINE__)); \
  static void MD_CAT(md_case_, __LINE__)()
#define CHECK(...) ::mini_doctest::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::mini_doctest::report(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...) \
  do { if (!CHECK(__VA_ARGS__)) throw ::mini_doctest::Failure(); } while (0)
#define REQUIRE_FALSE(...) \
  do { if (!CHECK_FALSE(__VA_ARGS__)) throw ::mini_doctest::Failure(); } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    bool md_thrown = false;                                                \
    try { (void)(expr); } catch (const T&) { md_thrown = true; } catch (...) {} \
    ::mini_doctest::report(md_thrown, __FILE__, __LINE__, "throws " #T ": " #expr); \
  } while (0)
#define FAIL(msg)                                                          \
  do { ::mini_doctest::report(false, __FILE__, __LINE__, msg); throw ::mini_doctest::Failure(); } while (0)
