// Minimal Catch2-subset shim (Catch2 is absent from this image) so the
// reference's own test suites compile in place unchanged. Supports exactly the
// macros those suites use: TEST_CASE, SECTION (runs once, inline), CHECK,
// REQUIRE, CHECK_FALSE, REQUIRE_FALSE, CHECK_THROWS_AS, REQUIRE_THROWS_AS,
// CHECK_NOTHROW, INFO, FAIL. Test infrastructure only.
#pragma once
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>
#include <sstream>

namespace shim {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline long& checks() { static long n = 0; return n; }
inline long& failures() { static long n = 0; return n; }
inline std::string& info() { static std::string s; return s; }
struct Abort {};
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
inline void report(bool ok, bool fatal, const char* expr, const char* file, int line) {
    ++checks();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, expr, info().c_str());
    if (fatal) throw Abort{};
}
}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name, ...)                                                       \
    static void SHIM_CAT(shim_case_, __LINE__)();                                  \
    static shim::Reg SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__)); \
    static void SHIM_CAT(shim_case_, __LINE__)()
#define SECTION(name) if (true)
#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) shim::report(static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) shim::report(!static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) shim::report(!static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define SHIM_THROWS(expr, type, fatal)                                               \
    do {                                                                             \
        bool shim_ok = false;                                                        \
        try { (void)(expr); } catch (const type&) { shim_ok = true; } catch (...) {} \
        shim::report(shim_ok, fatal, #expr " throws " #type, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_THROWS_AS(expr, type) SHIM_THROWS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) SHIM_THROWS(expr, type, true)
#define CHECK_NOTHROW(expr)                                                          \
    do {                                                                             \
        bool shim_ok = true;                                                         \
        try { (void)(expr); } catch (...) { shim_ok = false; }                       \
        shim::report(shim_ok, false, #expr " does not throw", __FILE__, __LINE__);   \
    } while (0)
#define INFO(msg) do { std::ostringstream shim_os; shim_os << msg; shim::info() = shim_os.str(); } while (0)
#define FAIL(msg) shim::report(false, true, msg, __FILE__, __LINE__)
