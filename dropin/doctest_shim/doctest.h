// Minimal stand-in for the doctest macros used by the reference's unit tests
// (the reference never shipped doctest: proj/.gitignore:2).  TEST INFRASTRUCTURE.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    double v, eps = 1.1920928955078125e-07 * 100, scale = 1.0;
    explicit Approx(double x) : v(x) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) < b.eps * (b.scale + std::fmax(std::fabs(a), std::fabs(b.v)));
    }
};
struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
};
namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
struct RequireFailed {};
inline void fail(const char* file, int line, const char* what) {
    ++failures();
    std::printf("  %s:%d: CHECK failed: %s\n", file, line, what);
}
}  // namespace detail
}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define DS_TEST_CASE_IMPL(fn, name) \
    static void fn(); \
    static doctest::detail::Reg DS_CAT(fn, _reg)(name, fn); \
    static void fn()
#define TEST_CASE(name) DS_TEST_CASE_IMPL(DS_CAT(ds_test_, __LINE__), name)
#define CHECK(...) do { if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define REQUIRE(...) do { if (!(__VA_ARGS__)) { doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    throw doctest::detail::RequireFailed{}; } } while (0)
#define CHECK_THROWS_AS(expr, T) do { bool ok_ = false; try { (void)(expr); } catch (const T&) { ok_ = true; } \
    catch (...) {} if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "throws " #T ": " #expr); } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, T) do { bool ok_ = false; try { (void)(expr); } \
    catch (const T& e_) { ok_ = std::string(e_.what()).find((contains).s) != std::string::npos; } catch (...) {} \
    if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "throws-with " #T ": " #expr); } while (0)
