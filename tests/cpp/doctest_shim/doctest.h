// Minimal stand-in for the doctest API subset the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, FAIL, doctest::Approx), so those
// test files compile unmodified here (doctest itself is not vendored in the
// reference). Written for this repo; not doctest's code. Test-only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) { return b.eq(a); }
    friend bool operator==(const Approx& b, double a) { return b.eq(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }

  private:
    bool eq(double a) const {  // relative tolerance around the larger magnitude (scale 1)
        return std::fabs(a - v_) < eps_ * (1.0 + std::max(std::fabs(a), std::fabs(v_)));
    }
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

// CHECK_THROWS_WITH_AS(expr, Contains("text"), Type)
struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
    bool operator()(const std::string& what) const { return what.find(s) != std::string::npos; }
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    if (!ok) {
        ++failures();
        std::printf("  FAILED %s:%d: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
    return ok;
}
// FAIL(part, part, ...): report the concatenated message, abort the test case
inline void append(std::string& out, const std::string& v) { out += v; }
inline void append(std::string& out, const char* v) { out += v; }
template <class T>
inline void append(std::string& out, const T& v) {
    out += std::to_string(v);
}
template <class... T>
[[noreturn]] inline void fail_with(const char* file, int line, const T&... parts) {
    std::string m;
    (append(m, parts), ...);
    check(false, m.c_str(), file, line, true);
    throw RequireFailed{};
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("  EXCEPTION %s: %s\n", c.name, e.what());
        }
        const bool ok = failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
    }
    std::printf("%zu test cases, %d failed, %d failed checks\n", registry().size(), failed_cases, failures());
    return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                                      \
    static void fn();                                                                                    \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);            \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(...) ::doctest::detail::fail_with(__FILE__, __LINE__, __VA_ARGS__)
#define CAPTURE(x) ((void)0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                           \
    do {                                                                                                   \
        bool ok_ = false;                                                                                  \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__& e_) {                                                                  \
            ok_ = (matcher)(e_.what());                                                                    \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        ::doctest::detail::check(ok_, "throws " #__VA_ARGS__ " with " #matcher ": " #expr, __FILE__, __LINE__, \
                                 false);                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                         \
    do {                                                                                                   \
        bool thrown_ = false;                                                                              \
        try {                                                                                              \
            (void)(expr);                                                                                  \
        } catch (const __VA_ARGS__&) {                                                                     \
            thrown_ = true;                                                                                \
        } catch (...) {                                                                                    \
        }                                                                                                  \
        ::doctest::detail::check(thrown_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false);  \
    } while (0)
