// doctest.h — minimal subset of the doctest API (TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, doctest::Approx) so the
// reference's own unit suites (/root/reference/proj/tests/test_*.cpp, which
// expect a vendored doctest that the reference does not ship) compile
// UNCHANGED against this repo's drop-in headers (include/dfa2/). Test
// infrastructure only. Each case runs in order; a failed CHECK is counted
// and reported, a failed REQUIRE or an escaping exception ends the case.
// Output: one "CASE <PASS|FAIL> <name>" line per case, then a summary; the
// exit code is the number of failed cases (capped at 255).
#pragma once
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
namespace detail {
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
inline long& checks() {
    static long c = 0;
    return c;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (ok)
        return;
    ++failures();
    std::printf("    %s:%d: %s(%s) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require)
        throw RequireFailed{};
}
}  // namespace detail

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

private:
    double v_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                           \
    static void fn();                                                     \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!(__VA_ARGS__), "!" #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, T)                                                      \
    do {                                                                              \
        bool thrown_ = false;                                                         \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const T&) {                                                          \
            thrown_ = true;                                                           \
        } catch (...) {                                                               \
        }                                                                             \
        doctest::detail::report(thrown_, #expr " throws " #T, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const std::string only = argc > 1 ? argv[1] : "";
    int failed_cases = 0, run = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (!only.empty() && std::string(c.name).find(only) == std::string::npos)
            continue;
        ++run;
        const int before = doctest::detail::failures();
        bool ok = true;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
            ok = false;
        } catch (const std::exception& e) {
            std::printf("    exception: %s\n", e.what());
            ok = false;
        } catch (...) {
            std::printf("    unknown exception\n");
            ok = false;
        }
        ok = ok && doctest::detail::failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("CASE %s %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("SUMMARY cases=%d failed=%d checks=%ld\n", run, failed_cases, doctest::detail::checks());
    return failed_cases > 255 ? 255 : failed_cases;
}
#endif
