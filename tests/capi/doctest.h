// Minimal doctest-compatible test shim (the reference's vendor/doctest.h is
// not shipped: SURVEY.md appendix A item 10). Supports exactly what the
// reference's C-ABI suite uses — TEST_CASE, CHECK / CHECK_FALSE / REQUIRE,
// doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so that
// proj/tests/test_capi.cpp compiles unmodified against include/primkit/primkit.h
// and links libprimkit.so (tests/capi/Makefile). Written for this repo.
#pragma once

#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    double value;
    double eps = 1.1920928955078125e-07 * 100;  // float epsilon x 100, as doctest
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline long& assertions() {
    static long a = 0;
    return a;
}
inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++assertions();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw RequireFailed{};
    }
    return ok;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                                        \
    static void fn();                                                                       \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                     \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
        }
        const bool ok = doctest::detail::failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed | assertions: %ld | %d failed\n",
                doctest::detail::registry().size(), doctest::detail::registry().size() - failed_cases,
                failed_cases, doctest::detail::assertions(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
