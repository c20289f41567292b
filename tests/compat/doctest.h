// Minimal doctest-compatible harness (TEST INFRASTRUCTURE ONLY) so the
// reference's unit suites (/root/reference/proj/tests/test_*.cpp, which expect
// the absent vendor/doctest) compile unchanged against the B200 drop-in
// library.  Implements exactly the subset those suites use: TEST_CASE,
// SUBCASE (one nesting level: each run of a case enters one not-yet-run
// subcase, the case re-runs until none is left), CHECK, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx and a main that prints a summary and exits
// non-zero on any failure.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <numeric>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double v, eps = 1.1920929e-05;  // doctest's default: 100 * float epsilon, relative
    explicit Approx(double x) : v(x) {}
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.v)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
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
struct State {
    std::set<int> done;      // subcase lines finished for the current case
    int entered = -1;        // subcase entered in this run
    long checks = 0, failed = 0;
    bool case_failed = false;
};
inline State& st() {
    static State s;
    return s;
}
struct Reg {
    Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline bool enter_subcase(int line) {
    auto& s = st();
    if (s.entered != -1 || s.done.count(line)) return false;
    s.entered = line;
    s.done.insert(line);
    return true;
}
inline void report(bool ok, const char* file, int line, const char* expr) {
    auto& s = st();
    ++s.checks;
    if (!ok) {
        ++s.failed;
        s.case_failed = true;
        std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
    }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                                   \
    static void fn();                                                              \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (::doctest::detail::enter_subcase(__LINE__))
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...)                                                               \
    do {                                                                           \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                   \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__); \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                 \
    do {                                                                           \
        bool doctest_ok_ = false;                                                  \
        try {                                                                      \
            (void)(expr);                                                          \
        } catch (const __VA_ARGS__&) {                                             \
            doctest_ok_ = true;                                                    \
        } catch (...) {                                                            \
        }                                                                          \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__,                 \
                                  "THROWS_AS(" #expr ", " #__VA_ARGS__ ")");       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    using namespace doctest::detail;
    auto& s = st();
    long cases = 0, failed_cases = 0;
    for (const auto& c : registry()) {
        ++cases;
        s.done.clear();
        s.case_failed = false;
        for (;;) {
            s.entered = -1;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failed;
                s.case_failed = true;
                std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
            }
            if (s.entered == -1) break;  // no subcase left to enter
        }
        if (s.case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-compat] test cases: %ld | %ld passed | %ld failed | checks: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, s.checks, s.failed);
    return failed_cases ? 1 : 0;
}
#endif
