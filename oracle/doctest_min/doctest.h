// TEST INFRASTRUCTURE ONLY.  A minimal doctest-compatible header (the
// reference's vendored doctest is absent from the image: proj/.gitignore:2) with
// exactly what the reference's suites use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, FAIL, doctest::Approx, and a main
// (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) that runs every case, or those whose
// name contains argv[1].  Exit status 0 iff no check failed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <map>
#include <set>  // (the real doctest pulls these in; the suites rely on it)
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
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
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++assertions();
    if (ok) return;
    ++failures();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

private:
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
};
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                              \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                \
    static doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__), \
                                                            __FILE__, __LINE__);                     \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::report(!static_cast<bool>(__VA_ARGS__), "!" #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(...) doctest::report(false, "FAIL", __FILE__, __LINE__, true)
#define CHECK_THROWS(expr)                                        \
    do {                                                          \
        bool doctest_ok_ = false;                                 \
        try {                                                     \
            (void)(expr);                                         \
        } catch (...) {                                           \
            doctest_ok_ = true;                                   \
        }                                                         \
        doctest::report(doctest_ok_, #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                             \
    do {                                                                       \
        bool doctest_ok_ = false;                                              \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const __VA_ARGS__&) {                                         \
            doctest_ok_ = true;                                                \
        } catch (...) {                                                        \
        }                                                                      \
        doctest::report(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    int run = 0, failed_cases = 0;
    for (const auto& tc : doctest::registry()) {
        if (argc > 1 && !std::strstr(tc.name, argv[1])) continue;
        ++run;
        const int before = doctest::failures();
        try {
            tc.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::failures();
            std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
        } catch (...) {
            ++doctest::failures();
            std::fprintf(stderr, "%s:%d: test case threw an unknown exception\n", tc.file, tc.line);
        }
        if (doctest::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-min] test cases: %d run, %d failed; assertions: %ld, %d failed\n", run, failed_cases,
                doctest::assertions(), doctest::failures());
    return doctest::failures() ? 1 : 0;
}
#endif
