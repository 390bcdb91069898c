// doctest.h -- minimal stand-in for the doctest single header the reference's
// tests include (proj/tests/*.cpp; the reference vendors doctest under vendor/,
// which is git-ignored and absent).  Enough of the API for the three test files
// the drop-in runs unchanged (test_pairwise/cluster/moments.cpp): TEST_CASE,
// CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, FAIL, MESSAGE,
// doctest::Approx(..).epsilon(..), and a main() that runs every case, honours
// `-tce=<name>` (skip cases whose name contains the text) and returns nonzero
// on any failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};

inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, what);
}

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) <= b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

private:
    double v_;
    double eps_ = 1.19209290e-07 * 100;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                   \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                   \
    static doctest::Register DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                                        \
    do {                                                                                                  \
        ++doctest::checks();                                                                              \
        if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                           \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                                      \
    do {                                                                                                  \
        ++doctest::checks();                                                                              \
        if (!(__VA_ARGS__)) {                                                                             \
            doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                                            \
            throw doctest::RequireFailed{};                                                               \
        }                                                                                                 \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                        \
    do {                                                                                                  \
        ++doctest::checks();                                                                              \
        bool doctest_ok_ = false;                                                                         \
        try {                                                                                             \
            (void)(expr);                                                                                 \
        } catch (const __VA_ARGS__&) {                                                                    \
            doctest_ok_ = true;                                                                           \
        } catch (...) {                                                                                   \
        }                                                                                                 \
        if (!doctest_ok_) doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, ...) CHECK_THROWS_AS(expr, __VA_ARGS__)
#define CHECK_NOTHROW(expr)                                                                               \
    do {                                                                                                  \
        ++doctest::checks();                                                                              \
        try {                                                                                             \
            (void)(expr);                                                                                 \
        } catch (...) {                                                                                   \
            doctest::report(__FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");                              \
        }                                                                                                 \
    } while (0)
#define FAIL(msg)                                                                                         \
    do {                                                                                                  \
        std::ostringstream doctest_os_;                                                                   \
        doctest_os_ << msg;                                                                               \
        doctest::report(__FILE__, __LINE__, doctest_os_.str().c_str());                                   \
        throw doctest::RequireFailed{};                                                                   \
    } while (0)
#define MESSAGE(msg)                                                                                      \
    do {                                                                                                  \
        std::ostringstream doctest_os_;                                                                   \
        doctest_os_ << msg;                                                                               \
        std::fprintf(stderr, "%s\n", doctest_os_.str().c_str());                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> skip;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "-tce=", 5) == 0) skip.emplace_back(argv[i] + 5);
    int ran = 0, skipped = 0, failed_cases = 0;
    for (const auto& c : doctest::registry()) {
        bool sk = false;
        for (const auto& s : skip)
            if (std::strstr(c.name, s.c_str())) sk = true;
        if (sk) {
            ++skipped;
            std::printf("[skip] %s\n", c.name);
            continue;
        }
        const int before = doctest::failures();
        try {
            c.fn();
        } catch (const doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::failures();
            std::fprintf(stderr, "[%s] unexpected exception: %s\n", c.name, e.what());
        }
        ++ran;
        const bool bad = doctest::failures() != before;
        failed_cases += bad;
        std::printf("[%s] %s\n", bad ? "FAIL" : " ok ", c.name);
    }
    std::printf("test cases: %d run, %d failed, %d skipped; checks: %d, failed: %d\n", ran, failed_cases, skipped,
                doctest::checks(), doctest::failures());
    return doctest::failures() ? 1 : 0;
}
#endif
