// doctest.h -- a minimal in-repo stand-in for the doctest macros the reference's unit tests
// use (proj/tests/*.cpp include "doctest.h"; the reference vendors doctest under vendor/,
// which is absent).  Written for this repo: test registration, CHECK/REQUIRE families,
// CHECK_THROWS_AS / CHECK_THROWS_WITH_AS and Approx.  No SUBCASE support (only the CLI test,
// out of scope, uses it).  Compile exactly one translation unit with
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN defined to get main().
#ifndef REFSUITE_DOCTEST_SHIM_H
#define REFSUITE_DOCTEST_SHIM_H

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase> &registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Stats {
    long checks = 0, failed_checks = 0;
    bool current_failed = false;
};
inline Stats &stats() {
    static Stats s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char *what, const char *file, int line, bool require) {
    Stats &s = stats();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", what);
    if (require) throw RequireFailed{};
}

struct Registrar {
    Registrar(const char *name, const char *file, int line, void (*fn)()) {
        registry().push_back(TestCase{name, file, line, fn});
    }
};

class Approx {
   public:
    explicit Approx(double v) : value_(v) {}
    Approx &epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx &scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx &a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx &a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx &a) { return !(lhs == a); }
    friend bool operator!=(const Approx &a, double rhs) { return !(rhs == a); }

   private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(p) DOCTEST_CAT(p, __LINE__)

#define TEST_CASE(name)                                                                              \
    static void DOCTEST_UNIQUE(doctest_fn_)();                                                       \
    static ::doctest::Registrar DOCTEST_UNIQUE(doctest_reg_)(name, __FILE__, __LINE__,                \
                                                             &DOCTEST_UNIQUE(doctest_fn_));          \
    static void DOCTEST_UNIQUE(doctest_fn_)()

#define CHECK(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_MESSAGE(cond, msg) ::doctest::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, true)

#define CAPTURE(...) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        bool doctest_ok = false;                                                                     \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (const __VA_ARGS__ &) {                                                              \
            doctest_ok = true;                                                                       \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::report(doctest_ok, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false);     \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, message, ...)                                                     \
    do {                                                                                             \
        bool doctest_ok = false;                                                                     \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (const __VA_ARGS__ &e) {                                                             \
            doctest_ok = std::string(e.what()) == std::string(message);                              \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::report(doctest_ok, #expr " throws " #__VA_ARGS__ " with " #message, __FILE__,      \
                          __LINE__, false);                                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const doctest::TestCase &tc : doctest::registry()) {
        doctest::stats().current_failed = false;
        try {
            tc.fn();
        } catch (const doctest::RequireFailed &) {
        } catch (const std::exception &e) {
            std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
            doctest::stats().current_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: test case threw a non-std exception\n", tc.file, tc.line);
            doctest::stats().current_failed = true;
        }
        if (doctest::stats().current_failed) {
            ++failed_cases;
            std::printf("[FAIL] %s\n", tc.name);
        } else {
            std::printf("[PASS] %s\n", tc.name);
        }
    }
    std::printf("test cases: %zu | %zu passed | %d failed; checks: %ld | %ld failed\n", doctest::registry().size(),
                doctest::registry().size() - (size_t)failed_cases, failed_cases, doctest::stats().checks,
                doctest::stats().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}
#endif

#endif
