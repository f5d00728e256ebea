// Minimal Catch2-compatible shim — TEST INFRASTRUCTURE.
//
// Catch2 is not installed in this image (the reference's
// tests/CMakeLists.txt:1 hard-codes /usr/local/include/catch2).  This header
// implements just the macros the reference's own unit tests use (TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, Catch::Approx with epsilon/margin) so those
// tests can be compiled UNMODIFIED against the reference headers and pin the
// oracle build (tests/test_reference_unit_tests.py).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace Catch {

struct Approx {
    double value;
    double eps = std::numeric_limits<float>::epsilon() * 100.0;
    double marg = 0.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& margin(double m) { marg = m; return *this; }
    bool matches(double other) const {
        const double d = std::fabs(other - value);
        return d <= marg || d <= eps * (std::fabs(value) + std::fabs(other)) * 0.5 * 2.0 ||
               d <= eps * std::fabs(value);
    }
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& b, double a) { return b.matches(a); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator!=(const Approx& b, double a) { return !b.matches(a); }

struct Registry {
    std::vector<std::pair<std::string, std::function<void()>>> tests;
    int checks = 0, failures = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().tests.emplace_back(name, fn); }
};

struct RequireFailed {};

inline void record(bool ok, const char* expr, const char* file, int line, bool require) {
    Registry& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        if (r.failures <= 5) std::printf("  FAILED %s:%d: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
}

}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                            \
    static void fn();                                                       \
    static Catch::Registrar CATCH_CAT(fn, _reg)(name, &fn);                 \
    static void fn()
#define TEST_CASE(name, ...) TEST_CASE_IMPL(CATCH_CAT(catch_test_, __LINE__), name)
#define CHECK(...) Catch::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) Catch::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                          \
    do {                                                                     \
        bool _caught = false;                                                \
        try { (void)(expr); } catch (const type&) { _caught = true; } catch (...) {} \
        Catch::record(_caught, #expr " throws " #type, __FILE__, __LINE__, false); \
    } while (0)

int main() {
    Catch::Registry& r = Catch::Registry::get();
    for (auto& t : r.tests) {
        const int before = r.failures;
        try {
            t.second();
        } catch (const Catch::RequireFailed&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::printf("  EXCEPTION %s\n", e.what());
        }
        std::printf("TEST %s: %s\n", t.first.c_str(), r.failures == before ? "PASS" : "FAIL");
    }
    std::printf("%zu test cases, %d assertions, %d failures\n", r.tests.size(), r.checks,
                r.failures);
    return r.failures == 0 ? 0 : 1;
}
