// mini_test.hpp — a tiny self-registering test harness (the reference's doctest is
// not vendored here).  TEST(name) { ... } with CHECK / CHECK_THROWS / REQUIRE.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace mini {

struct Case {
    const char* name;
    std::function<void()> fn;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Stats {
    long checks = 0;
    long failures = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}

struct Register {
    Register(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};

struct RequireFailed {};

inline void record(bool ok, const char* expr, const char* file, int line) {
    ++stats().checks;
    if (!ok) {
        ++stats().failures;
        std::printf("  FAILED %s:%d: %s\n", file, line, expr);
    }
}

inline int run_all(const char* filter) {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && std::string(c.name).find(filter) == std::string::npos) continue;
        const long before = stats().failures;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++stats().failures;
            std::printf("  EXCEPTION in %s: %s\n", c.name, e.what());
        }
        const bool ok = stats().failures == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu cases, %ld checks, %ld failed checks, %d failed cases\n", registry().size(),
                stats().checks, stats().failures, failed_cases);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST(name)                                                                     \
    static void MINI_CAT(mini_case_, __LINE__)();                                      \
    static mini::Register MINI_CAT(mini_reg_, __LINE__)(name, MINI_CAT(mini_case_, __LINE__)); \
    static void MINI_CAT(mini_case_, __LINE__)()
#define CHECK(expr) mini::record(static_cast<bool>(expr), #expr, __FILE__, __LINE__)
#define REQUIRE(expr)                                                 \
    do {                                                              \
        const bool ok_ = static_cast<bool>(expr);                     \
        mini::record(ok_, #expr, __FILE__, __LINE__);                 \
        if (!ok_) throw mini::RequireFailed{};                        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                   \
    do {                                                              \
        bool thrown_ = false;                                         \
        try {                                                         \
            (void)(expr);                                             \
        } catch (const type&) {                                       \
            thrown_ = true;                                           \
        } catch (...) {                                               \
        }                                                             \
        mini::record(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__); \
    } while (0)
