// Minimal doctest-compatible harness (doctest.h is not vendored with the
// reference). Enough of the API for the reference's unit tests
// (proj/tests/test_ellwarp.cpp, test_solver.cpp) to compile unchanged against
// this repository's drop-in headers. SUBCASEs run in sequence inside their
// TEST_CASE; REQUIRE aborts the current TEST_CASE.
#pragma once

#include <exception>
#include <iostream>
#include <string>
#include <vector>

namespace mini_doctest {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

struct Reg {
    Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};

struct State {
    long checks = 0;
    long failed = 0;
    std::string subcase;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireFailure {};

struct Subcase {
    explicit Subcase(const char* name) { state().subcase = name; }
    ~Subcase() { state().subcase.clear(); }
};

inline void check(bool ok, const char* expr, const char* file, int line, bool fatal) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed;
    std::cerr << file << ":" << line << ": CHECK FAILED: " << expr;
    if (!s.subcase.empty()) std::cerr << "  [subcase: " << s.subcase << "]";
    std::cerr << "\n";
    if (fatal) throw RequireFailure{};
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        const long before = state().failed;
        try {
            c.fn();
        } catch (const RequireFailure&) {
        } catch (const std::exception& e) {
            ++state().failed;
            std::cerr << c.file << ":" << c.line << ": exception in \"" << c.name << "\": " << e.what() << "\n";
        }
        const bool ok = state().failed == before;
        failed_cases += ok ? 0 : 1;
        std::cout << (ok ? "[ok]   " : "[FAIL] ") << c.name << "\n";
    }
    std::cout << "test cases: " << registry().size() << " | failed: " << failed_cases
              << " | checks: " << state().checks << " | failed checks: " << state().failed << std::endl;
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace mini_doctest

#define MD_CAT2(a, b) a##b
#define MD_CAT(a, b) MD_CAT2(a, b)
#define MD_TEST(name, id)                                                                  \
    static void id();                                                                      \
    static mini_doctest::Reg MD_CAT(id, _reg)(name, &id, __FILE__, __LINE__);              \
    static void id()
#define TEST_CASE(name) MD_TEST(name, MD_CAT(md_case_, __LINE__))
#define SUBCASE(name) if (mini_doctest::Subcase MD_CAT(md_sub_, __LINE__){name}; true)
#define CHECK(...) mini_doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) mini_doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, exc)                                                           \
    do {                                                                                     \
        bool md_ok = false;                                                                  \
        try {                                                                                \
            expr;                                                                            \
        } catch (const exc&) {                                                               \
            md_ok = true;                                                                    \
        } catch (...) {                                                                      \
        }                                                                                    \
        mini_doctest::check(md_ok, "throws " #exc ": " #expr, __FILE__, __LINE__, false);    \
    } while (0)
