// doctest.h — a minimal, self-written stand-in for the doctest single-header
// framework, covering exactly the macros the reference's unit suites use
// (TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, INFO, doctest::Approx, doctest::Contains).
//
// TEST INFRASTRUCTURE ONLY.  The reference ships its suites against
// vendor/doctest.h, which is not vendored in /root/reference,
// so this header lets tests/cxx/Makefile compile the reference's own test
// sources, unmodified, against the B200 library (include/parsa/*.hpp +
// libparsa.so).  Semantics follow doctest's documented behaviour:
//   * SUBCASE: the test case body is re-entered once per leaf subcase; code
//     outside the subcases runs on every pass.
//   * Approx: |a - b| < eps * (scale + max(|a|, |b|)), eps = 100 * FLT_EPSILON,
//     scale = 1.
//   * REQUIRE aborts the current test case; CHECK records and continues.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

struct Contains {
    std::string needle;
    explicit Contains(std::string s) : needle(std::move(s)) {}
};

namespace detail {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Reg {
    Reg(void (*fn)(), const char* name, const char* file, int line) { registry().push_back({fn, name, file, line}); }
};

struct State {
    int subcase_target = 0; // which leaf subcase this pass enters
    int subcase_seen = 0;   // subcases met so far in this pass
    int checks = 0;
    int failed_checks = 0;
    bool current_failed = false;
    const char* current_name = "";
    std::vector<std::function<void(std::ostream&)>> infos;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* file, int line, const char* macro, const char* expr) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.current_failed = true;
    std::ostringstream ctx;
    for (auto& i : s.infos) {
        ctx << "  logged: ";
        i(ctx);
        ctx << "\n";
    }
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n  test case: %s\n%s", file, line, macro, expr,
                 s.current_name, ctx.str().c_str());
}

struct Subcase {
    bool entered;
    explicit Subcase(const char*) {
        State& s = state();
        entered = (s.subcase_seen++ == s.subcase_target);
    }
    explicit operator bool() const { return entered; }
};

struct Info {
    explicit Info(std::function<void(std::ostream&)> f) { state().infos.push_back(std::move(f)); }
    ~Info() { state().infos.pop_back(); }
};

inline bool message_matches(const std::string& what, const char* exact) { return what == exact; }
inline bool message_matches(const std::string& what, const std::string& exact) { return what == exact; }
inline bool message_matches(const std::string& what, const Contains& c) {
    return what.find(c.needle) != std::string::npos;
}

inline int run_all() {
    int passed = 0, failed = 0;
    for (const TestCase& tc : registry()) {
        State& s = state();
        s.current_name = tc.name;
        s.current_failed = false;
        s.subcase_target = 0;
        for (;;) {
            s.subcase_seen = 0;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                s.current_failed = true;
                std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n  test case: %s\n", tc.file,
                             tc.line, e.what(), tc.name);
            } catch (...) {
                s.current_failed = true;
                std::fprintf(stderr, "%s:%d: ERROR: test case THREW an unknown exception\n  test case: %s\n",
                             tc.file, tc.line, tc.name);
            }
            s.infos.clear();
            if (++s.subcase_target >= s.subcase_seen) break;
        }
        if (s.current_failed) {
            ++failed;
            std::printf("[doctest] FAILED: %s\n", tc.name);
        } else {
            ++passed;
            std::printf("[doctest] passed: %s\n", tc.name);
        }
    }
    const State& s = state();
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", passed + failed, passed, failed);
    std::printf("[doctest] assertions: %d | %d passed | %d failed\n", s.checks, s.checks - s.failed_checks,
                s.failed_checks);
    return failed ? 1 : 0;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                        \
    static void fn();                                                                \
    static const doctest::detail::Reg reg(fn, name, __FILE__, __LINE__);              \
    static void fn()
#define DOCTEST_TEST_CASE_2(id, name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_fn_, id), DOCTEST_CAT(doctest_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_2(__COUNTER__, name)

#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_ANON(doctest_sub_){name})

#define INFO(...) \
    const doctest::detail::Info DOCTEST_ANON(doctest_info_)([&](std::ostream& doctest_os) { doctest_os << __VA_ARGS__; })

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__)
#define CHECK_FALSE(...) \
    doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__)
#define REQUIRE(...)                                                                                   \
    do {                                                                                               \
        const bool doctest_ok = static_cast<bool>(__VA_ARGS__);                                        \
        doctest::detail::report(doctest_ok, __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);              \
        if (!doctest_ok) throw doctest::detail::RequireAbort{};                                        \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_ok = false;                                                                       \
        try {                                                                                          \
            expr;                                                                                      \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_ok = true;                                                                         \
        } catch (...) {                                                                                \
        }                                                                                              \
        doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                        \
    do {                                                                                               \
        bool doctest_ok = false;                                                                       \
        try {                                                                                          \
            expr;                                                                                      \
        } catch (const __VA_ARGS__& doctest_e) {                                                       \
            doctest_ok = doctest::detail::message_matches(doctest_e.what(), matcher);                   \
        } catch (...) {                                                                                \
        }                                                                                              \
        doctest::detail::report(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr);        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
