// TEST INFRASTRUCTURE ONLY — a minimal stand-in for the doctest single header,
// which the reference expects under proj/vendor/ (git-ignored there and absent
// from /root/reference).  It implements exactly the API surface the
// reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL, WARN, doctest::Approx,
// doctest::Contains) so those tests compile unmodified, against the reference
// engine (to validate this header) and against the GPU engine through the
// engine.hpp shim (paper_1801_03065_b200/csrc/engine_shim.cpp).
#ifndef KK_DOCTEST_STANDIN_H
#define KK_DOCTEST_STANDIN_H

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e)
    {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b)
    {
        const double scale = std::fmax(std::fabs(a), std::fabs(b.v_));
        return std::fabs(a - b.v_) <= b.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }

private:
    double v_;
    double eps_ = 1.1920929e-05; // doctest's default: float epsilon * 100
};

class Contains {
public:
    explicit Contains(const char* s) : s_(s) {}
    bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }

private:
    std::string s_;
};

namespace detail {
struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry()
{
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct RequireFailed {};
struct Counters {
    long checks = 0, failed_checks = 0;
};
inline Counters& counters()
{
    static Counters c;
    return c;
}
inline bool& current_failed()
{
    static bool f = false;
    return f;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require)
{
    ++counters().checks;
    if (ok)
        return;
    ++counters().failed_checks;
    current_failed() = true;
    std::printf("%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require)
        throw RequireFailed{};
}
inline int run_all()
{
    int failed = 0;
    for (const TestCase& tc : registry()) {
        current_failed() = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            current_failed() = true;
        }
        if (current_failed()) {
            ++failed;
            std::printf("FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-standin] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - failed, failed);
    std::printf("[doctest-standin] assertions: %ld | %ld passed | %ld failed\n", counters().checks,
                counters().checks - counters().failed_checks, counters().failed_checks);
    return failed == 0 ? 0 : 1;
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, reg, name)                                                   \
    static void fn();                                                                     \
    static ::doctest::detail::Registrar reg(name, &fn, __FILE__, __LINE__);               \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(dt_case_, __LINE__), DOCTEST_CAT(dt_reg_, __LINE__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define WARN(...) ((void)0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                  \
        bool dt_caught = false;                                                           \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                    \
            dt_caught = true;                                                             \
        } catch (...) {                                                                   \
        }                                                                                 \
        ::doctest::detail::report(dt_caught, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                         \
    do {                                                                                  \
        bool dt_caught = false;                                                           \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const __VA_ARGS__& dt_e) {                                               \
            dt_caught = (matcher).matches(dt_e.what());                                   \
        } catch (...) {                                                                   \
        }                                                                                 \
        ::doctest::detail::report(dt_caught, "throws-with " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif

#endif
