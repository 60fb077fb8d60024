// TEST INFRASTRUCTURE ONLY — a minimal, from-scratch stand-in for the subset of the doctest
// API the reference's unit tests use (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// REQUIRE_MESSAGE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, INFO, CAPTURE, doctest::Approx,
// doctest::Contains). doctest itself is not vendored in /root/reference (proj/.gitignore), so
// this shim lets oracle/Makefile compile the reference's own test files unmodified against
// the B200 drop-in library (include/seghdc) and run them on the GPU box.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
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
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), what);
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

private:
    double v_;
    double eps_ = 1.19209290e-07 * 100;  // doctest's default: 100 * float epsilon
};

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
    bool matches(const std::string& m) const { return m.find(s) != std::string::npos; }
};
inline bool message_matches(const Contains& c, const std::string& m) { return c.matches(m); }
inline bool message_matches(const char* exact, const std::string& m) { return m == exact; }
inline bool message_matches(const std::string& exact, const std::string& m) { return m == exact; }

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                         \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                           \
    static ::doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define CHECK(...)                                                                    \
    do {                                                                              \
        if (!(__VA_ARGS__)) ::doctest::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK_FALSE(...)                                                              \
    do {                                                                              \
        if ((__VA_ARGS__)) ::doctest::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE(...)                                                                  \
    do {                                                                              \
        if (!(__VA_ARGS__)) {                                                         \
            ::doctest::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");      \
            throw ::doctest::RequireFailed{};                                         \
        }                                                                             \
    } while (0)
#define REQUIRE_MESSAGE(cond, ...) REQUIRE(cond)
#define CHECK_THROWS_AS(expr, exc)                                                    \
    do {                                                                              \
        bool caught_ = false;                                                         \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const exc&) {                                                        \
            caught_ = true;                                                           \
        } catch (...) {                                                               \
        }                                                                             \
        if (!caught_) ::doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #exc ")"); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, exc)                                      \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const exc& e_) {                                                     \
            ok_ = ::doctest::message_matches(matcher, std::string(e_.what()));        \
        } catch (...) {                                                               \
        }                                                                             \
        if (!ok_) ::doctest::report(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")"); \
    } while (0)
#define INFO(...) ((void)0)
#define CAPTURE(x) ((void)(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::registry()) {
        ::doctest::current() = tc.name;
        const int before = ::doctest::failures();
        try {
            tc.fn();
        } catch (const ::doctest::RequireFailed&) {
        } catch (const std::exception& e) {
            ::doctest::report(__FILE__, __LINE__, e.what());
        }
        ++cases;
        if (::doctest::failures() != before) ++failed_cases;
    }
    std::printf("[doctest shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
    return failed_cases ? 1 : 0;
}
#endif
