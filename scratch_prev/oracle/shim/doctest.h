// Minimal doctest-compatible shim (TEST INFRASTRUCTURE).  doctest itself is
// not vendored in /root/reference (proj/.gitignore:2) and there is no
// network; this implements exactly the subset the reference's unit tests use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, FAIL, FAIL_CHECK,
// doctest::Approx(...).epsilon(...)) so proj/tests/test_*.cpp compile
// unchanged against oracle/_ref/libpipesim.a.
#pragma once

#include <cmath>
#include <cstdio>
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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& asserts() {
    static int a = 0;
    return a;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, std::function<void()> fn) {
        registry().push_back({name, file, line, std::move(fn)});
    }
};
struct RequireFailed {};
inline void report(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}
template <class... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                              \
    static void fn();                                                                          \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn);   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define CHECK(...)                                                                             \
    do {                                                                                       \
        ++::doctest::detail::asserts();                                                        \
        if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")"); \
    } while (0)
#define CHECK_FALSE(...)                                                                       \
    do {                                                                                       \
        ++::doctest::detail::asserts();                                                        \
        if ((__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_FALSE(" #__VA_ARGS__ ")"); \
    } while (0)
#define REQUIRE(...)                                                                           \
    do {                                                                                       \
        ++::doctest::detail::asserts();                                                        \
        if (!(__VA_ARGS__)) {                                                                  \
            ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");        \
            throw ::doctest::detail::RequireFailed{};                                          \
        }                                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
    do {                                                                                       \
        ++::doctest::detail::asserts();                                                        \
        bool thrown_ok_ = false;                                                               \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            thrown_ok_ = true;                                                                 \
        } catch (...) {                                                                        \
        }                                                                                      \
        if (!thrown_ok_) ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #type ")"); \
    } while (0)
#define FAIL(...)                                                                              \
    do {                                                                                       \
        ::doctest::detail::report(__FILE__, __LINE__, ::doctest::detail::cat(__VA_ARGS__));   \
        throw ::doctest::detail::RequireFailed{};                                              \
    } while (0)
#define FAIL_CHECK(...) ::doctest::detail::report(__FILE__, __LINE__, ::doctest::detail::cat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        const int before = ::doctest::detail::failures();
        try {
            c.fn();
        } catch (const ::doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ::doctest::detail::report(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            ::doctest::detail::report(c.file, c.line, "unexpected exception");
        }
        if (::doctest::detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", c.name);
        }
    }
    const int n = (int)::doctest::detail::registry().size();
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %d\n", n,
                n - failed_cases, failed_cases, ::doctest::detail::asserts());
    return failed_cases ? 1 : 0;
}
#endif
