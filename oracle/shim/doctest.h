// Minimal doctest-compatible shim — TEST INFRASTRUCTURE ONLY.
//
// The reference's tests include <doctest.h> from proj/vendor/, which is gitignored and
// absent (proj/.gitignore:2). This header implements the macro subset they use
// (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS*, CHECK_NOTHROW, doctest::Approx,
// doctest::Contains) so the reference test files compile unmodified and validate the
// Eigen shim (oracle/shim/Eigen/Dense). Command line: `-tce=<substr>[,<substr>]`
// excludes test cases whose name contains a substring (used for the CLI-dependent
// cases of test_pipeline.cpp, whose CLI11 front-end is absent).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <map>
#include <set>
#include <tuple>
#include <unordered_map>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool equals(double lhs) const {
        return std::fabs(lhs - value_) <
               epsilon_ * (scale_ + std::max<double>(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double epsilon_;
    double scale_ = 1.0;
};

template <typename T>
bool operator==(const T& lhs, const Approx& rhs) { return rhs.equals(static_cast<double>(lhs)); }
template <typename T>
bool operator==(const Approx& lhs, const T& rhs) { return lhs.equals(static_cast<double>(rhs)); }
template <typename T>
bool operator!=(const T& lhs, const Approx& rhs) { return !rhs.equals(static_cast<double>(lhs)); }
template <typename T>
bool operator!=(const Approx& lhs, const T& rhs) { return !lhs.equals(static_cast<double>(rhs)); }
template <typename T>
bool operator<=(const T& lhs, const Approx& rhs) { return static_cast<double>(lhs) < rhs.value() || rhs.equals(static_cast<double>(lhs)); }
template <typename T>
bool operator>=(const T& lhs, const Approx& rhs) { return static_cast<double>(lhs) > rhs.value() || rhs.equals(static_cast<double>(lhs)); }
template <typename T>
bool operator<(const T& lhs, const Approx& rhs) { return static_cast<double>(lhs) < rhs.value() && !rhs.equals(static_cast<double>(lhs)); }
template <typename T>
bool operator>(const T& lhs, const Approx& rhs) { return static_cast<double>(lhs) > rhs.value() && !rhs.equals(static_cast<double>(lhs)); }

class Contains {
public:
    explicit Contains(const char* s) : s_(s) {}
    bool check_in(const std::string& text) const { return text.find(s_) != std::string::npos; }

private:
    std::string s_;
};

namespace detail {

struct RequireAbort {};

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
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
inline const char*& current() {
    static const char* c = "";
    return c;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line, bool require) {
    ++asserts();
    if (ok) return;
    ++failures();
    std::printf("%s:%d: FAILED in \"%s\": %s( %s )\n", file, line, current(), kind, expr);
    if (require) throw RequireAbort{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                    \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(               \
        name, __FILE__, __LINE__, &DOCTEST_CAT(doctest_fn_, __LINE__));                    \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define DOCTEST_ASSERT_IMPL(kind, require, ...)                                            \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
        } catch (const ::doctest::detail::RequireAbort&) {                                 \
            throw;                                                                         \
        } catch (...) {                                                                    \
            doctest_ok_ = false;                                                           \
        }                                                                                  \
        ::doctest::detail::report(doctest_ok_, kind, #__VA_ARGS__, __FILE__, __LINE__, require); \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", true, !(__VA_ARGS__))

#define DOCTEST_THROWS_AS_IMPL(kind, require, expr, ...)                                   \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            static_cast<void>(expr);                                                       \
        } catch (const __VA_ARGS__&) {                                                     \
            doctest_ok_ = true;                                                            \
        } catch (...) {                                                                    \
        }                                                                                  \
        ::doctest::detail::report(doctest_ok_, kind, #expr, __FILE__, __LINE__, require);  \
    } while (0)

#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("CHECK_THROWS_AS", false, expr, __VA_ARGS__)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS_IMPL("REQUIRE_THROWS_AS", true, expr, __VA_ARGS__)

#define CHECK_THROWS(...)                                                                  \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            static_cast<void>(__VA_ARGS__);                                                \
        } catch (...) {                                                                    \
            doctest_ok_ = true;                                                            \
        }                                                                                  \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_NOTHROW(...)                                                                 \
    do {                                                                                   \
        bool doctest_ok_ = true;                                                           \
        try {                                                                              \
            static_cast<void>(__VA_ARGS__);                                                \
        } catch (...) {                                                                    \
            doctest_ok_ = false;                                                           \
        }                                                                                  \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                           \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            static_cast<void>(expr);                                                       \
        } catch (const __VA_ARGS__& e) {                                                   \
            doctest_ok_ = (matcher).check_in(e.what());                                    \
        } catch (...) {                                                                    \
        }                                                                                  \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, false); \
    } while (0)

#define MESSAGE(...) ((void)0)
#define INFO(...) ((void)0)
#define CAPTURE(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> excludes;
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        const char* key = "-tce=";
        if (std::strncmp(a, key, std::strlen(key)) == 0) {
            std::stringstream ss(a + std::strlen(key));
            std::string item;
            while (std::getline(ss, item, ',')) excludes.push_back(item);
        }
    }
    int run = 0, failed_cases = 0, skipped = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        bool skip = false;
        for (const auto& ex : excludes)
            if (std::string(tc.name).find(ex) != std::string::npos) skip = true;
        if (skip) {
            ++skipped;
            continue;
        }
        ::doctest::detail::current() = tc.name;
        const int before = ::doctest::detail::failures();
        ++run;
        try {
            tc.fn();
        } catch (const ::doctest::detail::RequireAbort&) {
        } catch (const std::exception& e) {
            ++::doctest::detail::failures();
            std::printf("%s:%d: ERROR in \"%s\": unexpected exception: %s\n", tc.file, tc.line, tc.name, e.what());
        } catch (...) {
            ++::doctest::detail::failures();
            std::printf("%s:%d: ERROR in \"%s\": unexpected exception\n", tc.file, tc.line, tc.name);
        }
        if (::doctest::detail::failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d run | %d passed | %d failed | %d skipped; assertions: %d | %d failed\n",
                run, run - failed_cases, failed_cases, skipped, ::doctest::detail::asserts(),
                ::doctest::detail::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
