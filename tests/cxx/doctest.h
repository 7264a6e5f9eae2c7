// Minimal doctest-compatible test shim (doctest itself is not vendored in the
// reference, proj/.gitignore:2). Covers what the reference's render-path suites
// use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, INFO, FAIL, doctest::Approx
// with .epsilon(). Lets tests/cxx run the reference's own test sources unmodified.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::fmax(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct Abort {};
inline int& failures() {
    static int n = 0;
    return n;
}
inline int& checks() {
    static int n = 0;
    return n;
}
inline std::vector<std::string>& infos() {
    static std::vector<std::string> v;
    return v;
}
struct InfoScope {
    explicit InfoScope(const std::string& s) { infos().push_back(s); }
    ~InfoScope() { infos().pop_back(); }
};
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
    for (const auto& s : infos()) std::fprintf(stderr, "  with: %s\n", s.c_str());
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                           \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                           \
    static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name,                          \
                                                                   DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                                \
    do {                                                                                          \
        ++doctest::detail::checks();                                                              \
        if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);            \
    } while (0)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        ++doctest::detail::checks();                                                              \
        if (!(__VA_ARGS__)) {                                                                     \
            doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                            \
            throw doctest::detail::Abort{};                                                       \
        }                                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                               \
    do {                                                                                          \
        ++doctest::detail::checks();                                                              \
        bool threw_ = false;                                                                      \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const type&) {                                                                   \
            threw_ = true;                                                                        \
        } catch (...) {                                                                           \
        }                                                                                         \
        if (!threw_) doctest::detail::report(__FILE__, __LINE__, "throws " #type ": " #expr);     \
    } while (0)
#define FAIL(msg)                                                                                 \
    do {                                                                                          \
        doctest::detail::report(__FILE__, __LINE__, msg);                                         \
        throw doctest::detail::Abort{};                                                           \
    } while (0)
#define INFO(...)                                                                                 \
    std::ostringstream DOCTEST_CAT(doctest_os_, __LINE__);                                        \
    DOCTEST_CAT(doctest_os_, __LINE__) << __VA_ARGS__;                                            \
    doctest::detail::InfoScope DOCTEST_CAT(doctest_info_, __LINE__)(DOCTEST_CAT(doctest_os_, __LINE__).str())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;
        const int before = doctest::detail::failures();
        try {
            c.fn();
        } catch (const doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            doctest::detail::report(__FILE__, __LINE__, e.what());
        }
        const bool ok = doctest::detail::failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu test cases, %d failed, %d checks, %d failed checks\n", doctest::detail::registry().size(),
                failed_cases, doctest::detail::checks(), doctest::detail::failures());
    return failed_cases ? 1 : 0;
}
#endif
