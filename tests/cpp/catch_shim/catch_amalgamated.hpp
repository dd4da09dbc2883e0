// Minimal Catch2-compatible harness, written for this repo: just the API the reference's unit
// tests use (TEST_CASE, SECTION, REQUIRE, REQUIRE_FALSE, REQUIRE_THROWS_AS, Catch::Approx with
// epsilon / margin).  Catch2 itself is not in this image; this lets tests/cpp/Makefile compile
// the reference's own test sources, unmodified and in place, against this repo's drop-in headers
// (include/phiquad -> libpq_b200.so on the B200).
//
// Semantics follow Catch2 v3 where the tests depend on them:
// * a TEST_CASE with SECTIONs is run once per section, each run entering exactly one new section
//   (sections are not nested in these tests);
// * REQUIRE failures abort the current run of the test case; the binary exits 1 if any failed;
// * Approx(v): |x - v| <= margin, or |x - v| <= epsilon * (scale + |v|), epsilon defaulting to
//   100 * FLT_EPSILON.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool equals(double x) const {
        auto within = [](double a, double b, double m) { return a + m >= b && b + m >= a; };
        return within(value_, x, margin_) ||
               within(value_, x, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double margin_ = 0.0;
    double scale_ = 0.0;
};
template <class T>
bool operator==(const T& x, const Approx& a) {
    return a.equals(static_cast<double>(x));
}
template <class T>
bool operator==(const Approx& a, const T& x) {
    return a.equals(static_cast<double>(x));
}
template <class T>
bool operator!=(const T& x, const Approx& a) {
    return !a.equals(static_cast<double>(x));
}
template <class T>
bool operator!=(const Approx& a, const T& x) {
    return !a.equals(static_cast<double>(x));
}
template <class T>
bool operator<=(const T& x, const Approx& a) {
    return static_cast<double>(x) < a.value() || a.equals(static_cast<double>(x));
}
template <class T>
bool operator>=(const T& x, const Approx& a) {
    return static_cast<double>(x) > a.value() || a.equals(static_cast<double>(x));
}

namespace shim {

struct Failure : std::exception {};

struct Case {
    std::string name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    int target = 0, seen = 0;
    bool more = false;
    long long assertions = 0;
    int failed_runs = 0;
};
inline State& state() {
    static State s;
    return s;
}
inline bool enter_section() {
    State& s = state();
    const int idx = s.seen++;
    if (idx == s.target) return true;
    if (idx > s.target) s.more = true;
    return false;
}
[[noreturn]] inline void fail(const char* file, int line, const char* what) {
    std::printf("%s:%d: FAILED: %s\n", file, line, what);
    std::fflush(stdout);
    throw Failure{};
}
inline void check(bool ok, const char* file, int line, const char* what) {
    ++state().assertions;
    if (!ok) fail(file, line, what);
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        bool case_ok = true;
        State& s = state();
        s.target = 0;
        do {
            s.seen = 0;
            s.more = false;
            try {
                c.fn();
            } catch (const Failure&) {
                case_ok = false;
            } catch (const std::exception& e) {
                std::printf("test case \"%s\": unexpected exception: %s\n", c.name.c_str(), e.what());
                case_ok = false;
            } catch (...) {
                std::printf("test case \"%s\": unexpected exception\n", c.name.c_str());
                case_ok = false;
            }
            ++s.target;
        } while (s.more);
        if (!case_ok) {
            ++failed_cases;
            std::printf("test case FAILED: %s\n", c.name.c_str());
        }
    }
    std::printf("%zu test cases, %d failed, %lld assertions\n", registry().size(), failed_cases,
                state().assertions);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace shim
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_CASE(fn, name)                                                         \
    static void fn();                                                                     \
    static const ::Catch::shim::Registrar CATCH_SHIM_CAT(fn, _reg){name, &fn};            \
    static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_CASE(CATCH_SHIM_CAT(catch_shim_case_, __COUNTER__), name)
#define SECTION(name, ...) if (::Catch::shim::enter_section())
#define REQUIRE(...) ::Catch::shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE_FALSE(...) ::Catch::shim::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE_THROWS_AS(expr, type)                                                             \
    do {                                                                                          \
        ++::Catch::shim::state().assertions;                                                      \
        bool caught_ = false;                                                                     \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const type&) {                                                                   \
            caught_ = true;                                                                       \
        } catch (...) {                                                                           \
        }                                                                                         \
        if (!caught_) ::Catch::shim::fail(__FILE__, __LINE__, "expected " #type " from " #expr); \
    } while (0)

#ifdef CATCH_SHIM_MAIN
int main() { return ::Catch::shim::run_all(); }
#endif
