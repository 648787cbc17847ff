// Minimal Catch2-v3-compatible test harness (TEST_CASE, SECTION, REQUIRE*,
// FAIL, Catch::Approx) — just enough for the reference's unit-test sources
// (proj/tests/test_*.cpp) to compile UNCHANGED against this repo's
// include/aidw headers and run on the GPU (Catch2 itself is not in the
// image).  Semantics kept: a failed REQUIRE aborts the current test-case
// run; each top-level SECTION runs in its own pass of the test case; exit
// status is non-zero when anything failed.  Compile exactly one TU with
// AIDW_CATCH_MAIN defined (tests/cpp/catch_main.cpp) to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
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
    friend bool operator==(double lhs, const Approx& a) {
        const double diff = std::fabs(lhs - a.value_);
        return diff <= a.margin_ ||
               diff <= a.eps_ * (std::isinf(a.value_) ? 0.0 : std::fabs(a.value_));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100.0;
    double margin_ = 0.0;
};

}  // namespace Catch

namespace aidw_catch {

struct Failure {};  // thrown by a failed REQUIRE

struct Registry {
    struct Case {
        std::string name;
        std::function<void()> fn;
    };
    std::vector<Case> cases;
    // section tracking for the running case
    std::set<std::string> done;
    bool entered = false;
    std::string active;
    long assertions = 0, failed_assertions = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct AutoReg {
    AutoReg(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};

struct Section {
    bool run = false;
    std::string id;
    Section(const char* name, int line) : id(std::string(name) + "#" + std::to_string(line)) {
        auto& r = Registry::get();
        if (!r.entered && !r.done.count(id)) {
            r.entered = true;
            r.active = id;
            run = true;
        }
    }
    ~Section() {
        if (run) Registry::get().done.insert(id);
    }
    explicit operator bool() const { return run; }
};

inline void report(bool ok, const char* expr, const char* file, int line,
                   const std::string& extra = "") {
    auto& r = Registry::get();
    ++r.assertions;
    if (ok) return;
    ++r.failed_assertions;
    std::printf("  FAILED %s:%d: %s %s\n", file, line, expr, extra.c_str());
    throw Failure{};
}

inline int run_all(int argc, char** argv) {
    auto& r = Registry::get();
    int failed_cases = 0, run_cases = 0;
    for (auto& c : r.cases) {
        if (argc > 1) {
            bool match = false;
            for (int i = 1; i < argc; ++i)
                if (c.name.find(argv[i]) != std::string::npos) match = true;
            if (!match) continue;
        }
        ++run_cases;
        r.done.clear();
        bool case_failed = false;
        do {
            r.entered = false;
            try {
                c.fn();
            } catch (const Failure&) {
                case_failed = true;
                if (r.entered) r.done.insert(r.active);
            } catch (const std::exception& e) {
                case_failed = true;
                ++r.failed_assertions;
                std::printf("  FAILED: unexpected exception: %s\n", e.what());
                if (r.entered) r.done.insert(r.active);
            }
        } while (r.entered);
        std::printf("[%s] %s\n", case_failed ? "FAIL" : "PASS", c.name.c_str());
        failed_cases += case_failed ? 1 : 0;
    }
    std::printf("test cases: %d run, %d failed | assertions: %ld, %ld failed\n", run_cases,
                failed_cases, r.assertions, r.failed_assertions);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace aidw_catch

#define AIDW_CATCH_CAT2(a, b) a##b
#define AIDW_CATCH_CAT(a, b) AIDW_CATCH_CAT2(a, b)
#define AIDW_CATCH_FN AIDW_CATCH_CAT(aidw_catch_case_, __LINE__)

#define TEST_CASE(...)                                                                  \
    static void AIDW_CATCH_FN();                                                        \
    static ::aidw_catch::AutoReg AIDW_CATCH_CAT(aidw_catch_reg_, __LINE__)(             \
        ::aidw_catch::first_arg(__VA_ARGS__), &AIDW_CATCH_FN);                          \
    static void AIDW_CATCH_FN()

namespace aidw_catch {
inline const char* first_arg(const char* name, const char* = "") { return name; }
}  // namespace aidw_catch

#define SECTION(name) if (::aidw_catch::Section aidw_catch_section{name, __LINE__})

#define REQUIRE(...) ::aidw_catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE_FALSE(...) ::aidw_catch::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define CHECK(...) REQUIRE(__VA_ARGS__)

#define REQUIRE_NOTHROW(...)                                                          \
    do {                                                                              \
        bool aidw_ok = true;                                                          \
        std::string aidw_what;                                                        \
        try {                                                                         \
            (void)(__VA_ARGS__);                                                      \
        } catch (const std::exception& e) {                                           \
            aidw_ok = false;                                                          \
            aidw_what = e.what();                                                     \
        } catch (...) {                                                               \
            aidw_ok = false;                                                          \
        }                                                                             \
        ::aidw_catch::report(aidw_ok, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, aidw_what); \
    } while (0)

#define REQUIRE_THROWS(...)                                                           \
    do {                                                                              \
        bool aidw_threw = false;                                                      \
        try {                                                                         \
            (void)(__VA_ARGS__);                                                      \
        } catch (...) {                                                               \
            aidw_threw = true;                                                        \
        }                                                                             \
        ::aidw_catch::report(aidw_threw, "THROWS " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#define REQUIRE_THROWS_AS(expr, type)                                                 \
    do {                                                                              \
        bool aidw_right = false;                                                      \
        std::string aidw_what = "(no exception)";                                     \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type&) {                                                       \
            aidw_right = true;                                                        \
        } catch (const std::exception& e) {                                           \
            aidw_what = std::string("(other exception: ") + e.what() + ")";           \
        } catch (...) {                                                               \
            aidw_what = "(non-std exception)";                                        \
        }                                                                             \
        ::aidw_catch::report(aidw_right, "THROWS_AS " #type " " #expr, __FILE__, __LINE__, \
                             aidw_right ? "" : aidw_what);                            \
    } while (0)

#define FAIL(msg) ::aidw_catch::report(false, "FAIL", __FILE__, __LINE__, msg)

#ifdef AIDW_CATCH_MAIN
int main(int argc, char** argv) { return ::aidw_catch::run_all(argc, argv); }
#endif
