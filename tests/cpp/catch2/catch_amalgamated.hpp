// Minimal Catch2-compatible test harness (the subset the reference's PULSE
// tests use: TEST_CASE, SECTION with re-execution, CHECK/REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, INFO, Catch::Approx).  Lets the reference's
// own test sources compile unmodified against include/pulse/*.hpp.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};

// Section re-execution: each run of a test case executes the code outside
// sections plus exactly one not-yet-run section (one nesting level).
struct SectionState {
    int target = 0;       // index of the section to run this time
    int seen = 0;         // sections encountered this run
    bool ran_one = false;
};
inline SectionState& sections() {
    static SectionState s;
    return s;
}
inline bool enter_section() {
    auto& s = sections();
    const int i = s.seen++;
    if (i == s.target && !s.ran_one) {
        s.ran_one = true;
        return true;
    }
    return false;
}

struct Stats {
    int checks = 0, failures = 0;
    std::string current;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};

inline std::vector<std::string>& info_stack() {
    static std::vector<std::string> v;
    return v;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++stats().checks;
    if (ok) return;
    ++stats().failures;
    std::fprintf(stderr, "%s:%d: FAILED in '%s': %s\n", file, line, stats().current.c_str(), expr);
    for (auto& m : info_stack()) std::fprintf(stderr, "    with: %s\n", m.c_str());
    if (fatal) throw RequireFailed{};
}

struct InfoScope {
    explicit InfoScope(std::string m) { info_stack().push_back(std::move(m)); }
    ~InfoScope() { info_stack().pop_back(); }
};

inline int run_all() {
    int failed_cases = 0;
    for (auto& c : registry()) {
        stats().current = c.name;
        const int before = stats().failures;
        int target = 0;
        while (true) {
            auto& s = sections();
            s = SectionState{};
            s.target = target;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++stats().failures;
                std::fprintf(stderr, "'%s': unexpected exception: %s\n", c.name, e.what());
            } catch (...) {
                ++stats().failures;
                std::fprintf(stderr, "'%s': unexpected non-std exception\n", c.name);
            }
            info_stack().clear();
            if (++target >= sections().seen) break;
        }
        if (stats().failures != before) ++failed_cases;
    }
    std::printf("%s: %zu test cases, %d failed; %d assertions, %d failed\n",
                failed_cases ? "FAILED" : "All tests passed", registry().size(), failed_cases, stats().checks,
                stats().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace catch_shim

namespace Catch {
class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double x, const Approx& a) {
        return std::fabs(x - a.v_) <= std::max(a.margin_, a.eps_ * (1.0 + std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double x) { return x == a; }

private:
    double v_, margin_ = 0.0, eps_ = 1.1920929e-07 * 100;  // Catch2 default: 100 float ulps
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                               \
    static void fn();                                                          \
    static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn);          \
    static void fn()
#define TEST_CASE(name, ...) TEST_CASE_IMPL(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)
#define SECTION(name) if (catch_shim::enter_section())
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CATCH_SHIM_THROWS(expr, type, fatal)                                                                  \
    do {                                                                                                     \
        bool caught_ = false;                                                                                \
        try {                                                                                                \
            (void)(expr);                                                                                    \
        } catch (const type&) {                                                                              \
            caught_ = true;                                                                                  \
        } catch (const std::exception& e_) {                                                                 \
            std::fprintf(stderr, "    threw other exception: %s\n", e_.what());                            \
        } catch (...) {                                                                                      \
        }                                                                                                    \
        catch_shim::report(caught_, #expr " throws " #type, __FILE__, __LINE__, fatal);                      \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS(expr, type, false)
#define CAPTURE(...) ((void)0)  // Catch logs the values on failure; the shim reports the expression
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS(expr, type, true)
#define CHECK_NOTHROW(expr)                                                                    \
    do {                                                                                       \
        bool ok_ = true;                                                                       \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const std::exception& e_) {                                                   \
            ok_ = false;                                                                       \
            std::fprintf(stderr, "    threw: %s\n", e_.what());                              \
        } catch (...) {                                                                        \
            ok_ = false;                                                                       \
        }                                                                                      \
        catch_shim::report(ok_, #expr " does not throw", __FILE__, __LINE__, false);           \
    } while (0)
#define INFO(msg)                                                                 \
    catch_shim::InfoScope CATCH_SHIM_CAT(catch_shim_info_, __LINE__)(            \
        (std::ostringstream() << msg).str())
