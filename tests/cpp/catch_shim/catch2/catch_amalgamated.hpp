// TEST INFRASTRUCTURE. A Catch2-v3-compatible macro shim, just large enough to
// compile the reference's own unit suites (/root/reference/proj/tests/*.cpp)
// UNMODIFIED against the B200 drop-in headers (include/simplexmap/*.hpp ->
// include/simplexmap_b200.hpp). Catch2 itself is not installed here
// (SURVEY 0.5). Supported: TEST_CASE(name[, tags]), CHECK / REQUIRE /
// CHECK_FALSE / CHECK_NOTHROW / CHECK_THROWS_AS / CHECK_THAT /
// CHECK_THROWS_MATCHES, INFO, FAIL, Catch::Approx,
// Catch::Matchers::ContainsSubstring / MessageMatches. The runner (main) is
// catch_amalgamated.cpp, as with the real amalgamated Catch2.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace Catch {

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
struct RunState {
    long checks = 0, failures = 0;
    const char* current = "";
    std::vector<std::string> info;
};
inline RunState& state() {
    static RunState s;
    return s;
}
struct RequireFailure {};

inline void report(bool ok, const char* file, int line, const char* what, bool fatal,
                   const std::string& extra = {}) {
    RunState& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s%s%s\n", file, line, s.current, what,
                 extra.empty() ? "" : " -- ", extra.c_str());
    for (const auto& i : s.info) std::fprintf(stderr, "    with: %s\n", i.c_str());
    if (fatal) throw RequireFailure{};
}

struct InfoScope {
    explicit InfoScope(std::string msg) { state().info.push_back(std::move(msg)); }
    ~InfoScope() { state().info.pop_back(); }
};

// Catch::Approx: relative epsilon (default 100 float epsilons) or margin.
class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& margin(double m) { margin_ = m; return *this; }
    friend bool operator==(double a, const Approx& b) { return b.equal(a); }
    friend bool operator==(const Approx& b, double a) { return b.equal(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.equal(a); }

  private:
    bool equal(double a) const {
        const double d = std::fabs(a - v_);  // Catch2: margin, or eps relative to the target
        return d <= margin_ || d <= eps_ * (std::isinf(v_) ? 0.0 : std::fabs(v_));
    }
    double v_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100.0;
    double margin_ = 0.0;
};

namespace Matchers {
struct ContainsSubstring {
    explicit ContainsSubstring(std::string s) : s_(std::move(s)) {}
    bool match(const std::string& hay) const { return hay.find(s_) != std::string::npos; }
    std::string describe() const { return "contains \"" + s_ + "\""; }
    std::string s_;
};
struct Equals {
    explicit Equals(std::string s) : s_(std::move(s)) {}
    bool match(const std::string& v) const { return v == s_; }
    std::string describe() const { return "equals \"" + s_ + "\""; }
    std::string s_;
};
template <class Inner>
struct MessageMatchesT {
    Inner inner;
    bool match(const std::exception& e) const { return inner.match(e.what()); }
    std::string describe() const { return "message " + inner.describe(); }
};
template <class Inner>
MessageMatchesT<Inner> MessageMatches(Inner m) {
    return {std::move(m)};
}
}  // namespace Matchers

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TC(fn, name, ...)                                        \
    static void fn();                                                       \
    static ::Catch::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn);          \
    static void fn()
#define TEST_CASE(...) CATCH_SHIM_TC(CATCH_SHIM_CAT(catch_shim_tc_, __LINE__), __VA_ARGS__)

#define CATCH_SHIM_CHECK(expr, fatal, negate)                                                    \
    do {                                                                                         \
        bool catch_ok_ = false;                                                                  \
        std::string catch_x_;                                                                    \
        try {                                                                                    \
            catch_ok_ = static_cast<bool>(expr) != (negate);                                     \
        } catch (const std::exception& e) {                                                      \
            catch_x_ = std::string("threw: ") + e.what();                                        \
        } catch (...) {                                                                          \
            catch_x_ = "threw an unknown exception";                                             \
        }                                                                                        \
        ::Catch::report(catch_ok_, __FILE__, __LINE__, (negate) ? "!(" #expr ")" : #expr, fatal, \
                        catch_x_);                                                               \
    } while (0)
#define CHECK(...) CATCH_SHIM_CHECK((__VA_ARGS__), false, false)
#define REQUIRE(...) CATCH_SHIM_CHECK((__VA_ARGS__), true, false)
#define CHECK_FALSE(...) CATCH_SHIM_CHECK((__VA_ARGS__), false, true)
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK((__VA_ARGS__), true, true)

#define CATCH_SHIM_NOTHROW(expr, fatal)                                                 \
    do {                                                                                \
        std::string catch_x_;                                                           \
        bool catch_ok_ = true;                                                          \
        try {                                                                           \
            static_cast<void>(expr);                                                    \
        } catch (const std::exception& e) {                                             \
            catch_ok_ = false;                                                          \
            catch_x_ = e.what();                                                        \
        } catch (...) {                                                                 \
            catch_ok_ = false;                                                          \
        }                                                                               \
        ::Catch::report(catch_ok_, __FILE__, __LINE__, "nothrow: " #expr, fatal, catch_x_); \
    } while (0)
#define CHECK_NOTHROW(expr) CATCH_SHIM_NOTHROW(expr, false)
#define REQUIRE_NOTHROW(expr) CATCH_SHIM_NOTHROW(expr, true)

#define CATCH_SHIM_THROWS_AS(expr, type, fatal)                                                  \
    do {                                                                                         \
        bool catch_ok_ = false;                                                                  \
        std::string catch_x_ = "did not throw";                                                  \
        try {                                                                                    \
            static_cast<void>(expr);                                                             \
        } catch (const type&) {                                                                  \
            catch_ok_ = true;                                                                    \
        } catch (const std::exception& e) {                                                      \
            catch_x_ = std::string("threw another type: ") + e.what();                           \
        } catch (...) {                                                                          \
            catch_x_ = "threw another type";                                                     \
        }                                                                                        \
        ::Catch::report(catch_ok_, __FILE__, __LINE__, "throws " #type ": " #expr, fatal, catch_x_); \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCH_SHIM_THROWS_AS(expr, type, true)
#define CHECK_THROWS(expr) CATCH_SHIM_THROWS_AS(expr, std::exception, false)
#define REQUIRE_THROWS(expr) CATCH_SHIM_THROWS_AS(expr, std::exception, true)

#define CHECK_THAT(arg, matcher)                                                                    \
    do {                                                                                            \
        const auto& catch_m_ = (matcher);                                                           \
        ::Catch::report(catch_m_.match(arg), __FILE__, __LINE__, #arg " " #matcher, false,          \
                        catch_m_.describe());                                                       \
    } while (0)
#define REQUIRE_THAT(arg, matcher)                                                                  \
    do {                                                                                            \
        const auto& catch_m_ = (matcher);                                                           \
        ::Catch::report(catch_m_.match(arg), __FILE__, __LINE__, #arg " " #matcher, true,           \
                        catch_m_.describe());                                                       \
    } while (0)

#define CHECK_THROWS_MATCHES(expr, type, matcher)                                                 \
    do {                                                                                          \
        bool catch_ok_ = false;                                                                   \
        std::string catch_x_ = "did not throw";                                                   \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const type& e) {                                                                 \
            catch_ok_ = (matcher).match(e);                                                       \
            catch_x_ = e.what();                                                                  \
        } catch (...) {                                                                           \
            catch_x_ = "threw another type";                                                      \
        }                                                                                         \
        ::Catch::report(catch_ok_, __FILE__, __LINE__, "throws matching: " #expr, false, catch_x_); \
    } while (0)

#define INFO(msg)                                                              \
    ::Catch::InfoScope CATCH_SHIM_CAT(catch_info_, __LINE__)([&] {             \
        std::ostringstream catch_os_;                                          \
        catch_os_ << msg;                                                      \
        return catch_os_.str();                                                \
    }())
#define CAPTURE(x) INFO(#x " := " << (x))
#define FAIL(msg)                                                                        \
    do {                                                                                 \
        std::ostringstream catch_os_;                                                    \
        catch_os_ << msg;                                                                \
        ::Catch::report(false, __FILE__, __LINE__, "FAIL", true, catch_os_.str());       \
    } while (0)
#define SUCCEED(msg) ::Catch::report(true, __FILE__, __LINE__, "SUCCEED", false)
