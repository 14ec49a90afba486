// TEST INFRASTRUCTURE: a minimal stand-in for Catch2's single header (Catch2
// is not installed here), enough to compile and run the reference's own
// unit tests (proj/tests/*.cpp) against the drop-in headers: TEST_CASE,
// REQUIRE / REQUIRE_FALSE / REQUIRE_THROWS_AS, INFO and Catch::Approx with
// Catch2 v3's comparison rule.  main() runs every test case, or those whose
// name contains / whose tags contain an argument.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
    std::string name, tags;
    std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* tags, void (*fn)()) { registry().push_back({name, tags, fn}); }
};
struct Failure {
    std::string where;
};
inline std::string& info_text() {
    static std::string s;
    return s;
}

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
    bool equals(double other) const {
        auto within = [](double a, double b, double m) { return (a + m >= b) && (b + m >= a); };
        return within(value_, other, margin_) ||
               within(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    friend bool operator==(double a, const Approx& b) { return b.equals(a); }
    friend bool operator==(const Approx& a, double b) { return a.equals(b); }
    friend bool operator!=(double a, const Approx& b) { return !b.equals(a); }
    friend bool operator!=(const Approx& a, double b) { return !a.equals(b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.equals(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.equals(a); }
    friend bool operator<=(const Approx& a, double b) { return a.value_ < b || a.equals(b); }
    friend bool operator>=(const Approx& a, double b) { return a.value_ > b || a.equals(b); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double margin_ = 0.0;
    double scale_ = 0.0;
};

}  // namespace Catch

#define CATCH_CAT2(a, b) a##b
#define CATCH_CAT(a, b) CATCH_CAT2(a, b)
#define TEST_CASE(name, tags)                                                              \
    static void CATCH_CAT(catch_test_, __LINE__)();                                        \
    static ::Catch::Registrar CATCH_CAT(catch_reg_, __LINE__)(name, tags,                  \
                                                              &CATCH_CAT(catch_test_, __LINE__)); \
    static void CATCH_CAT(catch_test_, __LINE__)()
#define CATCH_FAIL_AT(text)                                                                 \
    do {                                                                                    \
        std::ostringstream o_;                                                              \
        o_ << __FILE__ << ":" << __LINE__ << ": " << text;                                  \
        throw ::Catch::Failure{o_.str()};                                                   \
    } while (0)
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        if (!(__VA_ARGS__)) CATCH_FAIL_AT("REQUIRE(" #__VA_ARGS__ ")");                     \
    } while (0)
#define REQUIRE_FALSE(...)                                                                  \
    do {                                                                                    \
        if ((__VA_ARGS__)) CATCH_FAIL_AT("REQUIRE_FALSE(" #__VA_ARGS__ ")");                \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                       \
    do {                                                                                    \
        bool caught_ = false;                                                               \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const type&) {                                                             \
            caught_ = true;                                                                 \
        } catch (...) {                                                                     \
        }                                                                                   \
        if (!caught_) CATCH_FAIL_AT("REQUIRE_THROWS_AS(" #expr ", " #type ")");             \
    } while (0)
#define INFO(msg)                                                                           \
    do {                                                                                    \
        std::ostringstream o_;                                                              \
        o_ << msg;                                                                          \
        ::Catch::info_text() = o_.str();                                                    \
    } while (0)

#ifdef CATCH_SHIM_MAIN
int main(int argc, char** argv) {
    int run = 0, failed = 0;
    for (const auto& t : ::Catch::registry()) {
        bool pick = argc < 2;
        for (int a = 1; a < argc; ++a)
            if (t.name.find(argv[a]) != std::string::npos || t.tags.find(argv[a]) != std::string::npos)
                pick = true;
        if (!pick) continue;
        ++run;
        ::Catch::info_text().clear();
        try {
            t.fn();
            std::printf("ok     %s\n", t.name.c_str());
        } catch (const ::Catch::Failure& f) {
            ++failed;
            std::printf("FAILED %s\n  %s\n  info: %s\n", t.name.c_str(), f.where.c_str(),
                        ::Catch::info_text().c_str());
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAILED %s\n  exception: %s\n", t.name.c_str(), e.what());
        }
        std::fflush(stdout);
    }
    std::printf("%d test cases, %d failed\n", run, failed);
    return failed ? 1 : 0;
}
#endif
