// TEST INFRASTRUCTURE — a minimal stand-in for the doctest single header
// (absent from the reference tree: proj/vendor/ is empty), enough to compile
// the reference's own unmodified tests/test_capi.cpp: TEST_CASE, CHECK,
// REQUIRE and a main() that runs every case and reports failures.
#pragma once
#include <cstdio>
#include <exception>
#include <vector>

namespace doctest_shim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Register {
    Register(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};
struct RequireFailed : std::exception {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    if (ok) return;
    ++failures();
    std::printf("FAIL %s:%d %s\n", file, line, expr);
    if (require) throw RequireFailed();
}
}  // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                       \
    static void fn();                                                                 \
    static doctest_shim::Register DOCTEST_CAT(fn, _reg)(name, &fn);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    for (const auto& c : doctest_shim::cases()) {
        try {
            c.fn();
        } catch (const doctest_shim::RequireFailed&) {
            std::printf("  (case aborted: %s)\n", c.name);
        } catch (const std::exception& e) {
            ++doctest_shim::failures();
            std::printf("FAIL exception in %s: %s\n", c.name, e.what());
        }
    }
    std::printf("%zu test cases, %d failed checks\n", doctest_shim::cases().size(), doctest_shim::failures());
    return doctest_shim::failures() ? 1 : 0;
}
#endif
