// TEST INFRASTRUCTURE. The runner of the Catch2 macro shim: runs every
// registered TEST_CASE (optionally only those whose name contains argv[1]),
// prints a summary, exits nonzero on any failure.
#include <catch2/catch_amalgamated.hpp>

#include <cstring>

int main(int argc, char** argv) {
    auto& s = Catch::state();
    int cases = 0, failed_cases = 0;
    for (const auto& tc : Catch::registry()) {
        if (argc > 1 && !std::strstr(tc.name, argv[1])) continue;
        ++cases;
        s.current = tc.name;
        const long before = s.failures;
        try {
            tc.fn();
        } catch (const Catch::RequireFailure&) {
        } catch (const std::exception& e) {
            ++s.failures;
            std::fprintf(stderr, "FAILED in \"%s\": unexpected exception: %s\n", tc.name, e.what());
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("test cases: %d | %d passed | %d failed\nassertions: %ld | %ld passed | %ld failed\n", cases,
                cases - failed_cases, failed_cases, s.checks, s.checks - s.failures, s.failures);
    return failed_cases ? 1 : 0;
}
