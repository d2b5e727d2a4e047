// Runner for the reference's doctest cases (TEST INFRASTRUCTURE): one line per
// case, "PASS name" / "FAIL name", exit code = number of failing cases.
#include <cstdio>
#include "doctest.h"

int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        const int before = doctest::detail::failures();
        bool threw = false;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            std::printf("  exception: %s\n", e.what());
            ++doctest::detail::failures();
        }
        const bool ok = doctest::detail::failures() == before && !threw;
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
        failed_cases += ok ? 0 : 1;
    }
    std::printf("%d cases, %d failed\n", int(doctest::detail::registry().size()), failed_cases);
    return failed_cases;
}
