// Runner for the Catch2-subset shim: runs every registered case, prints a
// summary line "cases=N checks=C failures=F", exits non-zero on failure.
#include "catch_amalgamated.hpp"

int main() {
    long failed_cases = 0;
    for (const auto& c : shim::registry()) {
        long before = shim::failures();
        shim::info().clear();
        try {
            c.fn();
        } catch (const shim::Abort&) {
        } catch (const std::exception& e) {
            ++shim::failures();
            std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
        }
        if (shim::failures() != before) ++failed_cases;
    }
    std::printf("cases=%zu checks=%ld failures=%ld failed_cases=%ld\n", shim::registry().size(),
                shim::checks(), shim::failures(), failed_cases);
    return shim::failures() ? 1 : 0;
}
