// TEST INFRASTRUCTURE: prints the reference's random branchy program for each seed
// (tests/test_util.hpp:79 gen_random_ll, the generator of scheduler_tests.cpp:124-147),
// separated by a line "; seed N".  Header-only use of the reference's test utilities.
#include <cstdio>
#include <cstdlib>

#include "test_util.hpp"

int main(int argc, char** argv) {
    const unsigned long lo = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 100;
    const unsigned long hi = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 200;
    for (unsigned long s = lo; s < hi; ++s) std::printf("; seed %lu\n%s", s, testutil::gen_random_ll(s).c_str());
    return 0;
}
