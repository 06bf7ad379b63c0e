// check_libm64.cpp — TEST INFRASTRUCTURE ONLY.
// Random-sample bitwise comparison of the double-precision glibc
// restatements (paper_2408_00018_b200/csrc/libm_glibc64.cuh) against the
// system libm over the argument ranges the reference's cost functions use.
//   ./check_libm64 [samples_per_range]
#define PSA_HD static inline
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "../paper_2408_00018_b200/csrc/libm_glibc64.cuh"

static uint64_t bits(double f) { uint64_t u; std::memcpy(&u, &f, 8); return u; }
static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand() { // xorshift64*
    rng_state ^= rng_state >> 12; rng_state ^= rng_state << 25; rng_state ^= rng_state >> 27;
    return double((rng_state * 0x2545F4914F6CDD1Dull) >> 11) * 0x1p-53;
}

int main(int argc, char** argv) {
    const long N = argc > 1 ? std::atol(argv[1]) : 1000000;
    double (*volatile lsin)(double) = ::sin;
    double (*volatile lcos)(double) = ::cos;
    double (*volatile lexp)(double) = ::exp;
    const double ranges[][2] = {{1e-9, 0.126}, {0.126, 0.855469}, {0.855469, 2.426265},
                                {2.426265, 23.0}, {23.0, 4000.0}, {-30.0, 30.0}};
    int fail = 0;
    for (auto& r : ranges) {
        long bs = 0, bc = 0;
        for (long i = 0; i < N; ++i) {
            const double x = r[0] + (r[1] - r[0]) * urand();
            if (bits(lsin(x)) != bits(psa::libm::sin(x))) { if (bs++ < 3) std::printf("  sin %a: %a vs %a\n", x, lsin(x), psa::libm::sin(x)); }
            if (bits(lcos(x)) != bits(psa::libm::cos(x))) { if (bc++ < 3) std::printf("  cos %a: %a vs %a\n", x, lcos(x), psa::libm::cos(x)); }
        }
        std::printf("sin/cos [%g, %g): sin %ld, cos %ld mismatches of %ld\n", r[0], r[1], bs, bc, N);
        fail |= bs || bc;
    }
    const double eranges[][2] = {{-745.2, -708.0}, {-708.0, 0.0}, {-1.0, 1.0}, {-1e-10, 1e-10}, {0.0, 709.0}};
    for (auto& r : eranges) {
        long be = 0;
        for (long i = 0; i < N; ++i) {
            const double x = r[0] + (r[1] - r[0]) * urand();
            if (bits(lexp(x)) != bits(psa::libm::exp(x))) { if (be++ < 3) std::printf("  exp %a: %a vs %a\n", x, lexp(x), psa::libm::exp(x)); }
        }
        std::printf("exp [%g, %g): %ld mismatches of %ld\n", r[0], r[1], be, N);
        fail |= be != 0;
    }
    return fail;
}
