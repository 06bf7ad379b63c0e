// check_libm.cpp — TEST INFRASTRUCTURE ONLY.
// Exhaustive (or strided) bitwise comparison of the glibc restatements in
// paper_2408_00018_b200/csrc/libm_glibc.cuh against the system libm.
//   ./check_libm [stride]      stride 1 = every float (about 5 minutes)
// Prints one line per function with the number of mismatches.
#define PSA_HD static inline
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include "../paper_2408_00018_b200/csrc/libm_glibc.cuh"

static uint32_t bits(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }
static float flt(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }

int main(int argc, char** argv) {
    const uint32_t stride = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 1;
    float (*volatile lsin)(float) = ::sinf;
    float (*volatile lcos)(float) = ::cosf;
    float (*volatile lexp)(float) = ::expf;
    unsigned long bad_s = 0, bad_c = 0, bad_e = 0, n_sc = 0, n_e = 0;
    // sinf / cosf: every finite float of both signs
    for (uint64_t u = 0; u < 0x7f800000ull; u += stride) {
        for (uint32_t sgn : {0u, 0x80000000u}) {
            const float x = flt(uint32_t(u) | sgn);
            if (bits(lsin(x)) != bits(psa::libm::sinf(x))) { if (bad_s++ < 5) std::printf("sinf %a\n", x); }
            if (bits(lcos(x)) != bits(psa::libm::cosf(x))) { if (bad_c++ < 5) std::printf("cosf %a\n", x); }
            ++n_sc;
        }
    }
    // expf: every float in [-inf, 89] (beyond overflows identically)
    for (uint64_t u = 0; u <= 0xff800000ull; u += stride) {
        const float x = flt(uint32_t(u));
        if (u < 0x80000000ull && x > 89.0f) continue;
        if (bits(lexp(x)) != bits(psa::libm::expf(x))) { if (bad_e++ < 5) std::printf("expf %a\n", x); }
        ++n_e;
    }
    std::printf("sinf: %lu mismatches of %lu\ncosf: %lu mismatches of %lu\nexpf: %lu mismatches of %lu\n",
                bad_s, n_sc, bad_c, n_sc, bad_e, n_e);
    return (bad_s || bad_c || bad_e) ? 1 : 0;
}
