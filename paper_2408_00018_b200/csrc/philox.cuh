// philox.cuh — counter-based streams, bit-identical to the reference.
//
// Reference: rng.hpp:13-18 (bit spec), :30-33 (constants), :39-52 (cipher),
// :66-81 (uniform and coordinate index).  Draw i of stream (seed, chain,
// level) is philox4x32_10({lo32(i), hi32(i), chain, level}, {lo32(seed),
// hi32(seed)}); only out[0], out[1] are used.
//
// Device layout: the ten round keys depend on the seed only, so the host
// precomputes them once (PhiloxKeys) and they reach the kernel as uniform
// kernel parameters; a draw then costs 10 x (2 IMAD.WIDE.U32 + 2 LOP3), with
// the dead half of the last round eliminated.
#pragma once

#include <stdint.h>

#ifndef PSA_HD
#define PSA_HD __host__ __device__ __forceinline__
#endif

namespace psa {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

struct PhiloxKeys {
    uint32_t k0[10];
    uint32_t k1[10];
};

PSA_HD PhiloxKeys make_keys(uint64_t seed) {
    PhiloxKeys k;
    uint32_t a = static_cast<uint32_t>(seed), b = static_cast<uint32_t>(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        k.k0[r] = a;
        k.k1[r] = b;
        a += kPhiloxW0;
        b += kPhiloxW1;
    }
    return k;
}

PSA_HD void mulhilo(uint32_t a, uint32_t m, uint32_t& hi, uint32_t& lo) {
    const uint64_t p = static_cast<uint64_t>(m) * a;
    hi = static_cast<uint32_t>(p >> 32);
    lo = static_cast<uint32_t>(p);
}

// Full 4x32 block (used by the KAT probe).
PSA_HD void philox4x32_10(uint32_t v[4], const PhiloxKeys& key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(v[0], kPhiloxM0, hi0, lo0);
        mulhilo(v[2], kPhiloxM1, hi1, lo1);
        const uint32_t n0 = hi1 ^ v[1] ^ key.k0[r];
        const uint32_t n2 = hi0 ^ v[3] ^ key.k1[r];
        v[0] = n0;
        v[1] = lo1;
        v[2] = n2;
        v[3] = lo0;
    }
}

// The 53-bit mantissa integer m of draw `counter`: u = m * 2^-53
// (rng.hpp:72-74: bits = out1<<32 | out0; u = (bits >> 11) * 2^-53).
PSA_HD uint64_t draw_bits53(uint64_t counter, uint32_t chain, uint32_t level,
                            const PhiloxKeys& key) {
    uint32_t v[4] = {static_cast<uint32_t>(counter), static_cast<uint32_t>(counter >> 32), chain,
                     level};
    philox4x32_10(v, key);
    const uint64_t bits = (static_cast<uint64_t>(v[1]) << 32) | static_cast<uint64_t>(v[0]);
    return bits >> 11;
}

PSA_HD double bits_to_uniform(uint64_t m) { return static_cast<double>(m) * 0x1.0p-53; }

// ---------------------------------------------------------------------------
// Per-(chain, level) precomputation for counters below 2^32.
//
// Draw i of stream (seed, c, l) enciphers {i, 0, c, l}.  In round 1 the
// product M1*c and the words it feeds do not depend on i, and in round 2 the
// product M0*v0 does not either, so for a fixed (c, l) a draw costs
// 17 IMAD.WIDE.U32 + 18 LOP3 instead of 20 + 20 plus key moves.  Identical
// bits to philox4x32_10 (tests/test_gpu_parity.py compares every stream).
// ---------------------------------------------------------------------------
struct PhiloxChain {
    uint32_t v0;   // round-1 out word 0: hi(M1*c) ^ k0[0]          (i < 2^32)
    uint32_t lvk;  // level ^ k1[0]
    uint32_t c2a;  // lo(M1*c) ^ k0[1]
    uint32_t c2b;  // hi(M0*v0) ^ k1[1]
    uint32_t c2lo; // lo(M0*v0)
};

PSA_HD PhiloxChain philox_chain(uint32_t chain, uint32_t level, const PhiloxKeys& key) {
    PhiloxChain pc;
    uint32_t hi1, lo1, hi0, lo0;
    mulhilo(chain, kPhiloxM1, hi1, lo1);
    pc.v0 = hi1 ^ key.k0[0];
    pc.lvk = level ^ key.k1[0];
    mulhilo(pc.v0, kPhiloxM0, hi0, lo0);
    pc.c2a = lo1 ^ key.k0[1];
    pc.c2b = hi0 ^ key.k1[1];
    pc.c2lo = lo0;
    return pc;
}

// 53-bit mantissa integer of draw `ctr` (< 2^32) of the chain's stream
PSA_HD uint64_t draw_bits53_fast(uint32_t ctr, const PhiloxChain& pc, const PhiloxKeys& key) {
    uint32_t hi, lo;
    // round 1: v = {pc.v0, lo(M1*c), hi(M0*ctr) ^ level ^ k1[0], lo(M0*ctr)}
    mulhilo(ctr, kPhiloxM0, hi, lo);
    const uint32_t r1v2 = hi ^ pc.lvk, r1v3 = lo;
    // round 2
    mulhilo(r1v2, kPhiloxM1, hi, lo);
    uint32_t v0 = hi ^ pc.c2a, v1 = lo, v2 = r1v3 ^ pc.c2b, v3 = pc.c2lo;
#pragma unroll
    for (int r = 2; r < 9; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(v0, kPhiloxM0, hi0, lo0);
        mulhilo(v2, kPhiloxM1, hi1, lo1);
        const uint32_t n0 = hi1 ^ v1 ^ key.k0[r];
        const uint32_t n2 = hi0 ^ v3 ^ key.k1[r];
        v0 = n0;
        v1 = lo1;
        v2 = n2;
        v3 = lo0;
    }
    // round 10: only out[0] and out[1] are used (rng.hpp:72-74)
    mulhilo(v2, kPhiloxM1, hi, lo);
    const uint32_t out0 = hi ^ v1 ^ key.k0[9];
    const uint32_t out1 = lo;
    return ((static_cast<uint64_t>(out1) << 32) | out0) >> 11;
}

// draw_bits53_fast with the first-round product supplied: p0 = M0 * ctr as a
// 64-bit integer (ctr < 2^32, so the product is exact).  Consecutive
// counters' products differ by M0, so a sweep can advance p0 with one
// 64-bit add instead of a multiply per draw.  Identical bits.
PSA_HD uint64_t draw_bits53_p0(uint64_t p0, const PhiloxChain& pc, const PhiloxKeys& key) {
    uint32_t hi = static_cast<uint32_t>(p0 >> 32), lo;
    const uint32_t r1v2 = hi ^ pc.lvk, r1v3 = static_cast<uint32_t>(p0);
    mulhilo(r1v2, kPhiloxM1, hi, lo);
    uint32_t v0 = hi ^ pc.c2a, v1 = lo, v2 = r1v3 ^ pc.c2b, v3 = pc.c2lo;
#pragma unroll
    for (int r = 2; r < 9; ++r) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(v0, kPhiloxM0, hi0, lo0);
        mulhilo(v2, kPhiloxM1, hi1, lo1);
        const uint32_t n0 = hi1 ^ v1 ^ key.k0[r];
        const uint32_t n2 = hi0 ^ v3 ^ key.k1[r];
        v0 = n0;
        v1 = lo1;
        v2 = n2;
        v3 = lo0;
    }
    mulhilo(v2, kPhiloxM1, hi, lo);
    const uint32_t out0 = hi ^ v1 ^ key.k0[9];
    const uint32_t out1 = lo;
    return ((static_cast<uint64_t>(out1) << 32) | out0) >> 11;
}

// rng.hpp:78-81 — d = int(u * n), clamped to n-1; u*n is one IEEE multiply.
PSA_HD int coordinate_index(double u, int n) {
    const int d = static_cast<int>(u * static_cast<double>(n));
    return d < n ? d : n - 1;
}

// float(u) for the single-precision Metropolis test (sa_core.cpp:51-53):
// rounding m to 24 bits then scaling by 2^-53 is exact, so this equals
// static_cast<float>(m * 2^-53) without a double round trip.
PSA_HD float bits_to_uniform_f32(uint64_t m) { return static_cast<float>(m) * 0x1.0p-53f; }

} // namespace psa
