// engine.cuh — device building blocks of the annealing engines.
//
//   * Cost<R, F>     : cache/energy interface over objectives.cuh families
//   * metropolis()   : sa_core.cpp:46-55
//   * sweep()        : sa_core.cpp:61-79, one chain, N trials, term-cached
//   * better()/argmin: engines.cpp:55-64 / :187-190 selection semantics
//
// Chain state layout (shared memory, structure-of-arrays): the cached value a
// of coordinate k for the thread `t` of a block of B threads lives at
// V[(k*A + a)*B + t], so the fold over k reads one 4- or 8-byte word per lane
// per step, consecutive lanes hit consecutive banks (conflict-free), and a
// proposal's scattered write V[(d*A+a)*B + t] is conflict-free too because the
// bank depends only on t.
#pragma once

#include <stdint.h>

#include "objectives.cuh"
#include "philox.cuh"
#include "engine_host.h"

namespace psa {

// ---------------------------------------------------------------------------
// Cost interface
// ---------------------------------------------------------------------------

template <class R, template <class> class F>
struct SepCost {
    using Fam = F<R>;
    static constexpr int A = Fam::kArrays;
    PSA_DEV static void cache(R x, int k, int, R* t) { Fam::term(x, k, t); }
    // fold over the column V (stride B), reference order k = 0..n-1
    PSA_DEV static R energy(const R* V, int B, int n, int) {
        R acc[A];
#pragma unroll
        for (int a = 0; a < A; ++a) acc[a] = Fam::init(a, n);
        const R* p = V;
#pragma unroll 4
        for (int k = 0; k < n; ++k) {
#pragma unroll
            for (int a = 0; a < A; ++a) acc[a] = fold<R>(Fam::op(a), acc[a], p[a * B]);
            p += A * B;
        }
        return Fam::finish(acc, n);
    }
};

template <class R>
struct ColumnX {
    const R* V;
    int B;
    PSA_DEV R operator()(int k) const { return V[k * B]; }
};

template <class R>
struct FullCost {
    static constexpr int A = 1;
    PSA_DEV static void cache(R x, int, int, R* t) { t[0] = x; }
    PSA_DEV static R energy(const R* V, int B, int n, int family) {
        const ColumnX<R> x{V, B};
        switch (family) {
        case PSA_FN_BRANIN: return Branin<R>::eval(x, n);
        case PSA_FN_DEKKERS_AARTS: return DekkersAarts<R>::eval(x, n);
        case PSA_FN_EASOM: return Easom<R>::eval(x, n);
        case PSA_FN_GOLDSTEIN_PRICE: return GoldsteinPrice<R>::eval(x, n);
        case PSA_FN_HIMMELBLAU: return Himmelblau<R>::eval(x, n);
        case PSA_FN_LEVY_MONTALVO: return LevyMontalvo<R>::eval(x, n);
        case PSA_FN_MOD_LANGERMAN: return ModLangerman<R>::eval(x, n);
        case PSA_FN_ROSENBROCK: return Rosenbrock<R>::eval(x, n);
        case PSA_FN_SIX_HUMP_CAMEL: return SixHumpCamel<R>::eval(x, n);
        case PSA_FN_SHEKEL5: return Shekel<R, 5>::eval(x, n);
        case PSA_FN_SHEKEL7: return Shekel<R, 7>::eval(x, n);
        case PSA_FN_SHEKEL10: return Shekel<R, 10>::eval(x, n);
        case PSA_FN_SHEKEL_FOXHOLES: return ShekelFoxholes<R>::eval(x, n);
        default: return R(__int_as_float(0x7fc00000));
        }
    }
};

// ---------------------------------------------------------------------------
// Metropolis rule — sa_core.cpp:46-55 (the draw is consumed by the caller)
// ---------------------------------------------------------------------------

template <class R>
struct Accept;

template <>
struct Accept<double> {
    PSA_DEV static bool test(double delta_e, double temperature, uint64_t m) {
        return bits_to_uniform(m) <= libm::exp(-delta_e / temperature);
    }
};

template <>
struct Accept<float> {
    PSA_DEV static bool test(double delta_e, double temperature, uint64_t m) {
        return bits_to_uniform_f32(m) <=
               libm::expf(-static_cast<float>(delta_e) / static_cast<float>(temperature));
    }
};

// ---------------------------------------------------------------------------
// Box description
// ---------------------------------------------------------------------------

struct Box {
    const double* lower; // shared-memory copies (n entries) when !uniform
    const double* width;
    double lo0, w0;      // the common bound when every coordinate has the same box
    bool uniform;
    PSA_DEV double lo(int d) const { return uniform ? lo0 : lower[d]; }
    PSA_DEV double wd(int d) const { return uniform ? w0 : width[d]; }
    // compute_neighbour, sa_core.cpp:40-42: lower[d] + u*width(d) (mul, then add)
    PSA_DEV double point(int d, double u) const { return lo(d) + u * wd(d); }
};

// ---------------------------------------------------------------------------
// One chain's sweep: sa_core.cpp:61-79
// ---------------------------------------------------------------------------

struct SweepStats {
    uint64_t evals;
    uint64_t draws;
};

// V: this thread's column (V = base + threadIdx.x), stride B.
// Returns the end energy; accept bits go to mask[w*mask_stride], w = j/32.
// If x != nullptr (asynchronous engine), accepted coordinates are also
// written to the double-precision point x[k*B] (stride B).
template <class R, class Cost>
PSA_DEV R sweep(R* V, int B, int n, int family, R E, double temperature, uint32_t chain,
                uint32_t level, uint64_t ctr, int N, const Box& box, const PhiloxKeys& keys,
                uint32_t* mask, size_t mask_stride, double* x, SweepStats& st) {
    constexpr int A = Cost::A;
    uint32_t word = 0;
    for (int j = 0; j < N; ++j) {
        const uint64_t m1 = draw_bits53(ctr, chain, level, keys);
        const int d = coordinate_index(bits_to_uniform(m1), n);
        const uint64_t m2 = draw_bits53(ctr + 1, chain, level, keys);
        const double xnew = box.point(d, bits_to_uniform(m2));
        R tn[A], to[A];
        Cost::cache(static_cast<R>(xnew), d, n, tn);
        R* slot = V + static_cast<size_t>(d) * A * B;
#pragma unroll
        for (int a = 0; a < A; ++a) {
            to[a] = slot[a * B];
            slot[a * B] = tn[a];
        }
        const R trial = Cost::energy(V, B, n, family);
        const double delta_e = static_cast<double>(trial) - static_cast<double>(E);
        bool acc = true;
        if (!(delta_e <= 0)) {
            const uint64_t m3 = draw_bits53(ctr + 2, chain, level, keys);
            acc = Accept<R>::test(delta_e, temperature, m3);
        }
        ctr += 3;
        if (acc) {
            E = trial;
            word |= 1u << (j & 31);
            if (x) x[static_cast<size_t>(d) * B] = xnew;
        } else {
#pragma unroll
            for (int a = 0; a < A; ++a) slot[a * B] = to[a];
        }
        if ((j & 31) == 31 || j == N - 1) {
            if (mask) mask[static_cast<size_t>(j >> 5) * mask_stride] = word;
            word = 0;
        }
    }
    st.evals += static_cast<uint64_t>(N);
    st.draws += 3ull * static_cast<uint64_t>(N);
    return E;
}

// ---------------------------------------------------------------------------
// Selection — engines.cpp:55-64, :187-190.  The serial scan
//   winner = 0; for c: if (E[c] < E[winner]) winner = c;
// is reproduced by a total order: (a) chain 0 with a NaN energy wins
// (nothing compares below NaN), (b) NaNs elsewhere never win, (c) smaller
// energy wins, (d) equal energies (including -0 == +0) go to the smaller
// chain index.  Any reduction tree over this order returns the scan's winner.
// ---------------------------------------------------------------------------

PSA_HD bool is_nan(double v) { return v != v; }

PSA_HD bool better(const Cand& a, const Cand& b) {
    if (b.c == INT32_MAX) return a.c != INT32_MAX;
    if (a.c == INT32_MAX) return false;
    const bool an = is_nan(a.e), bn = is_nan(b.e);
    if (an || bn) {
        if (an && a.c == 0) return true;
        if (bn && b.c == 0) return false;
        if (an && bn) return a.c < b.c;
        return bn;
    }
    if (a.e < b.e) return true;
    if (b.e < a.e) return false;
    return a.c < b.c;
}

PSA_DEV Cand empty_cand() { return Cand{__longlong_as_double(0x7ff0000000000000ll), INT32_MAX, -1}; }

PSA_DEV Cand shfl_cand(const Cand& v, int src_lane_xor) {
    Cand o;
    o.e = __shfl_xor_sync(0xffffffffu, v.e, src_lane_xor);
    o.c = __shfl_xor_sync(0xffffffffu, v.c, src_lane_xor);
    o.aux = __shfl_xor_sync(0xffffffffu, v.aux, src_lane_xor);
    return o;
}

PSA_DEV Cand warp_argmin(Cand v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const Cand w = shfl_cand(v, o);
        if (better(w, v)) v = w;
    }
    return v;
}

// Block-wide argmin; every thread gets the result.  `scratch` holds >= 33 Cands.
PSA_DEV Cand block_argmin(Cand v, Cand* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_argmin(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        Cand w = lane < nw ? scratch[lane] : empty_cand();
        w = warp_argmin(w);
        if (lane == 0) scratch[32] = w;
    }
    __syncthreads();
    return scratch[32];
}

} // namespace psa
