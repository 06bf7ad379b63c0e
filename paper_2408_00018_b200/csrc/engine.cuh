// engine.cuh — device building blocks of the annealing engines.
//
//   * Cost<R, F>     : cache/energy interface over objectives.cuh families
//   * metropolis()   : sa_core.cpp:46-55
//   * sweep()        : sa_core.cpp:61-79, one chain, N trials, term-cached
//   * better()/argmin: engines.cpp:55-64 / :187-190 selection semantics
//
// Chain state layout: see "Chain-state rows" below.
#pragma once

#include <stdint.h>

#include "objectives.cuh"
#include "philox.cuh"
#include "engine_host.h"

namespace psa {

// ---------------------------------------------------------------------------
// Chain-state rows
//
// Each thread owns one contiguous row of S cached values (R elements) in
// shared memory: value a of coordinate k at row[k*A + a].  S is padded so the
// row stride is 4 (mod 8) 32-bit words: a warp's 16-byte loads of the same
// offset then fall into distinct bank quads (conflict-free LDS.128), and the
// fold addresses every element with an immediate offset from one base
// register.  16 bytes carry 4 f32 or 2 f64 terms.
// ---------------------------------------------------------------------------

template <class R>
PSA_HD int row_stride(int n, int A) {
    int words = n * A * static_cast<int>(sizeof(R) / 4);
    words = (words + 3) & ~3;         // whole 16-byte vectors
    if ((words & 7) == 0) words += 4; // stride = 4 (mod 8) words
    return words / static_cast<int>(sizeof(R) / 4);
}

template <class R>
struct Vec16;
template <>
struct Vec16<float> {
    using T = float4;
    static constexpr int W = 4;
    PSA_DEV static float get(const float4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
};
template <>
struct Vec16<double> {
    using T = double2;
    static constexpr int W = 2;
    PSA_DEV static double get(const double2& v, int i) { return i == 0 ? v.x : v.y; }
};

// Large-n layout: when a thread's row does not fit in shared memory the rows
// live in HBM as warp tiles of 16-byte vectors: value i of lane l of warp w
// at base[((w * nv + i / W) * 32 + l) * W + i % W] (W = 4 f32 / 2 f64 values
// per vector, nv vectors per row).  A warp's fold loads of one vector are a
// single coalesced 512-byte LDG.128, and successive vectors are adjacent, so
// the fold streams one contiguous tile (no TLB thrashing across a
// thread-strided layout); p = the lane's first value, s = 32 * W.
template <class R>
struct StridedRow {
    static constexpr int W = 16 / static_cast<int>(sizeof(R));
    R* p;
    size_t s;
    PSA_DEV R& operator[](int i) const { return p[static_cast<size_t>(i / W) * s + (i % W)]; }
};

template <class T>
struct IsStrided {
    static constexpr bool value = false;
};
template <class R>
struct IsStrided<StridedRow<R>> {
    static constexpr bool value = true;
};

// ---------------------------------------------------------------------------
// Cost interface
// ---------------------------------------------------------------------------

template <class F, class = void>
struct HasCommon {
    static constexpr bool value = false;
};
template <class F>
struct HasCommon<F, decltype(void(F::kHasCommon))> {
    static constexpr bool value = F::kHasCommon;
};

template <class R, template <class> class F>
struct SepCost {
    using Fam = F<R>;
    static constexpr int A = Fam::kArrays;
    static_assert(Vec16<R>::W % A == 0, "array count must divide the vector width");
    PSA_DEV static void cache(R x, int k, int, R* t) { Fam::term(x, k, t); }
    // branch-free cache for the hot loop when the family provides one
    PSA_DEV static void cache_common(R x, int k, int n, R* t, bool& ok) {
        if constexpr (HasCommon<Fam>::value) {
            Fam::term_common(x, k, t, ok);
        } else {
            cache(x, k, n, t);
            ok = true;
        }
    }
    // fold over a 16-byte aligned row, reference order k = 0..n-1 per array.
    // NT > 0: the dimension is a compile-time constant and the fold is one
    // straight-line block (no loop), so the scheduler can interleave the
    // next trial's independent Philox work into the FADD dependency chain.
    template <int NT = 0>
    PSA_DEV static R energy(const R* row, int n_rt, int family) {
        const int n = NT > 0 ? NT : n_rt;
        R acc[A];
        fold_acc<NT>(row, n, acc);
        (void)family;
        return Fam::finish(acc, n);
    }
    // the accumulators of the fold, before finish()
    template <int NT = 0>
    PSA_DEV static void fold_acc(const R* row, int n_rt, R* acc) {
        using V = Vec16<R>;
        const int n = NT > 0 ? NT : n_rt;
#pragma unroll
        for (int a = 0; a < A; ++a) acc[a] = Fam::init(a, n);
        const int m = n * A;
        const int mv = m / V::W;
        const typename V::T* p = reinterpret_cast<const typename V::T*>(row);
        if constexpr (NT > 0) {
            constexpr int NV = (NT * A) / V::W;
#ifndef PSA_FOLD_PREFETCH
#define PSA_FOLD_PREFETCH 4
#endif
#if PSA_FOLD_PREFETCH > 0
            // loads run PSA_FOLD_PREFETCH vectors ahead of the FADD chain so
            // the shared-memory latency stays hidden behind it
            constexpr int PF = PSA_FOLD_PREFETCH < NV ? PSA_FOLD_PREFETCH : NV;
            typename V::T buf[PF];
#pragma unroll
            for (int q = 0; q < PF; ++q) buf[q] = p[q];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const typename V::T v = buf[q % PF];
                if (q + PF < NV) buf[q % PF] = p[q + PF];
#pragma unroll
                for (int i = 0; i < V::W; ++i) acc[i % A] = fold<R>(Fam::op(i % A), acc[i % A], V::get(v, i));
            }
#else
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const typename V::T v = p[q];
#pragma unroll
                for (int i = 0; i < V::W; ++i) acc[i % A] = fold<R>(Fam::op(i % A), acc[i % A], V::get(v, i));
            }
#endif
#pragma unroll
            for (int e = ((NT * A) / V::W) * V::W; e < NT * A; ++e)
                acc[e % A] = fold<R>(Fam::op(e % A), acc[e % A], row[e]);
        } else {
#pragma unroll 5
            for (int q = 0; q < mv; ++q) {
                const typename V::T v = p[q];
#pragma unroll
                for (int i = 0; i < V::W; ++i) acc[i % A] = fold<R>(Fam::op(i % A), acc[i % A], V::get(v, i));
            }
            for (int e = mv * V::W; e < m; ++e) acc[e % A] = fold<R>(Fam::op(e % A), acc[e % A], row[e]);
        }
    }
    // the HBM layout (StridedRow): 16-byte vector loads, issued 8 at a time
    // so that 128 B per thread are in flight; same fold order
    template <class Row>
    PSA_DEV static R energy_any(const Row& row, int n, int) {
        using V = Vec16<R>;
        R acc[A];
#pragma unroll
        for (int a = 0; a < A; ++a) acc[a] = Fam::init(a, n);
        const int m = n * A;
        const int full = m / V::W; // whole vectors
        auto ld = [&](int q) { return *reinterpret_cast<const typename V::T*>(row.p + static_cast<size_t>(q) * row.s); };
        auto fold_vec = [&](const typename V::T& v) {
#pragma unroll
            for (int w = 0; w < V::W; ++w) acc[w % A] = fold<R>(Fam::op(w % A), acc[w % A], V::get(v, w));
        };
        int q = 0;
        for (; q + 8 <= full; q += 8) {
            typename V::T v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = ld(q + i);
#pragma unroll
            for (int i = 0; i < 8; ++i) fold_vec(v[i]);
        }
        for (; q < full; ++q) fold_vec(ld(q));
        if (m % V::W) { // (W is a multiple of A, so element e = full*W + w has array w % A)
            const typename V::T v = ld(full);
            for (int w = 0; w < m % V::W; ++w) acc[w % A] = fold<R>(Fam::op(w % A), acc[w % A], V::get(v, w));
        }
        return Fam::finish(acc, n);
    }
};

template <class R, class Row = const R*>
struct RowX {
    Row row;
    PSA_DEV R operator()(int k) const { return row[k]; }
};

// PSA_FN_CONSTANT: f = c, a per-objective parameter (the constant fixtures of
// test_engines.cpp:91-99 and test_sa_core.cpp:140-160).  Every kernel that
// can evaluate FullCost copies c from its arguments into this block-shared
// slot before its first evaluation (fn_param_init).
static __shared__ double psa_fn_param_s;

template <class R>
struct FullCost {
    static constexpr int A = 1;
    PSA_DEV static void cache(R x, int, int, R* t) { t[0] = x; }
    PSA_DEV static void cache_common(R x, int k, int n, R* t, bool& ok) {
        cache(x, k, n, t);
        ok = true;
    }
    template <int NT = 0>
    PSA_DEV static R energy(const R* row, int n, int family) {
        return energy_any(row, n, family);
    }
    template <class Row>
    PSA_DEV static R energy_any(const Row& row, int n, int family) {
        const RowX<R, Row> x{row};
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
        case PSA_FN_CONSTANT: return static_cast<R>(psa_fn_param_s);
        default: return R(__int_as_float(0x7fc00000));
        }
    }
};

template <class Cost>
struct IsFullCost {
    static constexpr bool value = false;
};
template <class R>
struct IsFullCost<FullCost<R>> {
    static constexpr bool value = true;
};

// block-wide: the family parameter into psa_fn_param_s (FullCost kernels)
template <class Cost>
PSA_DEV void fn_param_init(double c) {
    if constexpr (IsFullCost<Cost>::value) {
        if (threadIdx.x == 0) psa_fn_param_s = c;
        __syncthreads();
    }
}

// energy of a chain row of either layout
template <class Cost, int NT, class Row>
PSA_DEV auto row_energy(const Row& row, int n, int family) {
    if constexpr (IsStrided<Row>::value) return Cost::energy_any(row, n, family);
    else return Cost::template energy<NT>(row, n, family);
}

// ---------------------------------------------------------------------------
// Metropolis rule — sa_core.cpp:46-55 (the draw is consumed by the caller)
// ---------------------------------------------------------------------------

template <class R>
struct Accept;

// exact reference tests (sa_core.cpp:52-54)
template <>
struct Accept<double> {
    PSA_DEV static bool exact(double delta_e, double temperature, uint64_t m) {
        return bits_to_uniform(m) <= libm::exp(-delta_e / temperature);
    }
};

template <>
struct Accept<float> {
    PSA_DEV static bool exact(double delta_e, double temperature, uint64_t m) {
        return bits_to_uniform_f32(m) <=
               libm::expf(-static_cast<float>(delta_e) / static_cast<float>(temperature));
    }
};

// log2(x), MUFU.LG2 (absolute error below 2^-22 for normal x; 0 -> -inf)
PSA_DEV float lg2_approx(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// The Metropolis decision (sa_core.cpp:46-55) with a branch-free pre-test in
// the log domain; returns 1 accept, 0 reject, -1 undecided.
//  * d = trial - E in R has the sign of the reference's double difference
//    (subtracting two floats never flips the sign, is zero only for equal
//    values, and is NaN exactly when the double one is; for R = double it
//    is the reference's own difference), so d <= 0 is the downhill test.
//  * uphill, the reference accepts iff u <= exp(-dE/T), i.e. iff
//    x = dE*log2(e)/T <= L = -log2(u).  The device forms x = float(d)*k2
//    (k2 = log2(e)/T rounded to a normal float: relative error below 2^-22
//    in all) and, from the acceptance draw alone, the band [lo, hi] =
//    [L - 2^-13, L + 2^-13] with L = 53 - lg2.approx(float(m)) (MUFU.LG2's
//    error, 2^-22 absolute, or even relative to |log2| <= 53, plus float(m)'s
//    rounding stay below 2^-16 for u = m*2^-53, m >= 1; L <= 53).  x < lo accepts and
//    x > hi rejects with certainty: the errors of x (|x| * 2^-22 < 2^-15 for
//    |x| <= 60; a larger x is far beyond hi), of L, and of the reference's own
//    exp / expf rounding and float(u) (relative 2^-23 each, below 2^-22 in
//    the log domain) add up to about 2^-15, inside the 2^-13 margin (the
//    margin was 2^-10 in round 1; every undecided draw costs the exact test,
//    and in the deferred-fold sweep two folds, so it is as small as the error
//    budget allows — psa_device_metropolis_check counts disagreements with
//    the exact test on draws placed at the boundary).  m == 0, NaNs, a
//    k2 outside the normal floats and the band itself report undecided and
//    the caller runs the exact glibc-restated test.
//  * The band depends only on the draw, which the counter-based streams give
//    ahead of the trial, so only an FADD, an FMUL and two compares follow the
//    fold on the chain's critical path.
struct MBand {
    float lo, hi;
};

PSA_DEV MBand metropolis_band(uint64_t m) {
    const float l = lg2_approx(__ull2float_rn(m));
    const float nan = __int_as_float(0x7fffffff);
    return MBand{m ? 0x1.a7ffcp+5f - l : nan, m ? 0x1.a8004p+5f - l : nan}; // 53 -/+ 2^-13
}

// log2(e) / T as the pre-test's factor; NaN (always undecided) unless normal
PSA_DEV float metropolis_k2(double temperature) {
    const float k2 = static_cast<float>(1.4426950408889634 / temperature);
    return (k2 >= 0x1.0p-126f && k2 <= 0x1.0p+126f) ? k2 : __int_as_float(0x7fffffff);
}

template <class R>
PSA_DEV int metropolis_fast(R trial, R E, float k2, MBand b) {
    const R d = trial - E;
    const float x = static_cast<float>(d) * k2;
    const bool acc = (d <= R(0)) | (x < b.lo);
    const bool rej = x > b.hi;
    return acc ? 1 : (rej ? 0 : -1);
}

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
    // UB: the box is known to be uniform at compile time (no per-coordinate
    // bound loads in the hot loop)
    template <bool UB>
    PSA_DEV double point_t(int d, double u) const { return UB ? lo0 + u * w0 : point(d, u); }
};

// ---------------------------------------------------------------------------
// One chain's sweep: sa_core.cpp:61-79
// ---------------------------------------------------------------------------

struct SweepStats {
    uint64_t evals;
    uint64_t draws;
    uint64_t settles = 0; // deferred fold: decisions settled by exact folds
};

// row: this thread's 16-byte aligned shared-memory state row (Row = R*), or
// its HBM structure-of-arrays row (Row = StridedRow<R>).  Returns the end
// energy; accept bits go to mask[w*mask_stride], w = j/32.  If x != nullptr
// (asynchronous engine), accepted coordinates are also written to the
// double-precision point of this chain, x[k * x_stride].
//
// The three draws of trial j+1 do not depend on trial j's outcome (the
// streams are counter-based), so they are issued before the fold of trial j
// and overlap its dependent FADD chain; the acceptance draw is therefore
// computed even for downhill moves (it is consumed either way, rng.hpp).
template <class R, class Cost, int NT = 0, class Row = R*>
PSA_DEV R sweep(Row row, int n_rt, int family, R E, double temperature, uint32_t chain,
                uint32_t level, uint32_t ctr, int N, const Box& box, const PhiloxKeys& keys,
                uint32_t* mask, size_t mask_stride, double* x, size_t x_stride, SweepStats& st) {
    constexpr int A = Cost::A;
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature); // log2(e) / T
    const PhiloxChain pc = philox_chain(chain, level, keys);
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53; // u*n == m*(n*2^-53) exactly
    // Two-stage software pipeline over the trials (the streams are counter-
    // based, so every draw is known in advance).  While trial j's fold and
    // decision run, the same iteration builds trial j+1's new term from
    // draws made one iteration earlier and makes trial j+2's three draws:
    // three independent dependency chains the scheduler interleaves, instead
    // of one long Philox -> index -> sinf chain per trial.  Trials run in
    // words of 32 (one accept-mask word each).
    int d;          // trial j: coordinate, value, new cached term, acceptance draw
    double xnew;
    R tn[A];
    uint64_t m3;
    uint64_t q1, q2, q3; // trial j+1's draws
    {
        const uint64_t m1 = draw_bits53_fast(ctr, pc, keys);
        const uint64_t m2 = draw_bits53_fast(ctr + 1, pc, keys);
        m3 = draw_bits53_fast(ctr + 2, pc, keys);
        d = min(static_cast<int>(static_cast<double>(m1) * idx_scale), n - 1);
        xnew = box.point(d, bits_to_uniform(m2));
        Cost::cache(static_cast<R>(xnew), d, n, tn);
        q1 = draw_bits53_fast(ctr + 3, pc, keys);
        q2 = draw_bits53_fast(ctr + 4, pc, keys);
        q3 = draw_bits53_fast(ctr + 5, pc, keys);
    }
    for (int j0 = 0; j0 < N; j0 += 32) {
    const int jn = N - j0 < 32 ? N - j0 : 32;
    uint32_t word = 0;
    for (int j = 0; j < jn; ++j) {
        R to[A];
#pragma unroll
        for (int a = 0; a < A; ++a) {
            to[a] = row[d * A + a];
            row[d * A + a] = tn[a];
        }
        // trial j+1's proposal from its draws, trial j+2's draws
        const int dn = min(static_cast<int>(static_cast<double>(q1) * idx_scale), n - 1);
        const double xn = box.point(dn, bits_to_uniform(q2));
        R tnn[A];
        bool ok;
        Cost::cache_common(static_cast<R>(xn), dn, n, tnn, ok);
        const uint64_t r1 = draw_bits53_fast(ctr + 6, pc, keys);
        const uint64_t r2 = draw_bits53_fast(ctr + 7, pc, keys);
        const uint64_t r3 = draw_bits53_fast(ctr + 8, pc, keys);
        const MBand b3 = metropolis_band(m3);
#ifndef PSA_NO_PIN
        // materialise them here so the scheduler interleaves them into the
        // fold's FADD latency chain (left alone, the compiler sinks them)
        asm volatile("" ::"l"(r1), "l"(r2), "l"(r3), "r"(dn), "f"(b3.lo), "f"(b3.hi));
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if constexpr (sizeof(R) == 4) asm volatile("" ::"f"(tnn[a]));
            else asm volatile("" ::"d"(tnn[a]));
        }
#endif
        const R trial = row_energy<Cost, NT>(row, n, family);
        // rare paths behind warp-uniform branches
        if (__any_sync(__activemask(), !ok))
            if (!ok) Cost::cache(static_cast<R>(xn), dn, n, tnn); // general path, practically never

        // sa_core.cpp:46-55 (the acceptance draw is consumed either way)
        int r = metropolis_fast<R>(trial, E, k2, b3);
        if (__any_sync(__activemask(), r < 0))
            if (r < 0) r = Accept<R>::exact(static_cast<double>(trial) - static_cast<double>(E), temperature, m3);
        const bool acc = r != 0;
        ctr += 3;
        if (acc) {
            E = trial;
            word |= 1u << j;
            if (x) x[static_cast<size_t>(d) * x_stride] = xnew;
        } else {
#pragma unroll
            for (int a = 0; a < A; ++a) row[d * A + a] = to[a];
        }
        d = dn;
        xnew = xn;
        m3 = q3;
        q1 = r1;
        q2 = r2;
        q3 = r3;
#pragma unroll
        for (int a = 0; a < A; ++a) tn[a] = tnn[a];
    }
    if (mask) mask[static_cast<size_t>(j0 >> 5) * mask_stride] = word;
    }
    st.evals += static_cast<uint64_t>(N);
    st.draws += 3ull * static_cast<uint64_t>(N);
    return E;
}

// ---------------------------------------------------------------------------
// Deferred fold: Metropolis decisions from an energy interval
//
// For the affine families of objectives.cuh (LazyOf: E = finish(s), s one
// additive fold of the cached terms, finish(s) = alpha*s up to fin_round
// roundings) a trial's exact energy matters only when its decision depends
// on the last bits.  Let S(X) = init + sigma * sum_k t_k be the exact real
// sum of a state's terms.  The energy the reference computes — the fold in
// index order in R, then finish — satisfies |E(X) - alpha S(X)| <= rE for
// every state of the box (lazy_radius, host):
//   * each of the n fold adds rounds by at most u|partial|, and |partial_k|
//     <= |init| + sum_{j<=k} Tmax_j (Tmax_k bounds |t_k| over the box,
//     LazyOf::term_bound), so the fold is within u(1+2nu)(n|init| +
//     sum_k (n-k) Tmax_k) of S;
//   * finish rounds fin_round times (u relative to the largest |E|).
// A trial changes one term, so S(trial) - S(old) = sigma (t' - t_d) exactly,
// and the reference's difference d = E(trial) - E(old) lies within
//   q +- rr,   q = alpha * sigma * (t' - t_d)  (computed in R),
// rr = 2 rE plus the rounding of q and of the interval ends (host margin).
// No running sum is kept: the interval comes from the two cached terms.
// The decision of sa_core.cpp:46-55 is certain when hi = q + rr <= 0 or
// x(hi) < band.lo (accept: every d of the interval accepts, and x is
// monotone in d) or when lo = q - rr > 0 and x(lo) > band.hi (reject) — the
// log-domain band of metropolis_fast, whose 2^-13 margin already covers the
// rounding of x.  Otherwise (a warp-uniform rare branch) the old state and
// the trial are folded exactly and metropolis_fast / Accept::exact decide as
// in sweep().  Decisions are therefore the reference's; the energies that
// leave the sweep (the end energy, every energy compared in a settled
// decision) are exact folds.  An accepted move writes its term to the row,
// a rejected one touches nothing.  NaN or inf anywhere makes every
// comparison false, i.e. the exact path.
// ---------------------------------------------------------------------------

// the half-width rr of the interval of d (host)
template <class R, template <class> class F>
double lazy_radius(int n, const double* lower, const double* upper) {
    using Fam = F<R>;
    using L = LazyOf<Fam>;
    const double u = sizeof(R) == 4 ? 0x1.0p-24 : 0x1.0p-53;
    const double init = fabs(static_cast<double>(Fam::init(0, n)));
    double tsum = 0, wmax = 0, tmax = 0;
    for (int k = 0; k < n; ++k) {
        const double t = L::term_bound(lower[k], upper[k]) * (1.0 + 0x1.0p-16);
        tsum += t;
        wmax += static_cast<double>(n - k) * t;
        tmax = fmax(tmax, t);
    }
    const double a = fabs(L::alpha(n));
    const double fold = u * (1.0 + 2.0 * n * u) * (static_cast<double>(n) * init + wmax);
    const double cmax = a * (init + tsum);                   // bounds |E|
    const double rE = a * fold + L::fin_round * u * cmax;    // |E - alpha S|
    const double margin = 32.0 * u * a * tmax + 4.0 * u * cmax; // q, alpha, hi/lo roundings
    return (2.0 * rE + margin) * 1.01;
}

#ifndef PSA_LAZY_UNROLL
#define PSA_LAZY_UNROLL 2 // measured: 2 > 1 (+2%, no rotation moves) > 4 at low T
#endif
constexpr int kLazyUnroll = PSA_LAZY_UNROLL;
constexpr unsigned kFullWarp = 0xffffffffu;

// sweep_lazy is called by all 32 lanes of a warp together (the caller runs
// idle lanes on a duplicate chain with mask == nullptr and a scratch
// SweepStats), so its votes take the full mask: no divergence checks.

template <class R, class Cost, int NT = 0, class Row = R*, bool UB = false>
PSA_DEV R sweep_lazy(Row row, int n_rt, int family, R E, double temperature, uint32_t chain, uint32_t level,
                     uint32_t ctr, int N, const Box& box, const PhiloxKeys& keys, uint32_t* mask,
                     size_t mask_stride, double* x, size_t x_stride, SweepStats& st, R rr, R alpha) {
    using L = LazyOf<typename Cost::Fam>;
    static_assert(Cost::A == 1, "deferred fold: one accumulator");
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature);
    const PhiloxChain pc = philox_chain(chain, level, keys);
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    const R sa = L::sigma > 0 ? alpha : -alpha;
    bool have = true; // E is the exact energy of the row
    int d;
    double xnew;
    R tn[1];
    uint64_t m3;
    uint64_t q1, q2, q3;
    {
        const uint64_t m1 = draw_bits53_fast(ctr, pc, keys);
        const uint64_t m2 = draw_bits53_fast(ctr + 1, pc, keys);
        m3 = draw_bits53_fast(ctr + 2, pc, keys);
        d = min(static_cast<int>(static_cast<double>(m1) * idx_scale), n - 1);
        xnew = box.point_t<UB>(d, bits_to_uniform(m2));
        Cost::cache(static_cast<R>(xnew), d, n, tn);
        q1 = draw_bits53_fast(ctr + 3, pc, keys);
        q2 = draw_bits53_fast(ctr + 4, pc, keys);
        q3 = draw_bits53_fast(ctr + 5, pc, keys);
    }
#ifndef PSA_P0_MUL
    uint64_t p6 = static_cast<uint64_t>(kPhiloxM0) * (ctr + 6); // M0 * (counter of the next draw batch)
#endif
    // the cached term a trial replaces is loaded one trial ahead (HBM rows:
    // the load latency overlaps the previous trial)
    R to = row[d];
    for (int j0 = 0; j0 < N; j0 += 32) {
        const int jn = N - j0 < 32 ? N - j0 : 32;
        uint32_t word = 0;
#pragma unroll kLazyUnroll
        for (int j = 0; j < jn; ++j) {
            const int dn = min(static_cast<int>(static_cast<double>(q1) * idx_scale), n - 1);
            const R tp = row[dn]; // next trial's replaced term (fixed up below if this trial writes dn)
            const double xn = box.point_t<UB>(dn, bits_to_uniform(q2));
            R tnn[1];
            bool ok;
            Cost::cache_common(static_cast<R>(xn), dn, n, tnn, ok);
#ifndef PSA_P0_MUL
            // first-round products by addition (draw_bits53_p0)
            const uint64_t r1 = draw_bits53_p0(p6, pc, keys);
            const uint64_t r2 = draw_bits53_p0(p6 + kPhiloxM0, pc, keys);
            const uint64_t r3 = draw_bits53_p0(p6 + 2ull * kPhiloxM0, pc, keys);
            p6 += 3ull * kPhiloxM0;
#else
            const uint64_t r1 = draw_bits53_fast(ctr + 6, pc, keys);
            const uint64_t r2 = draw_bits53_fast(ctr + 7, pc, keys);
            const uint64_t r3 = draw_bits53_fast(ctr + 8, pc, keys);
#endif
            const MBand b3 = metropolis_band(m3);
            // the interval decision
            const R q = (tn[0] - to) * sa;
            const R hi = q + rr, lo = q - rr;
            const float xh = static_cast<float>(hi) * k2, xl = static_cast<float>(lo) * k2;
            int r = ((hi <= R(0)) | (xh < b3.lo)) ? 1 : (((lo > R(0)) & (xl > b3.hi)) ? 0 : -1);
            bool settled = false;
            // one warp vote on the common path for both rare cases
            if (__any_sync(kFullWarp, (!ok) | (r < 0))) {
                if (!ok) Cost::cache(static_cast<R>(xn), dn, n, tnn); // general term path
            if (__any_sync(kFullWarp, r < 0)) {
                // rare: fold exactly (the whole warp folds; every lane whose
                // energy is stale takes the exact old value for free)
                if (__any_sync(kFullWarp, (r < 0) & !have)) {
                    const R eo = row_energy<Cost, NT>(row, n, family);
                    if (!have) {
                        E = eo;
                        have = true;
                    }
                }
                if (r < 0) row[d] = tn[0];
                const R et = row_energy<Cost, NT>(row, n, family);
                if (r < 0) {
                    int v = metropolis_fast<R>(et, E, k2, b3);
                    if (v < 0) v = Accept<R>::exact(static_cast<double>(et) - static_cast<double>(E), temperature, m3);
                    if (v) E = et;
                    else row[d] = to;
                    r = v;
                    settled = true;
                    st.settles += 1;
                }
            }
            }
            if (r && !settled) {
                row[d] = tn[0];
                have = false;
            }
            ctr += 3;
            word |= static_cast<uint32_t>(r) << j; // r is 0 or 1 here
            if (r) {
                if (x) x[static_cast<size_t>(d) * x_stride] = xnew;
            }
            to = (r && dn == d) ? tn[0] : tp;
            d = dn;
            xnew = xn;
            m3 = q3;
            q1 = r1;
            q2 = r2;
            q3 = r3;
            tn[0] = tnn[0];
        }
        if (mask) mask[static_cast<size_t>(j0 >> 5) * mask_stride] = word;
    }
    // the end energy is the exact fold
    if (__any_sync(kFullWarp, !have)) {
        const R e = row_energy<Cost, NT>(row, n, family);
        if (!have) E = e;
    }
    st.evals += static_cast<uint64_t>(N);
    st.draws += 3ull * static_cast<uint64_t>(N);
    return E;
}

// ---------------------------------------------------------------------------
// Chain pairs: two chains per thread, folded with packed FP32x2 adds
//
// sm_100 issues FADD2/FMUL2 (PTX add/sub/mul.rn.f32x2): two IEEE binary32
// operations, each rounded exactly like FADD/FMUL, in one instruction.  The
// term fold is a serial chain per chain, so it cannot be split; but two
// independent chains (A, B) folded side by side halve the instructions of
// the fold, which is a third of the trial's issue budget.  Pair rows
// interleave the chains: element e = k*A + a holds (t_e of A, t_e of B) as
// one 8-byte word, so a 16-byte LDS feeds two FADD2.
// ---------------------------------------------------------------------------

struct F2 {
    unsigned long long v;
};

PSA_DEV F2 f2_make(float lo, float hi) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
PSA_DEV void f2_split(F2 x, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x.v)); }

// the fold step of objectives.cuh (kAdd / kSub / kMul), on both lanes
PSA_DEV F2 f2_fold(int op, F2 acc, F2 t) {
    F2 r;
    if (op == kAdd) asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(acc.v), "l"(t.v));
    else if (op == kSub) asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(acc.v), "l"(t.v));
    else asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(acc.v), "l"(t.v));
    return r;
}

// energies of both chains of a pair row (n*A interleaved elements)
template <class Fam, int NT>
PSA_DEV void pair_energy(const float* row, int n_rt, float& eA, float& eB) {
    constexpr int A = Fam::kArrays;
    const int n = NT > 0 ? NT : n_rt;
    const unsigned long long* u = reinterpret_cast<const unsigned long long*>(row);
    F2 acc[A];
#pragma unroll
    for (int a = 0; a < A; ++a) {
        const float i0 = Fam::init(a, n);
        acc[a] = f2_make(i0, i0);
    }
    if constexpr (NT > 0) {
        constexpr int M = NT * A;     // elements
        constexpr int NV = M / 2;     // 16-byte vectors
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(u);
        constexpr int PF = 4 < NV ? 4 : NV; // vectors loaded ahead of the FADD2 chain
        ulonglong2 buf[PF > 0 ? PF : 1];
#pragma unroll
        for (int q = 0; q < PF; ++q) buf[q] = p[q];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const ulonglong2 v = buf[q % PF];
            if (q + PF < NV) buf[q % PF] = p[q + PF];
            acc[(2 * q) % A] = f2_fold(Fam::op((2 * q) % A), acc[(2 * q) % A], F2{v.x});
            acc[(2 * q + 1) % A] = f2_fold(Fam::op((2 * q + 1) % A), acc[(2 * q + 1) % A], F2{v.y});
        }
        if constexpr (M % 2) acc[(M - 1) % A] = f2_fold(Fam::op((M - 1) % A), acc[(M - 1) % A], F2{u[M - 1]});
    } else {
        const int M = n * A;
#pragma unroll 4
        for (int e = 0; e < M; ++e) acc[e % A] = f2_fold(Fam::op(e % A), acc[e % A], F2{u[e]});
    }
    float ra[A], rb[A];
#pragma unroll
    for (int a = 0; a < A; ++a) f2_split(acc[a], ra[a], rb[a]);
    eA = Fam::finish(ra, n);
    eB = Fam::finish(rb, n);
}


// One level of N trials for the chain pair (cA, cB) of a pair row: the
// sweep() of sa_core.cpp:61-79 for two chains at once.  Each chain's draws,
// proposals, energies and decisions are exactly those of sweep(); only the
// fold is shared (FADD2).  Accept bits go to maskA/maskB[w * mask_stride].
// (V1, kX = true: no masks; the chains' double-precision points xa/xb are
// updated by accepted moves, x[k * xs].)  Trials run in words of 32, one
// accept-mask word each.
template <template <class> class F, int NT, bool kX = false>
PSA_DEV void sweep_pair(float* row, int n_rt, float& EA, float& EB, double temperature, uint32_t cA,
                        uint32_t cB, uint32_t level, uint32_t ctr, int N, const Box& box, const PhiloxKeys& keys,
                        uint32_t* maskA, uint32_t* maskB, size_t mask_stride, double* xa = nullptr,
                        double* xb = nullptr, size_t xs = 0) {
    using Fam = F<float>;
    using Cost = SepCost<float, F>;
    constexpr int A = Fam::kArrays;
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature); // log2(e) / T
    const PhiloxChain pa = philox_chain(cA, level, keys);
    const PhiloxChain pb = philox_chain(cB, level, keys);
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    int dA, dB;
    double xA, xB;
    float tA[A], tB[A];
    {
        const uint64_t a1 = draw_bits53_fast(ctr, pa, keys), a2 = draw_bits53_fast(ctr + 1, pa, keys);
        const uint64_t b1 = draw_bits53_fast(ctr, pb, keys), b2 = draw_bits53_fast(ctr + 1, pb, keys);
        dA = min(static_cast<int>(static_cast<double>(a1) * idx_scale), n - 1);
        dB = min(static_cast<int>(static_cast<double>(b1) * idx_scale), n - 1);
        xA = box.point(dA, bits_to_uniform(a2));
        xB = box.point(dB, bits_to_uniform(b2));
        Cost::cache(static_cast<float>(xA), dA, n, tA);
        Cost::cache(static_cast<float>(xB), dB, n, tB);
    }
    for (int j0 = 0; j0 < N; j0 += 32) {
    const int jn = N - j0 < 32 ? N - j0 : 32;
    uint32_t wordA = 0, wordB = 0;
    for (int j = 0; j < jn; ++j) {
        float oA[A], oB[A];
#pragma unroll
        for (int a = 0; a < A; ++a) {
            float* sa = row + 2 * (dA * A + a);
            float* sb = row + 2 * (dB * A + a) + 1;
            oA[a] = *sa;
            *sa = tA[a];
            oB[a] = *sb;
            *sb = tB[a];
        }
        // independent of this trial's outcome: its acceptance draws and the
        // next proposals (counter-based streams)
        const uint64_t mA = draw_bits53_fast(ctr + 2, pa, keys);
        const uint64_t mB = draw_bits53_fast(ctr + 2, pb, keys);
        const uint64_t a1 = draw_bits53_fast(ctr + 3, pa, keys), a2 = draw_bits53_fast(ctr + 4, pa, keys);
        const uint64_t b1 = draw_bits53_fast(ctr + 3, pb, keys), b2 = draw_bits53_fast(ctr + 4, pb, keys);
        const int nA = min(static_cast<int>(static_cast<double>(a1) * idx_scale), n - 1);
        const int nB = min(static_cast<int>(static_cast<double>(b1) * idx_scale), n - 1);
        const double yA = box.point(nA, bits_to_uniform(a2));
        const double yB = box.point(nB, bits_to_uniform(b2));
        float uA[A], uB[A];
        bool okA, okB;
        Cost::cache_common(static_cast<float>(yA), nA, n, uA, okA);
        Cost::cache_common(static_cast<float>(yB), nB, n, uB, okB);
        const MBand bA = metropolis_band(mA), bB = metropolis_band(mB);
        asm volatile("" ::"f"(bA.lo), "f"(bA.hi), "f"(bB.lo), "f"(bB.hi), "r"(nA), "r"(nB));
#pragma unroll
        for (int a = 0; a < A; ++a) asm volatile("" ::"f"(uA[a]), "f"(uB[a]));

        float trA, trB;
        pair_energy<Fam, NT>(row, n, trA, trB);
        // rare paths behind warp-uniform branches (no reconvergence barrier
        // on the common path)
        if (__any_sync(__activemask(), !(okA & okB))) {
            if (!okA) Cost::cache(static_cast<float>(yA), nA, n, uA);
            if (!okB) Cost::cache(static_cast<float>(yB), nB, n, uB);
        }
        int rA = metropolis_fast<float>(trA, EA, k2, bA);
        int rB = metropolis_fast<float>(trB, EB, k2, bB);
        if (__any_sync(__activemask(), (rA < 0) | (rB < 0))) {
            if (rA < 0) rA = Accept<float>::exact(static_cast<double>(trA) - static_cast<double>(EA), temperature, mA);
            if (rB < 0) rB = Accept<float>::exact(static_cast<double>(trB) - static_cast<double>(EB), temperature, mB);
        }
        ctr += 3;
        EA = rA ? trA : EA;
        EB = rB ? trB : EB;
        wordA |= static_cast<uint32_t>(rA) << j;
        wordB |= static_cast<uint32_t>(rB) << j;
        if constexpr (kX) {
            if (rA) xa[static_cast<size_t>(dA) * xs] = xA;
            if (rB) xb[static_cast<size_t>(dB) * xs] = xB;
        }
#pragma unroll
        for (int a = 0; a < A; ++a) {
            if (!rA) row[2 * (dA * A + a)] = oA[a];
            if (!rB) row[2 * (dB * A + a) + 1] = oB[a];
        }
        dA = nA;
        dB = nB;
        xA = yA;
        xB = yB;
#pragma unroll
        for (int a = 0; a < A; ++a) {
            tA[a] = uA[a];
            tB[a] = uB[a];
        }
    }
    if constexpr (!kX) {
        maskA[static_cast<size_t>(j0 >> 5) * mask_stride] = wordA;
        maskB[static_cast<size_t>(j0 >> 5) * mask_stride] = wordB;
    }
    }
}

// Deferred fold for a chain pair (binary32 affine families): sweep_lazy's
// interval decisions for two chains per thread, on a pair row (element k =
// (t_k of A, t_k of B)), so the rare exact folds of both chains are one
// FADD2 fold (pair_energy) and the loop, constants and mask words are shared
// by two chains.  Called by all 32 lanes of a warp together.
template <template <class> class F, int NT>
PSA_DEV void sweep_lazy_pair(float* row, int n_rt, float& EA, float& EB, double temperature, uint32_t cA,
                             uint32_t cB, uint32_t level, uint32_t ctr, int N, const Box& box,
                             const PhiloxKeys& keys, uint32_t* maskA, uint32_t* maskB, size_t mask_stride,
                             SweepStats& st, float rr, float alpha, bool cntA, bool cntB) {
    using Fam = F<float>;
    using Cost = SepCost<float, F>;
    using L = LazyOf<Fam>;
    static_assert(Fam::kArrays == 1, "deferred fold: one accumulator");
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature);
    const PhiloxChain pa = philox_chain(cA, level, keys);
    const PhiloxChain pb = philox_chain(cB, level, keys);
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    const float sa = L::sigma > 0 ? alpha : -alpha;
    bool haveA = true, haveB = true;
    int dA, dB;
    float tA, tB;
    {
        const uint64_t a1 = draw_bits53_fast(ctr, pa, keys), a2 = draw_bits53_fast(ctr + 1, pa, keys);
        const uint64_t b1 = draw_bits53_fast(ctr, pb, keys), b2 = draw_bits53_fast(ctr + 1, pb, keys);
        dA = min(static_cast<int>(static_cast<double>(a1) * idx_scale), n - 1);
        dB = min(static_cast<int>(static_cast<double>(b1) * idx_scale), n - 1);
        float t[1];
        Cost::cache(static_cast<float>(box.point(dA, bits_to_uniform(a2))), dA, n, t);
        tA = t[0];
        Cost::cache(static_cast<float>(box.point(dB, bits_to_uniform(b2))), dB, n, t);
        tB = t[0];
    }
    for (int j0 = 0; j0 < N; j0 += 32) {
        const int jn = N - j0 < 32 ? N - j0 : 32;
        uint32_t wordA = 0, wordB = 0;
        for (int j = 0; j < jn; ++j) {
            const float oA = row[2 * dA], oB = row[2 * dB + 1];
            // independent of this trial's outcome: its acceptance draws and
            // the next proposals
            const uint64_t mA = draw_bits53_fast(ctr + 2, pa, keys);
            const uint64_t mB = draw_bits53_fast(ctr + 2, pb, keys);
            const uint64_t a1 = draw_bits53_fast(ctr + 3, pa, keys), a2 = draw_bits53_fast(ctr + 4, pa, keys);
            const uint64_t b1 = draw_bits53_fast(ctr + 3, pb, keys), b2 = draw_bits53_fast(ctr + 4, pb, keys);
            const int nA = min(static_cast<int>(static_cast<double>(a1) * idx_scale), n - 1);
            const int nB = min(static_cast<int>(static_cast<double>(b1) * idx_scale), n - 1);
            const double yA = box.point(nA, bits_to_uniform(a2));
            const double yB = box.point(nB, bits_to_uniform(b2));
            float uA[1], uB[1];
            bool okA, okB;
            Cost::cache_common(static_cast<float>(yA), nA, n, uA, okA);
            Cost::cache_common(static_cast<float>(yB), nB, n, uB, okB);
            const MBand bA = metropolis_band(mA), bB = metropolis_band(mB);
            // the interval decisions
            const float qA = (tA - oA) * sa, qB = (tB - oB) * sa;
            const float hA = qA + rr, lA = qA - rr, hB = qB + rr, lB = qB - rr;
            int rA = ((hA <= 0.0f) | (hA * k2 < bA.lo)) ? 1 : (((lA > 0.0f) & (lA * k2 > bA.hi)) ? 0 : -1);
            int rB = ((hB <= 0.0f) | (hB * k2 < bB.lo)) ? 1 : (((lB > 0.0f) & (lB * k2 > bB.hi)) ? 0 : -1);
            bool setA = false, setB = false;
            if (__any_sync(kFullWarp, (!(okA & okB)) | (rA < 0) | (rB < 0))) {
                if (!okA) Cost::cache(static_cast<float>(yA), nA, n, uA);
                if (!okB) Cost::cache(static_cast<float>(yB), nB, n, uB);
                if (__any_sync(kFullWarp, (rA < 0) | (rB < 0))) {
                    if (__any_sync(kFullWarp, ((rA < 0) & !haveA) | ((rB < 0) & !haveB))) {
                        float eA, eB;
                        pair_energy<Fam, NT>(row, n, eA, eB);
                        if (!haveA) EA = eA;
                        if (!haveB) EB = eB;
                        haveA = haveB = true;
                    }
                    if (rA < 0) row[2 * dA] = tA;
                    if (rB < 0) row[2 * dB + 1] = tB;
                    float eA, eB;
                    pair_energy<Fam, NT>(row, n, eA, eB);
                    if (rA < 0) {
                        int v = metropolis_fast<float>(eA, EA, k2, bA);
                        if (v < 0) v = Accept<float>::exact(static_cast<double>(eA) - static_cast<double>(EA), temperature, mA);
                        if (v) EA = eA;
                        else row[2 * dA] = oA;
                        rA = v;
                        setA = true;
                        st.settles += cntA;
                    }
                    if (rB < 0) {
                        int v = metropolis_fast<float>(eB, EB, k2, bB);
                        if (v < 0) v = Accept<float>::exact(static_cast<double>(eB) - static_cast<double>(EB), temperature, mB);
                        if (v) EB = eB;
                        else row[2 * dB + 1] = oB;
                        rB = v;
                        setB = true;
                        st.settles += cntB;
                    }
                }
            }
            if (rA && !setA) {
                row[2 * dA] = tA;
                haveA = false;
            }
            if (rB && !setB) {
                row[2 * dB + 1] = tB;
                haveB = false;
            }
            ctr += 3;
            wordA |= static_cast<uint32_t>(rA) << j;
            wordB |= static_cast<uint32_t>(rB) << j;
            dA = nA;
            dB = nB;
            tA = uA[0];
            tB = uB[0];
        }
        if (maskA) maskA[static_cast<size_t>(j0 >> 5) * mask_stride] = wordA;
        if (maskB) maskB[static_cast<size_t>(j0 >> 5) * mask_stride] = wordB;
    }
    if (__any_sync(kFullWarp, !(haveA & haveB))) {
        float eA, eB;
        pair_energy<Fam, NT>(row, n, eA, eB);
        if (!haveA) EA = eA;
        if (!haveB) EB = eB;
    }
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

constexpr double kInf = __builtin_huge_val();

// A start-scan candidate (engines.cpp:161-167: `if (E[c] < best_f)` from
// best_f = +inf): NaN and +inf energies never qualify.
PSA_DEV Cand start_cand(double e, int32_t c) { return e < kInf ? Cand{e, c, 0} : empty_cand(); }

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
