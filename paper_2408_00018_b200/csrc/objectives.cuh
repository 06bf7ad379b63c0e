// objectives.cuh — device cost functions (the paper's test suite).
//
// Each family mirrors one formula template of objectives.cpp operation for
// operation (the translation unit is compiled with -fmad=false, so no a*b+c
// is contracted, matching the reference's baseline-x86-64 build), and calls
// the glibc restatements for sin/cos/exp so f32 and f64 costs are
// bit-identical to the reference's.
//
// Two shapes of family:
//
//  * separable (kSeparable = true): f = finish(fold_k term_k(x_k)), where the
//    fold runs over k in index order.  The engine caches term_k per chain, so
//    a one-coordinate Metropolis proposal recomputes ONE term (2
//    transcendentals) and re-folds the cached terms in the reference's
//    sequential order — the result is bit-identical to a full evaluation.
//  * full (kSeparable = false): the cache holds x_k itself (as Real) and
//    energy() evaluates the whole formula.
//
// Cache layout seen by energy(): V(k, a) returns cached value a of
// coordinate k (a < kArrays).
#pragma once

#include <stdint.h>

#include "libm_glibc.cuh"
#include "libm_glibc64.cuh"
#include "parsa_suite_data.h"

#ifndef PSA_DEV
#define PSA_DEV __device__ __forceinline__
#endif

namespace psa {

// ---- math dispatch: glibc-exact transcendental, IEEE sqrt ---------------
template <class R>
struct Math;

template <>
struct Math<double> {
    PSA_HD static double sin(double x) { return libm::sin(x); }
    PSA_HD static double cos(double x) { return libm::cos(x); }
    PSA_HD static double exp(double x) { return libm::exp(x); }
    PSA_HD static double sqrt(double x) {
#ifdef __CUDA_ARCH__
        return __dsqrt_rn(x);
#else
        return __builtin_sqrt(x);
#endif
    }
    PSA_HD static double fabs(double x) { return libm::fabs64(x); }
};

template <>
struct Math<float> {
    PSA_HD static float sin(float x) { return libm::sinf(x); }
    PSA_HD static float cos(float x) { return libm::cosf(x); }
    PSA_HD static float exp(float x) { return libm::expf(x); }
    PSA_HD static float sqrt(float x) {
#ifdef __CUDA_ARCH__
        return __fsqrt_rn(x);
#else
        return __builtin_sqrtf(x);
#endif
    }
    PSA_HD static float fabs(float x) {
#ifdef __CUDA_ARCH__
        return __uint_as_float(libm::asuint(x) & 0x7fffffffu);
#else
        return __builtin_fabsf(x);
#endif
    }
};

// pi_v<Real> (objectives.cpp:20-21): the long-double literal rounded to Real
template <class R>
struct Pi;
template <>
struct Pi<double> {
    static constexpr double v = 3.141592653589793;
};
template <>
struct Pi<float> {
    static constexpr float v = 3.14159265f;
};

// std::exp(Real(1)) is constant-folded (correctly rounded) by the reference build
template <class R>
struct Euler;
template <>
struct Euler<double> {
    static constexpr double v = 0x1.5bf0a8b145769p+1;
};
template <>
struct Euler<float> {
    static constexpr float v = 0x1.5bf0a8p+1f;
};

// Suite tables (parsa_suite_data.h): device copies in global memory.
#ifdef __CUDACC__
__device__ const double kFoxADev[PSA_FOX_ROWS][PSA_FOX_COLS] = PSA_FOX_A_INIT;
__device__ const double kFoxCDev[PSA_FOX_ROWS] = PSA_FOX_C_INIT;
__device__ const double kShekelADev[10][4] = PSA_SHEKEL_A_INIT;
__device__ const double kShekelCDev[10] = PSA_SHEKEL_C_INIT;
#endif
PSA_HD double fox_a(int i, int j) {
#ifdef __CUDA_ARCH__
    return kFoxADev[i][j];
#else
    return psa_fox_a[i][j];
#endif
}
PSA_HD double fox_c(int i) {
#ifdef __CUDA_ARCH__
    return kFoxCDev[i];
#else
    return psa_fox_c[i];
#endif
}
PSA_HD double shekel_a(int i, int j) {
#ifdef __CUDA_ARCH__
    return kShekelADev[i][j];
#else
    return psa_shekel_a[i][j];
#endif
}
PSA_HD double shekel_c(int i) {
#ifdef __CUDA_ARCH__
    return kShekelCDev[i];
#else
    return psa_shekel_c[i];
#endif
}

enum Fold { kAdd = 0, kSub = 1, kMul = 2 };

template <class R>
PSA_HD R fold(int op, R acc, R t) {
    return op == kAdd ? acc + t : (op == kSub ? acc - t : acc * t);
}

// ------------------------------------------------------------------------
// Separable families
// ------------------------------------------------------------------------

// objectives.cpp:23-29  s += x*sin(sqrt|x|); return -s/n
template <class R>
struct Schwefel {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    static constexpr bool kHasCommon = true;
    PSA_HD static void term(R x, int, R* t) { t[0] = x * Math<R>::sin(Math<R>::sqrt(Math<R>::fabs(x))); }
    // branch-free common path (see libm_glibc.cuh); ok=false -> use term()
    PSA_HD static void term_common(R x, int k, R* t, bool& ok) {
        if constexpr (sizeof(R) == 4) {
            bool ok1, ok2;
            const float sq = libm::sqrtf_common(Math<float>::fabs(x), ok1);
            const float sn = libm::sinf_common(sq, ok2);
            t[0] = x * sn;
            ok = ok1 & ok2;
        } else {
            term(x, k, t);
            ok = true;
        }
    }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int n) { return -acc[0] / R(n); }
};

// objectives.cpp:31-41  sq += x*x; cs += cos(2*pi*x)
template <class R>
struct Ackley {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 2;
    PSA_HD static void term(R x, int, R* t) {
        t[0] = x * x;
        t[1] = Math<R>::cos(R(2) * Pi<R>::v * x);
    }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int n) {
        const R inv_n = R(1) / R(n);
        return R(-20) * Math<R>::exp(R(-0.2) * Math<R>::sqrt(inv_n * acc[0])) -
               Math<R>::exp(inv_n * acc[1]) + R(20) + Euler<R>::v;
    }
};

// objectives.cpp:54-62  c += cos(5*pi*x); q += x*x; return q - 0.1*c
template <class R>
struct CosineMixture {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 2;
    PSA_HD static void term(R x, int, R* t) {
        t[0] = Math<R>::cos(R(5) * Pi<R>::v * x);
        t[1] = x * x;
    }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int) { return acc[1] - R(0.1) * acc[0]; }
};

// objectives.cpp:77-83  sq += x*x; return -exp(-0.5*sq)
template <class R>
struct Exponential {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) { t[0] = x * x; }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int) { return -Math<R>::exp(R(-0.5) * acc[0]); }
};

// objectives.cpp:99-107  sum += x*x/4000; prod *= cos(x/sqrt(i+1))
template <class R>
struct Griewank {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 2;
    PSA_HD static void term(R x, int k, R* t) {
        t[0] = x * x / R(4000);
        t[1] = Math<R>::cos(x / Math<R>::sqrt(R(k + 1)));
    }
    PSA_HD static R init(int a, int) { return a == 0 ? R(0) : R(1); }
    PSA_HD static int op(int a) { return a == 0 ? kAdd : kMul; }
    PSA_HD static R finish(const R* acc, int) { return R(1) + acc[0] - acc[1]; }
};

// objectives.cpp:187-198  f -= sin(x)*s^16*s^4, s = sin((i+1)*x*x/pi)
template <class R>
struct Michalewicz {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int k, R* t) {
        const R s = Math<R>::sin(R(k + 1) * x * x / Pi<R>::v);
        const R s2 = s * s;
        const R s4 = s2 * s2;
        const R s16 = s4 * s4 * s4 * s4;
        t[0] = Math<R>::sin(x) * s16 * s4;
    }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kSub; }
    PSA_HD static R finish(const R* acc, int) { return acc[0]; }
};

// objectives.cpp:200-206  f = 10n; f += x*x - 10*cos(2*pi*x)
template <class R>
struct Rastrigin {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) { t[0] = x * x - R(10) * Math<R>::cos(R(2) * Pi<R>::v * x); }
    PSA_HD static R init(int, int n) { return R(10) * R(n); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int) { return acc[0]; }
};

// objectives.cpp:223-230  r = sqrt(sum x^2); 1 - cos(2*pi*r) + 0.1*r
template <class R>
struct Salomon {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) { t[0] = x * x; }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int) {
        const R r = Math<R>::sqrt(acc[0]);
        return R(1) - Math<R>::cos(R(2) * Pi<R>::v * r) + R(0.1) * r;
    }
};

// objectives.cpp:239-248  f = 1; f *= sum_j j*cos((j+1)*x + j)
template <class R>
struct Shubert {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) {
        R s = 0;
        for (int j = 1; j <= 5; ++j) s += R(j) * Math<R>::cos(R(j + 1) * x + R(j));
        t[0] = s;
    }
    PSA_HD static R init(int, int) { return R(1); }
    PSA_HD static int op(int) { return kMul; }
    PSA_HD static R finish(const R* acc, int) { return acc[0]; }
};

// bowl fixture (test_nelder_mead.cpp:17-38)
template <class R>
struct Sphere {
    static constexpr bool kSeparable = true;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) { t[0] = x * x; }
    PSA_HD static R init(int, int) { return R(0); }
    PSA_HD static int op(int) { return kAdd; }
    PSA_HD static R finish(const R* acc, int) { return acc[0]; }
};

// ------------------------------------------------------------------------
// Deferred-fold traits (engine.cuh, sweep_lazy)
//
// Families whose energy is an affine image of ONE additive fold:
//   E = finish(s),  s = init (+/-) t_0 (+/-) t_1 ... (+/-) t_{n-1}  (sigma = +1 / -1)
//   finish(s) = alpha(n) * s, rounded fin_round times.
// For those the engine tracks S = init + sigma * sum t_k in double and settles
// a Metropolis decision from an interval around alpha*S whenever the interval
// is conclusive (engine.cuh explains the bound); term_bound(lo, hi) bounds
// |t| of a coordinate over [lo, hi] for the computed (rounded) term.
// ------------------------------------------------------------------------

template <class Fam>
struct LazyOf {
    static constexpr bool value = false;
};
template <class R>
struct LazyOf<Schwefel<R>> { // -s/n: one rounding (the division; negation is exact)
    static constexpr bool value = true;
    static constexpr int sigma = 1;
    static constexpr int fin_round = 1;
    PSA_HD static double alpha(int n) { return -1.0 / static_cast<double>(n); }
    // |x sin(sqrt|x|)| <= |x| (|sin| <= 1 for the glibc-exact sin)
    static double term_bound(double lo, double hi) { return fmax(fabs(lo), fabs(hi)); }
};
template <class R>
struct LazyOf<Rastrigin<R>> { // s from init 10n, finish = identity
    static constexpr bool value = true;
    static constexpr int sigma = 1;
    static constexpr int fin_round = 0;
    PSA_HD static double alpha(int) { return 1.0; }
    static double term_bound(double lo, double hi) {
        const double m = fmax(fabs(lo), fabs(hi));
        return m * m + 10.0;
    }
};
template <class R>
struct LazyOf<Sphere<R>> {
    static constexpr bool value = true;
    static constexpr int sigma = 1;
    static constexpr int fin_round = 0;
    PSA_HD static double alpha(int) { return 1.0; }
    static double term_bound(double lo, double hi) {
        const double m = fmax(fabs(lo), fabs(hi));
        return m * m;
    }
};
template <class R>
struct LazyOf<Michalewicz<R>> { // f = 0 - t_0 - t_1 ...
    static constexpr bool value = true;
    static constexpr int sigma = -1;
    static constexpr int fin_round = 0;
    PSA_HD static double alpha(int) { return 1.0; }
    static double term_bound(double, double) { return 1.0; } // |sin(x) s^20| <= 1
};

// ------------------------------------------------------------------------
// Full-evaluation families: X(k) returns x_k as Real
// ------------------------------------------------------------------------

template <class R>
struct Branin { // objectives.cpp:43-49
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R pi = Pi<R>::v;
        const R a = x(1) - R(5.1) / (R(4) * pi * pi) * x(0) * x(0) + R(5) / pi * x(0) - R(6);
        return a * a + R(10) * (R(1) - R(1) / (R(8) * pi)) * Math<R>::cos(x(0)) + R(10);
    }
};

template <class R>
struct DekkersAarts { // :64-69
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R r2 = x(0) * x(0) + x(1) * x(1);
        const R r4 = r2 * r2;
        return R(1e5) * x(0) * x(0) + x(1) * x(1) - r4 + R(1e-5) * r4 * r4;
    }
};

template <class R>
struct Easom { // :71-75
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R dx = x(0) - Pi<R>::v, dy = x(1) - Pi<R>::v;
        return -Math<R>::cos(x(0)) * Math<R>::cos(x(1)) * Math<R>::exp(-dx * dx - dy * dy);
    }
};

template <class R>
struct GoldsteinPrice { // :85-94
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R a = x(0) + x(1) + R(1);
        const R b = R(19) - R(14) * x(0) + R(3) * x(0) * x(0) - R(14) * x(1) + R(6) * x(0) * x(1) +
                    R(3) * x(1) * x(1);
        const R c = R(2) * x(0) - R(3) * x(1);
        const R d = R(18) - R(32) * x(0) + R(12) * x(0) * x(0) + R(48) * x(1) - R(36) * x(0) * x(1) +
                    R(27) * x(1) * x(1);
        return (R(1) + a * a * b) * (R(30) + c * c * d);
    }
};

template <class R>
struct Himmelblau { // :109-114
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R a = x(0) * x(0) + x(1) - R(11);
        const R b = x(0) + x(1) * x(1) - R(7);
        return a * a + b * b;
    }
};

template <class R>
struct LevyMontalvo { // :116-131
    template <class X>
    PSA_HD static R y(const X& x, int i) { return R(1) + (x(i) + R(1)) / R(4); }
    PSA_HD static R sin2(R t) {
        const R s = Math<R>::sin(t);
        return s * s;
    }
    template <class X>
    PSA_HD static R eval(const X& x, int n) {
        const R pi = Pi<R>::v;
        R acc = R(10) * sin2(pi * y(x, 0));
        for (int i = 0; i + 1 < n; ++i) {
            const R d = y(x, i) - R(1);
            acc += d * d * (R(1) + R(10) * sin2(pi * y(x, i + 1)));
        }
        const R dn = y(x, n - 1) - R(1);
        acc += dn * dn;
        return pi / R(n) * acc;
    }
};

template <class R>
struct ModLangerman { // :172-185 (n <= 10)
    template <class X>
    PSA_HD static R eval(const X& x, int n) {
        const R pi = Pi<R>::v;
        R f = 0;
        for (int i = 0; i < 5; ++i) {
            R d2 = 0;
            for (int j = 0; j < n; ++j) {
                const R d = x(j) - R(fox_a(i, j));
                d2 += d * d;
            }
            f -= R(fox_c(i)) * Math<R>::exp(-d2 / pi) * Math<R>::cos(pi * d2);
        }
        return f;
    }
};

template <class R>
struct Rosenbrock { // :212-221
    template <class X>
    PSA_HD static R eval(const X& x, int n) {
        R f = 0;
        for (int i = 0; i + 1 < n; ++i) {
            const R a = x(i + 1) - x(i) * x(i);
            const R b = R(1) - x(i);
            f += R(100) * a * a + b * b;
        }
        return f;
    }
};

template <class R>
struct SixHumpCamel { // :232-237
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        const R x2 = x(0) * x(0);
        const R y2 = x(1) * x(1);
        return (R(4) - R(2.1) * x2 + x2 * x2 / R(3)) * x2 + x(0) * x(1) + (R(-4) + R(4) * y2) * y2;
    }
};

template <class R, int M>
struct Shekel { // :258-270 (always 4 coordinates)
    template <class X>
    PSA_HD static R eval(const X& x, int) {
        R f = 0;
        for (int i = 0; i < M; ++i) {
            R d2 = 0;
            for (int j = 0; j < 4; ++j) {
                const R d = x(j) - R(shekel_a(i, j));
                d2 += d * d;
            }
            f -= R(1) / (d2 + R(shekel_c(i)));
        }
        return f;
    }
};

template <class R>
struct ShekelFoxholes { // :272-284 (n <= 10)
    template <class X>
    PSA_HD static R eval(const X& x, int n) {
        R f = 0;
        for (int i = 0; i < PSA_FOX_ROWS; ++i) {
            R d2 = 0;
            for (int j = 0; j < n; ++j) {
                const R d = x(j) - R(fox_a(i, j));
                d2 += d * d;
            }
            f -= R(1) / (d2 + R(fox_c(i)));
        }
        return f;
    }
};

// Wrap a full-evaluation formula into the engine's cache interface: the
// cached value of coordinate k is x_k itself.
template <class R, class F>
struct Full {
    static constexpr bool kSeparable = false;
    static constexpr int kArrays = 1;
    PSA_HD static void term(R x, int, R* t) { t[0] = x; }
};

} // namespace psa
