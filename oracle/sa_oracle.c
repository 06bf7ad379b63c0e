/*
 * sa_oracle.c — TEST INFRASTRUCTURE ONLY (see sa_oracle.h).
 *
 * Plain-C restatement of the reference algorithm, serial, calling the system
 * glibc libm exactly like the reference (objectives.cpp uses std::sin etc.,
 * which resolve to glibc's IFUNC-dispatched sin/sinf/...).  Build flags keep
 * the reference's arithmetic: no -march (baseline x86-64, so no FMA
 * contraction), -ffp-contract=off, no -ffast-math.
 */
#include "sa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "parsa_suite_data.h"
#include "parsa_stdsort.h"

/* ------------------------------------------------------------------------ */
/* RNG — rng.hpp                                                             */
/* ------------------------------------------------------------------------ */

/* rng.hpp:30-33 Philox constants */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

/* rng.hpp:39-52 */
void orc_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t v0 = ctr[0], v1 = ctr[1], v2 = ctr[2], v3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)PHILOX_M0 * v0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * v2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ v1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ v3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        v0 = n0; v1 = n1; v2 = n2; v3 = n3;
        k0 += PHILOX_W0;
        k1 += PHILOX_W1;
    }
    out[0] = v0; out[1] = v1; out[2] = v2; out[3] = v3;
}

/* rng.hpp:56-91 UniformStream */
typedef struct stream {
    uint32_t k0, k1, chain, level;
    uint64_t counter;
} stream;

static stream make_stream(uint64_t seed, uint32_t chain, uint32_t level) {
    stream s = {(uint32_t)seed, (uint32_t)(seed >> 32), chain, level, 0};
    return s;
}

/* rng.hpp:66-75 */
static double next_uniform(stream* s) {
    uint32_t ctr[4] = {(uint32_t)s->counter, (uint32_t)(s->counter >> 32), s->chain, s->level};
    uint32_t out[4];
    orc_philox4x32_10(ctr, s->k0, s->k1, out);
    s->counter++;
    uint64_t bits = ((uint64_t)out[1] << 32) | (uint64_t)out[0];
    return (double)(bits >> 11) * 0x1.0p-53;
}

/* rng.hpp:78-81 */
int32_t orc_coordinate_index(double u, int32_t n) {
    int d = (int)(u * (double)n);
    return d < n ? d : n - 1;
}

static int next_coordinate_index(stream* s, int n) { return orc_coordinate_index(next_uniform(s), n); }

void orc_uniforms(uint64_t seed, uint32_t chain, uint32_t level, uint64_t first, int32_t count,
                  double* out) {
    stream s = make_stream(seed, chain, level);
    s.counter = first;
    for (int i = 0; i < count; ++i) out[i] = next_uniform(&s);
}

/* ------------------------------------------------------------------------ */
/* Schedule — sa_core.cpp                                                    */
/* ------------------------------------------------------------------------ */

/* sa_core.cpp:8-15: 0 ok; 1 t_min/t0, 2 rho, 3 sweep_length */
int32_t orc_schedule_validate(const psa_schedule* s) {
    if (!(s->t0 > 0) || !(s->t_min > 0) || !(s->t_min < s->t0)) return 1;
    if (!(s->rho > 0) || !(s->rho < 1)) return 2;
    if (s->sweep_length < 1) return 3;
    return 0;
}

/* sa_core.cpp:17-27 — do-while by repeated multiplication */
int32_t orc_ladder(const psa_schedule* s, double* temps, int32_t capacity) {
    int32_t levels = 0;
    double t = s->t0;
    do {
        if (temps && levels < capacity) temps[levels] = t;
        ++levels;
        t *= s->rho;
    } while (t > s->t_min);
    return levels;
}

/* sa_core.cpp:29-35 */
uint64_t orc_expected_evaluations(const psa_schedule* s, int32_t n_chains) {
    uint64_t levels = (uint64_t)orc_ladder(s, NULL, 0);
    return (uint64_t)n_chains * (1 + (uint64_t)s->sweep_length * levels);
}

/* ------------------------------------------------------------------------ */
/* Objectives — objectives.cpp:20-284, instantiated for double and float     */
/* ------------------------------------------------------------------------ */

#define PI_D 3.141592653589793
#define PI_F 3.14159265f

/* One macro body per precision keeps the two instantiations textually
 * identical, like the reference's `template <class Real>`. */
/* PSA_FN_CONSTANT's value: set from the psa_objective by every entry point
   (orc_set_fn_param for the bare evaluators) */
static double orc_fn_param = 0.0;
void orc_set_fn_param(double c) { orc_fn_param = c; }

#define DEFINE_SUITE(R, SFX, SIN, COS, EXP, SQRT, FABS, PI)                                    \
    static R schwefel_##SFX(const R* x, int n) { /* objectives.cpp:23-29 */                    \
        R s = 0;                                                                               \
        for (int i = 0; i < n; ++i) s += x[i] * SIN(SQRT(FABS(x[i])));                         \
        return -s / (R)n;                                                                      \
    }                                                                                          \
    static R ackley_##SFX(const R* x, int n) { /* :31-41 */                                    \
        R sq = 0, cs = 0;                                                                      \
        for (int i = 0; i < n; ++i) {                                                          \
            sq += x[i] * x[i];                                                                 \
            cs += COS((R)2 * PI * x[i]);                                                       \
        }                                                                                      \
        const R inv_n = (R)1 / (R)n;                                                           \
        return (R)(-20) * EXP((R)(-0.2) * SQRT(inv_n * sq)) - EXP(inv_n * cs) + (R)20 +        \
               EXP((R)1);                                                                      \
    }                                                                                          \
    static R branin_##SFX(const R* x, int n) { /* :43-49 */                                    \
        (void)n;                                                                               \
        const R a = x[1] - (R)5.1 / ((R)4 * PI * PI) * x[0] * x[0] + (R)5 / PI * x[0] - (R)6;  \
        return a * a + (R)10 * ((R)1 - (R)1 / ((R)8 * PI)) * COS(x[0]) + (R)10;                \
    }                                                                                          \
    static R cosine_mixture_##SFX(const R* x, int n) { /* :54-62 */                            \
        R c = 0, q = 0;                                                                        \
        for (int i = 0; i < n; ++i) {                                                          \
            c += COS((R)5 * PI * x[i]);                                                        \
            q += x[i] * x[i];                                                                  \
        }                                                                                      \
        return q - (R)0.1 * c;                                                                 \
    }                                                                                          \
    static R dekkers_aarts_##SFX(const R* x, int n) { /* :64-69 */                             \
        (void)n;                                                                               \
        const R r2 = x[0] * x[0] + x[1] * x[1];                                                \
        const R r4 = r2 * r2;                                                                  \
        return (R)1e5 * x[0] * x[0] + x[1] * x[1] - r4 + (R)1e-5 * r4 * r4;                    \
    }                                                                                          \
    static R easom_##SFX(const R* x, int n) { /* :71-75 */                                     \
        (void)n;                                                                               \
        const R dx = x[0] - PI, dy = x[1] - PI;                                                \
        return -COS(x[0]) * COS(x[1]) * EXP(-dx * dx - dy * dy);                               \
    }                                                                                          \
    static R exponential_##SFX(const R* x, int n) { /* :77-83 */                               \
        R sq = 0;                                                                              \
        for (int i = 0; i < n; ++i) sq += x[i] * x[i];                                         \
        return -EXP((R)(-0.5) * sq);                                                           \
    }                                                                                          \
    static R goldstein_price_##SFX(const R* x, int n) { /* :85-94 */                           \
        (void)n;                                                                               \
        const R a = x[0] + x[1] + (R)1;                                                        \
        const R b = (R)19 - (R)14 * x[0] + (R)3 * x[0] * x[0] - (R)14 * x[1] +                 \
                    (R)6 * x[0] * x[1] + (R)3 * x[1] * x[1];                                   \
        const R c = (R)2 * x[0] - (R)3 * x[1];                                                 \
        const R d = (R)18 - (R)32 * x[0] + (R)12 * x[0] * x[0] + (R)48 * x[1] -                \
                    (R)36 * x[0] * x[1] + (R)27 * x[1] * x[1];                                 \
        return ((R)1 + a * a * b) * ((R)30 + c * c * d);                                       \
    }                                                                                          \
    static R griewank_##SFX(const R* x, int n) { /* :99-107 */                                 \
        R sum = 0, prod = 1;                                                                   \
        for (int i = 0; i < n; ++i) {                                                          \
            sum += x[i] * x[i] / (R)4000;                                                      \
            prod *= COS(x[i] / SQRT((R)(i + 1)));                                              \
        }                                                                                      \
        return (R)1 + sum - prod;                                                              \
    }                                                                                          \
    static R himmelblau_##SFX(const R* x, int n) { /* :109-114 */                              \
        (void)n;                                                                               \
        const R a = x[0] * x[0] + x[1] - (R)11;                                                \
        const R b = x[0] + x[1] * x[1] - (R)7;                                                 \
        return a * a + b * b;                                                                  \
    }                                                                                          \
    static R levy_y_##SFX(const R* x, int i) { return (R)1 + (x[i] + (R)1) / (R)4; }           \
    static R levy_sin2_##SFX(R t) {                                                            \
        const R s = SIN(t);                                                                    \
        return s * s;                                                                          \
    }                                                                                          \
    static R levy_montalvo_##SFX(const R* x, int n) { /* :116-131 */                           \
        R acc = (R)10 * levy_sin2_##SFX(PI * levy_y_##SFX(x, 0));                              \
        for (int i = 0; i + 1 < n; ++i) {                                                      \
            const R d = levy_y_##SFX(x, i) - (R)1;                                             \
            acc += d * d * ((R)1 + (R)10 * levy_sin2_##SFX(PI * levy_y_##SFX(x, i + 1)));      \
        }                                                                                      \
        const R dn = levy_y_##SFX(x, n - 1) - (R)1;                                            \
        acc += dn * dn;                                                                        \
        return PI / (R)n * acc;                                                                \
    }                                                                                          \
    static R langerman_##SFX(const R* x, int n) { /* :172-185 */                               \
        R f = 0;                                                                               \
        for (int i = 0; i < 5; ++i) {                                                          \
            R d2 = 0;                                                                          \
            for (int j = 0; j < n; ++j) {                                                      \
                const R d = x[j] - (R)psa_fox_a[i][j];                                         \
                d2 += d * d;                                                                   \
            }                                                                                  \
            f -= (R)psa_fox_c[i] * EXP(-d2 / PI) * COS(PI * d2);                               \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R michalewicz_##SFX(const R* x, int n) { /* :187-198 */                             \
        R f = 0;                                                                               \
        for (int i = 0; i < n; ++i) {                                                          \
            const R s = SIN((R)(i + 1) * x[i] * x[i] / PI);                                    \
            const R s2 = s * s;                                                                \
            const R s4 = s2 * s2;                                                              \
            const R s16 = s4 * s4 * s4 * s4;                                                   \
            f -= SIN(x[i]) * s16 * s4;                                                         \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R rastrigin_##SFX(const R* x, int n) { /* :200-206 */                               \
        R f = (R)10 * (R)n;                                                                    \
        for (int i = 0; i < n; ++i) f += x[i] * x[i] - (R)10 * COS((R)2 * PI * x[i]);          \
        return f;                                                                              \
    }                                                                                          \
    static R rosenbrock_##SFX(const R* x, int n) { /* :212-221 */                              \
        R f = 0;                                                                               \
        for (int i = 0; i + 1 < n; ++i) {                                                      \
            const R a = x[i + 1] - x[i] * x[i];                                                \
            const R b = (R)1 - x[i];                                                           \
            f += (R)100 * a * a + b * b;                                                       \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R salomon_##SFX(const R* x, int n) { /* :223-230 */                                 \
        R sq = 0;                                                                              \
        for (int i = 0; i < n; ++i) sq += x[i] * x[i];                                         \
        const R r = SQRT(sq);                                                                  \
        return (R)1 - COS((R)2 * PI * r) + (R)0.1 * r;                                         \
    }                                                                                          \
    static R six_hump_##SFX(const R* x, int n) { /* :232-237 */                                \
        (void)n;                                                                               \
        const R x2 = x[0] * x[0];                                                              \
        const R y2 = x[1] * x[1];                                                              \
        return ((R)4 - (R)2.1 * x2 + x2 * x2 / (R)3) * x2 + x[0] * x[1] +                      \
               ((R)(-4) + (R)4 * y2) * y2;                                                     \
    }                                                                                          \
    static R shubert_##SFX(const R* x, int n) { /* :239-248 */                                 \
        R f = 1;                                                                               \
        for (int i = 0; i < n; ++i) {                                                          \
            R s = 0;                                                                           \
            for (int j = 1; j <= 5; ++j) s += (R)j * COS((R)(j + 1) * x[i] + (R)j);            \
            f *= s;                                                                            \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R shekel_##SFX(const R* x, int m) { /* :258-270 (m rows; n fixed at 4) */           \
        R f = 0;                                                                               \
        for (int i = 0; i < m; ++i) {                                                          \
            R d2 = 0;                                                                          \
            for (int j = 0; j < 4; ++j) {                                                      \
                const R d = x[j] - (R)psa_shekel_a[i][j];                                      \
                d2 += d * d;                                                                   \
            }                                                                                  \
            f -= (R)1 / (d2 + (R)psa_shekel_c[i]);                                             \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R foxholes_##SFX(const R* x, int n) { /* :272-284 */                                \
        R f = 0;                                                                               \
        for (int i = 0; i < PSA_FOX_ROWS; ++i) {                                               \
            R d2 = 0;                                                                          \
            for (int j = 0; j < n; ++j) {                                                      \
                const R d = x[j] - (R)psa_fox_a[i][j];                                         \
                d2 += d * d;                                                                   \
            }                                                                                  \
            f -= (R)1 / (d2 + (R)psa_fox_c[i]);                                                \
        }                                                                                      \
        return f;                                                                              \
    }                                                                                          \
    static R sphere_##SFX(const R* x, int n) { /* test_nelder_mead.cpp:17-38 bowl */           \
        R s = 0;                                                                               \
        for (int i = 0; i < n; ++i) s += x[i] * x[i];                                          \
        return s;                                                                              \
    }                                                                                          \
    static R eval_##SFX(int family, const R* x, int n) {                                       \
        switch (family) {                                                                      \
        case PSA_FN_SCHWEFEL: return schwefel_##SFX(x, n);                                     \
        case PSA_FN_ACKLEY: return ackley_##SFX(x, n);                                         \
        case PSA_FN_BRANIN: return branin_##SFX(x, n);                                         \
        case PSA_FN_COSINE_MIXTURE: return cosine_mixture_##SFX(x, n);                         \
        case PSA_FN_DEKKERS_AARTS: return dekkers_aarts_##SFX(x, n);                           \
        case PSA_FN_EASOM: return easom_##SFX(x, n);                                           \
        case PSA_FN_EXPONENTIAL: return exponential_##SFX(x, n);                               \
        case PSA_FN_GOLDSTEIN_PRICE: return goldstein_price_##SFX(x, n);                       \
        case PSA_FN_GRIEWANK: return griewank_##SFX(x, n);                                     \
        case PSA_FN_HIMMELBLAU: return himmelblau_##SFX(x, n);                                 \
        case PSA_FN_LEVY_MONTALVO: return levy_montalvo_##SFX(x, n);                           \
        case PSA_FN_MOD_LANGERMAN: return langerman_##SFX(x, n);                               \
        case PSA_FN_MICHALEWICZ: return michalewicz_##SFX(x, n);                               \
        case PSA_FN_RASTRIGIN: return rastrigin_##SFX(x, n);                                   \
        case PSA_FN_ROSENBROCK: return rosenbrock_##SFX(x, n);                                 \
        case PSA_FN_SALOMON: return salomon_##SFX(x, n);                                       \
        case PSA_FN_SIX_HUMP_CAMEL: return six_hump_##SFX(x, n);                               \
        case PSA_FN_SHUBERT: return shubert_##SFX(x, n);                                       \
        case PSA_FN_SHEKEL5: return shekel_##SFX(x, 5);                                        \
        case PSA_FN_SHEKEL7: return shekel_##SFX(x, 7);                                        \
        case PSA_FN_SHEKEL10: return shekel_##SFX(x, 10);                                      \
        case PSA_FN_SHEKEL_FOXHOLES: return foxholes_##SFX(x, n);                              \
        case PSA_FN_SPHERE: return sphere_##SFX(x, n);                                         \
        case PSA_FN_CONSTANT: return (R)orc_fn_param;                                          \
        default: return (R)NAN;                                                                \
        }                                                                                      \
    }

DEFINE_SUITE(double, d, sin, cos, exp, sqrt, fabs, PI_D)
DEFINE_SUITE(float, f, sinf, cosf, expf, sqrtf, fabsf, PI_F)

/* objectives.cpp:498-501 */
double orc_evaluate(int32_t family, int32_t n, const double* x) { return eval_d(family, x, n); }

/* objectives.cpp:503-510: round every coordinate to float, evaluate in float */
double orc_evaluate_single(int32_t family, int32_t n, const double* x) {
    float buf[1024];
    float* b = n <= 1024 ? buf : (float*)malloc(sizeof(float) * (size_t)n);
    for (int k = 0; k < n; ++k) b[k] = (float)x[k];
    double r = (double)eval_f(family, b, n);
    if (b != buf) free(b);
    return r;
}

/* sa_core.cpp:57-59 */
static double chain_energy(const psa_objective* f, const double* x, int prec) {
    return prec == PSA_F32 ? orc_evaluate_single(f->family, f->dim, x)
                           : orc_evaluate(f->family, f->dim, x);
}

/* ------------------------------------------------------------------------ */
/* SA core — sa_core.cpp:46-79                                               */
/* ------------------------------------------------------------------------ */

/* sa_core.cpp:46-55 */
static int metropolis_accept(double delta_e, double temperature, stream* s, int prec) {
    const double u = next_uniform(s); /* consumed on every step */
    if (delta_e <= 0) return 1;
    if (prec == PSA_F32)
        return (float)u <= expf(-(float)delta_e / (float)temperature);
    return u <= exp(-delta_e / temperature);
}

typedef struct chain {
    double* x;
    double energy;
    stream st;
} chain;

/* sa_core.cpp:61-79; returns the accept bits in `mask` if non-NULL */
static void metropolis_sweep(chain* c, const psa_objective* f, const double* width,
                             double temperature, int n_steps, int prec, uint64_t* evals,
                             uint32_t* mask) {
    const int n = f->dim;
    for (int step = 0; step < n_steps; ++step) {
        const int d = next_coordinate_index(&c->st, n);
        const double u = next_uniform(&c->st);
        const double old = c->x[d];
        c->x[d] = f->lower[d] + u * width[d];
        const double trial = chain_energy(f, c->x, prec);
        ++*evals;
        if (metropolis_accept(trial - c->energy, temperature, &c->st, prec)) {
            c->energy = trial;
            if (mask) mask[step >> 5] |= 1u << (step & 31);
        } else {
            c->x[d] = old;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Engines — engines.cpp                                                     */
/* ------------------------------------------------------------------------ */

/* engines.cpp:55-64 */
int32_t orc_reduce_min(const double* f, const int32_t* chain, int32_t count) {
    if (count <= 0) return -1;
    int32_t best = 0;
    for (int32_t i = 0; i < count; ++i)
        if (f[i] < f[best] || (f[i] == f[best] && chain[i] < chain[best])) best = i;
    return best;
}

static int contains(const psa_objective* f, const double* x) {
    for (int k = 0; k < f->dim; ++k)
        if (x[k] < f->lower[k] || x[k] > f->upper[k]) return 0;
    return 1;
}

/* engines.cpp:36-41 (box centre: objectives.cpp:484-488) */
static int resolve_start(const psa_objective* f, const psa_engine_config* cfg, double* start) {
    const int n = f->dim;
    if (cfg->start_point && cfg->start_point_len > 0) {
        if (cfg->start_point_len != n) return PSA_ERR_INVALID_ARGUMENT;
        memcpy(start, cfg->start_point, sizeof(double) * (size_t)n);
    } else {
        for (int k = 0; k < n; ++k) start[k] = 0.5 * (f->lower[k] + f->upper[k]);
    }
    if (!contains(f, start)) return PSA_ERR_INVALID_ARGUMENT;
    return 0;
}

/* engines.cpp:43-46 */
static void draw_random_start(double* x, const psa_objective* f, const double* width, stream* s) {
    for (int k = 0; k < f->dim; ++k) x[k] = f->lower[k] + next_uniform(s) * width[k];
}

/* engines.cpp:48-51 */
static uint64_t cumulative_evals_at(const psa_engine_config* cfg, int level) {
    return (uint64_t)cfg->n_chains * (1 + (uint64_t)cfg->schedule.sweep_length * (uint64_t)(level + 1));
}

static double* widths(const psa_objective* f) {
    double* w = (double*)malloc(sizeof(double) * (size_t)f->dim);
    for (int k = 0; k < f->dim; ++k) w[k] = f->upper[k] - f->lower[k]; /* BoxDomain::width */
    return w;
}

static void trace_push(psa_run_result* out, int level, uint64_t cum, double best) {
    if (out->trace && out->trace_len < out->trace_capacity) {
        psa_trace_point* p = &out->trace[out->trace_len];
        p->level = level;
        p->reserved = 0;
        p->cumulative_evals = cum;
        p->best_f = best;
    }
    out->trace_len++;
}

/* engines.cpp:131-207 */
int32_t orc_run_synchronous(const psa_objective* f, const psa_engine_config* cfg,
                            psa_run_result* out, orc_level_detail* detail) {
    orc_fn_param = f->param;
    if (orc_schedule_validate(&cfg->schedule)) return PSA_ERR_INVALID_ARGUMENT;
    if (cfg->n_chains < 1) return PSA_ERR_INVALID_ARGUMENT;
    const int n = f->dim, C = cfg->n_chains, N = cfg->schedule.sweep_length;
    const int levels = orc_ladder(&cfg->schedule, NULL, 0);
    double* temps = (double*)malloc(sizeof(double) * (size_t)levels);
    orc_ladder(&cfg->schedule, temps, levels);
    double* start = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = resolve_start(f, cfg, start);
    if (rc) { free(temps); free(start); return rc; }
    double* width = widths(f);
    const int mask_words = (N + 31) / 32;

    chain* ch = (chain*)calloc((size_t)C, sizeof(chain));
    double* xs = (double*)malloc(sizeof(double) * (size_t)C * (size_t)n);
    uint64_t* evals = (uint64_t*)calloc((size_t)C, sizeof(uint64_t));
    uint64_t* draws = (uint64_t*)calloc((size_t)C, sizeof(uint64_t));
    uint32_t* masks = (uint32_t*)calloc((size_t)C * (size_t)mask_words, sizeof(uint32_t));

    out->trace_len = 0;
    out->best_f = INFINITY;
    out->winning_chain = 0;
    double* best_x = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(best_x, start, sizeof(double) * (size_t)n);

    /* engines.cpp:149-160 level-0 starts */
    for (int c = 0; c < C; ++c) {
        ch[c].x = xs + (size_t)c * (size_t)n;
        ch[c].st = make_stream(cfg->seed, (uint32_t)c, 0);
        memcpy(ch[c].x, start, sizeof(double) * (size_t)n);
        if (cfg->start_mode == PSA_RANDOM_PER_CHAIN) draw_random_start(ch[c].x, f, width, &ch[c].st);
        ch[c].energy = chain_energy(f, ch[c].x, cfg->precision);
        evals[c] = 1;
    }
    /* engines.cpp:161-167 */
    for (int c = 0; c < C; ++c) {
        if (ch[c].energy < out->best_f) {
            out->best_f = ch[c].energy;
            memcpy(best_x, ch[c].x, sizeof(double) * (size_t)n);
            out->winning_chain = c;
        }
    }
    double* level_start = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(level_start, best_x, sizeof(double) * (size_t)n);
    double level_start_e = out->best_f;

    for (int l = 0; l < levels; ++l) { /* engines.cpp:171-199 */
        const double temperature = temps[l];
        for (int c = 0; c < C; ++c) {
            if (l > 0) {
                ch[c].st = make_stream(cfg->seed, (uint32_t)c, (uint32_t)l);
                memcpy(ch[c].x, level_start, sizeof(double) * (size_t)n);
                ch[c].energy = level_start_e;
            }
            uint32_t* m = masks + (size_t)c * (size_t)mask_words;
            memset(m, 0, sizeof(uint32_t) * (size_t)mask_words);
            metropolis_sweep(&ch[c], f, width, temperature, N, cfg->precision, &evals[c], m);
            draws[c] += ch[c].st.counter;
        }
        int winner = 0; /* engines.cpp:187-190 */
        for (int c = 1; c < C; ++c)
            if (ch[c].energy < ch[winner].energy) winner = c;
        memcpy(level_start, ch[winner].x, sizeof(double) * (size_t)n);
        level_start_e = ch[winner].energy;
        if (detail) {
            if (detail->winner) detail->winner[l] = winner;
            if (detail->winner_f) detail->winner_f[l] = level_start_e;
            if (detail->accept_mask)
                memcpy(detail->accept_mask + (size_t)l * (size_t)mask_words,
                       masks + (size_t)winner * (size_t)mask_words, sizeof(uint32_t) * (size_t)mask_words);
        }
        if (level_start_e < out->best_f) { /* engines.cpp:193-197 */
            out->best_f = level_start_e;
            memcpy(best_x, level_start, sizeof(double) * (size_t)n);
            out->winning_chain = winner;
        }
        trace_push(out, l, cumulative_evals_at(cfg, l), out->best_f);
    }

    out->evaluations = 0;
    out->rng_draws = 0;
    for (int c = 0; c < C; ++c) out->evaluations += evals[c];
    for (int c = 0; c < C; ++c) out->rng_draws += draws[c];
    if (out->best_x) memcpy(out->best_x, best_x, sizeof(double) * (size_t)n);
    out->has_phases = 0;
    out->wall_time_s = 0;

    free(temps); free(start); free(width); free(ch); free(xs); free(evals); free(draws);
    free(masks); free(best_x); free(level_start);
    return 0;
}

/* engines.cpp:66-123 */
int32_t orc_run_asynchronous(const psa_objective* f, const psa_engine_config* cfg,
                             psa_run_result* out) {
    orc_fn_param = f->param;
    if (orc_schedule_validate(&cfg->schedule)) return PSA_ERR_INVALID_ARGUMENT;
    if (cfg->n_chains < 1) return PSA_ERR_INVALID_ARGUMENT;
    const int n = f->dim, C = cfg->n_chains, N = cfg->schedule.sweep_length;
    const int levels = orc_ladder(&cfg->schedule, NULL, 0);
    double* temps = (double*)malloc(sizeof(double) * (size_t)levels);
    orc_ladder(&cfg->schedule, temps, levels);
    double* start = (double*)malloc(sizeof(double) * (size_t)n);
    int rc = resolve_start(f, cfg, start);
    if (rc) { free(temps); free(start); return rc; }
    double* width = widths(f);

    chain* ch = (chain*)calloc((size_t)C, sizeof(chain));
    double* xs = (double*)malloc(sizeof(double) * (size_t)C * (size_t)n);
    uint64_t* evals = (uint64_t*)calloc((size_t)C, sizeof(uint64_t));
    double* best_by_level = (double*)malloc(sizeof(double) * (size_t)C * (size_t)levels);

    for (int c = 0; c < C; ++c) { /* engines.cpp:81-97 */
        ch[c].x = xs + (size_t)c * (size_t)n;
        ch[c].st = make_stream(cfg->seed, (uint32_t)c, 0);
        memcpy(ch[c].x, start, sizeof(double) * (size_t)n);
        if (cfg->start_mode == PSA_RANDOM_PER_CHAIN) draw_random_start(ch[c].x, f, width, &ch[c].st);
        ch[c].energy = chain_energy(f, ch[c].x, cfg->precision);
        evals[c] = 1;
        double chain_best = ch[c].energy;
        for (int l = 0; l < levels; ++l) {
            metropolis_sweep(&ch[c], f, width, temps[l], N, cfg->precision, &evals[c], NULL);
            /* std::min(chain_best, energy) == (energy < chain_best) ? energy : chain_best */
            chain_best = ch[c].energy < chain_best ? ch[c].energy : chain_best;
            best_by_level[(size_t)c * (size_t)levels + (size_t)l] = chain_best;
        }
    }
    out->trace_len = 0;
    for (int l = 0; l < levels; ++l) { /* engines.cpp:101-106 */
        double m = INFINITY;
        for (int c = 0; c < C; ++c) {
            const double v = best_by_level[(size_t)c * (size_t)levels + (size_t)l];
            m = v < m ? v : m; /* std::min(m, v) */
        }
        trace_push(out, l, cumulative_evals_at(cfg, l), m);
    }
    int winner = 0; /* engines.cpp:110-116 */
    for (int c = 1; c < C; ++c)
        if (ch[c].energy < ch[winner].energy) winner = c;
    if (out->best_x) memcpy(out->best_x, ch[winner].x, sizeof(double) * (size_t)n);
    out->best_f = ch[winner].energy;
    out->winning_chain = winner;
    out->evaluations = 0;
    out->rng_draws = 0;
    for (int c = 0; c < C; ++c) {
        out->evaluations += evals[c];
        out->rng_draws += ch[c].st.counter;
    }
    out->has_phases = 0;
    out->wall_time_s = 0;
    free(temps); free(start); free(width); free(ch); free(xs); free(evals); free(best_by_level);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Nelder–Mead and hybrid — nelder_mead.cpp                                  */
/* ------------------------------------------------------------------------ */

/* The simplex as vertex ids: X[id*n + k], f[id]; pos[] is the physical
 * order of std::vector<Vertex> simplex (nelder_mead.cpp:50), which
 * std::sort permutes — restated exactly by psa_std_sort (libstdc++). */

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* nelder_mead.cpp:30-35 */
static int nm_validate(const psa_nm_config* c) {
    if (!(c->reflect > 0) || !(c->expand > 1) || !(c->contract > 0) || !(c->contract < 1) ||
        !(c->shrink > 0) || !(c->shrink < 1))
        return PSA_ERR_INVALID_ARGUMENT;
    return 0;
}

/* nelder_mead.cpp:37-115 (always f64) */
int32_t orc_nelder_mead_minimize(const psa_objective* f, const double* x_start,
                                 const psa_nm_config* cfg, psa_nm_result* out) {
    orc_fn_param = f->param;
    if (nm_validate(cfg)) return PSA_ERR_INVALID_ARGUMENT;
    if (!contains(f, x_start)) return PSA_ERR_INVALID_ARGUMENT;
    const int n = f->dim;
    uint64_t evals = 0;
#define NM_EVAL(xx) (++evals, orc_evaluate(f->family, n, (xx)))
    double* X = (double*)malloc(sizeof(double) * (size_t)(n + 1) * (size_t)n);
    double* fv = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    int* pos = (int*)malloc(sizeof(int) * (size_t)(n + 1));
#define VX(id) (X + (size_t)(id) * (size_t)n)
    for (int v = 0; v <= n; ++v) pos[v] = v;
    memcpy(VX(0), x_start, sizeof(double) * (size_t)n);
    fv[0] = NM_EVAL(VX(0));
    for (int k = 0; k < n; ++k) { /* nelder_mead.cpp:52-58 */
        double* x = VX(k + 1);
        memcpy(x, x_start, sizeof(double) * (size_t)n);
        const double step = 0.05 * (f->upper[k] - f->lower[k]);
        x[k] = (x[k] + step <= f->upper[k]) ? x[k] + step : x[k] - step;
        fv[k + 1] = NM_EVAL(x);
    }
    psa_std_sort(pos, n + 1, fv); /* :60 */
    double* cen = (double*)malloc(sizeof(double) * (size_t)n);
    double* xr = (double*)malloc(sizeof(double) * (size_t)n);
    double* xe = (double*)malloc(sizeof(double) * (size_t)n);
    double* xc = (double*)malloc(sizeof(double) * (size_t)n);
    const int max_iters = cfg->max_iters > 0 ? cfg->max_iters : 50000 * n;
    int iter = 0;
    for (; iter < max_iters; ++iter) {
        /* nelder_mead.cpp:67-68, simplex_diameter :21-27 */
        double diam = 0;
        for (int i = 1; i <= n; ++i)
            for (int k = 0; k < n; ++k) {
                const double a = fabs(VX(pos[i])[k] - VX(pos[0])[k]);
                diam = diam < a ? a : diam; /* std::max(d, a) */
            }
        if (fv[pos[n]] - fv[pos[0]] <= cfg->f_tol || diam <= cfg->x_tol) break;
        for (int k = 0; k < n; ++k) cen[k] = 0.0; /* :70-73 */
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < n; ++k) cen[k] += VX(pos[i])[k] / n;
        const int w = pos[n];
        double* worst = VX(w);
        const double worst_f = fv[w];
        for (int k = 0; k < n; ++k) xr[k] = clampd(cen[k] + cfg->reflect * (cen[k] - worst[k]), f->lower[k], f->upper[k]);
        const double fr = NM_EVAL(xr);
        if (fr < fv[pos[0]]) {
            for (int k = 0; k < n; ++k) xe[k] = clampd(cen[k] + cfg->expand * (xr[k] - cen[k]), f->lower[k], f->upper[k]);
            const double fe = NM_EVAL(xe);
            if (fe < fr) { memcpy(worst, xe, sizeof(double) * (size_t)n); fv[w] = fe; }
            else { memcpy(worst, xr, sizeof(double) * (size_t)n); fv[w] = fr; }
        } else if (fr < fv[pos[n - 1]]) {
            memcpy(worst, xr, sizeof(double) * (size_t)n);
            fv[w] = fr;
        } else {
            const int outside = fr < worst_f;
            for (int k = 0; k < n; ++k) {
                const double toward = outside ? xr[k] : worst[k];
                xc[k] = clampd(cen[k] + cfg->contract * (toward - cen[k]), f->lower[k], f->upper[k]);
            }
            const double fc = NM_EVAL(xc);
            if (fc < (outside ? fr : worst_f)) {
                memcpy(worst, xc, sizeof(double) * (size_t)n);
                fv[w] = fc;
            } else {
                const double* x0 = VX(pos[0]);
                for (int i = 1; i <= n; ++i) {
                    double* xi = VX(pos[i]);
                    for (int k = 0; k < n; ++k)
                        xi[k] = clampd(x0[k] + cfg->shrink * (xi[k] - x0[k]), f->lower[k], f->upper[k]);
                    fv[pos[i]] = NM_EVAL(xi);
                }
            }
        }
        psa_std_sort(pos, n + 1, fv); /* :111 */
    }
#undef NM_EVAL
    if (out->x_best) memcpy(out->x_best, VX(pos[0]), sizeof(double) * (size_t)n);
    out->f_best = fv[pos[0]];
    out->iterations = iter;
    out->evaluations = evals;
#undef VX
    free(X); free(fv); free(pos); free(cen); free(xr); free(xe); free(xc);
    return 0;
}

/* nelder_mead.cpp:117-136 */
int32_t orc_hybrid_run(const psa_objective* f, const psa_engine_config* cfg,
                       const psa_schedule* truncated, const psa_nm_config* nm,
                       psa_run_result* out) {
    orc_fn_param = f->param;
    psa_engine_config sa = *cfg;
    sa.schedule = *truncated;
    const int cap = out->trace_capacity;
    int rc = orc_run_synchronous(f, &sa, out, NULL);
    if (rc) return rc;
    const double sa_best = out->best_f;
    double* xb = (double*)malloc(sizeof(double) * (size_t)f->dim);
    psa_nm_result r = {xb, 0, 0, 0, 0};
    rc = orc_nelder_mead_minimize(f, out->best_x, nm, &r);
    if (rc) { free(xb); return rc; }
    if (r.f_best <= out->best_f) {
        out->best_f = r.f_best;
        memcpy(out->best_x, xb, sizeof(double) * (size_t)f->dim);
    }
    out->has_phases = 1;
    out->sa_evaluations = out->evaluations;
    out->refine_evaluations = r.evaluations;
    out->sa_best_f = sa_best;
    out->evaluations += r.evaluations;
    (void)cap;
    trace_push(out, out->trace_len, out->evaluations, out->best_f);
    free(xb);
    return 0;
}
