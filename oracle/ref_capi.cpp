// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// the reference's own sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libparsa_ref.so.  The reference namespace
// is renamed to parsa_ref (-Dparsa=parsa_ref) so it can sit beside the
// drop-in library in one process.  Used to pin the C restatement
// (sa_oracle.c), to generate tests/golden/, and as the CPU baseline arm of
// bench.py (`--impl reference`).  Nothing in the product links it.
#include <omp.h>

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "parsa/engines.hpp"
#include "parsa/nelder_mead.hpp"
#include "parsa/objectives.hpp"
#include "parsa/rng.hpp"
#include "parsa/sa_core.hpp"
#include "parsa_b200.h"

using namespace parsa_ref;

namespace {

thread_local std::string g_err;

// Registry entry whose formula template implements each psa_family; the
// dimension and box are then overridden (eval_f64/eval_f32 take n as an
// argument, objectives.hpp:36-37, so any n works).
const char* family_template_id(int family) {
    static const char* ids[] = {"F0_a", "F1_a", "F2",   "F3_a", "F4",   "F5",   "F6",  "F7",
                                "F8_a", "F9",   "F10_a", "F11_a", "F12_a", "F13_a", "F14", "F15",
                                "F16",  "F17",  "F18_a", "F18_b", "F18_c", "F19_a"};
    if (family < 0 || family >= int(sizeof(ids) / sizeof(ids[0]))) return nullptr;
    return ids[family];
}

double sphere_f64(const double* x, int n) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}
float sphere_f32(const float* x, int n) {
    float s = 0;
    for (int i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}

// PSA_FN_CONSTANT: the constant fixtures of test_engines.cpp:91-99 and
// test_sa_core.cpp:140-160 (value from the objective's param)
double g_constant = 0.0;
double constant_f64(const double*, int) { return g_constant; }
float constant_f32(const float*, int) { return static_cast<float>(g_constant); }

ObjectiveFunction make_objective(const psa_objective* o) {
    ObjectiveFunction f;
    if (o->family == PSA_FN_CONSTANT) {
        g_constant = o->param;
        f.id = "constant";
        f.name = "constant";
        f.eval_f64 = constant_f64;
        f.eval_f32 = constant_f32;
    } else if (o->family == PSA_FN_SPHERE) {
        f.id = "sphere";
        f.name = "sphere";
        f.eval_f64 = sphere_f64;
        f.eval_f32 = sphere_f32;
    } else {
        const char* id = family_template_id(o->family);
        if (!id) throw std::out_of_range("unknown family");
        f = registry_get(id);
    }
    if (o->id) f.id = o->id;
    f.dim = o->dim;
    f.domain.lower.assign(o->lower, o->lower + o->dim);
    f.domain.upper.assign(o->upper, o->upper + o->dim);
    return f;
}

EngineConfig make_config(const psa_objective* o, const psa_engine_config* c) {
    (void)o;
    EngineConfig cfg;
    cfg.n_chains = c->n_chains;
    cfg.start_mode = c->start_mode == PSA_RANDOM_PER_CHAIN ? StartMode::random_per_chain
                                                           : StartMode::shared_point;
    if (c->start_point && c->start_point_len > 0)
        cfg.start_point.assign(c->start_point, c->start_point + c->start_point_len);
    cfg.schedule = {c->schedule.t0, c->schedule.t_min, c->schedule.rho, c->schedule.sweep_length};
    cfg.precision = c->precision == PSA_F32 ? Precision::f32 : Precision::f64;
    cfg.seed = c->seed;
    cfg.workers = c->workers;
    return cfg;
}

void fill_result(const RunResult& r, psa_run_result* out) {
    if (out->best_x) std::memcpy(out->best_x, r.best_x.data(), sizeof(double) * r.best_x.size());
    out->best_f = r.best_f;
    out->evaluations = r.evaluations;
    out->wall_time_s = r.wall_time_s;
    out->winning_chain = r.winning_chain;
    out->rng_draws = r.rng_draws;
    out->trace_len = int32_t(r.trace.size());
    for (std::size_t i = 0; i < r.trace.size() && int(i) < out->trace_capacity; ++i) {
        out->trace[i].level = r.trace[i].level;
        out->trace[i].reserved = 0;
        out->trace[i].cumulative_evals = r.trace[i].cumulative_evals;
        out->trace[i].best_f = r.trace[i].best_f;
    }
    out->has_phases = r.phases.has_value();
    if (r.phases) {
        out->sa_evaluations = r.phases->sa_evaluations;
        out->refine_evaluations = r.phases->refine_evaluations;
        out->sa_best_f = r.phases->sa_best_f;
    }
}

template <class Fn>
int32_t guarded(Fn&& fn) {
    try {
        fn();
        return PSA_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PSA_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return PSA_ERR_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return PSA_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PSA_ERR_CUDA;
    }
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int32_t ref_max_threads(void) { return omp_get_max_threads(); }

void ref_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    parsa_ref::detail::Block4x32 b{{ctr[0], ctr[1], ctr[2], ctr[3]}};
    const auto r = parsa_ref::detail::philox4x32_10(b, k0, k1);
    for (int i = 0; i < 4; ++i) out[i] = r.v[i];
}

// draws 0..count-1 of stream (seed, chain, level)
void ref_uniforms(uint64_t seed, uint32_t chain, uint32_t level, int32_t count, double* out) {
    auto s = make_stream({seed, chain, level});
    for (int i = 0; i < count; ++i) out[i] = s.next_uniform();
}

void ref_coordinate_indices(uint64_t seed, uint32_t chain, uint32_t level, int32_t n,
                            int32_t count, int32_t* out) {
    auto s = make_stream({seed, chain, level});
    for (int i = 0; i < count; ++i) out[i] = s.next_coordinate_index(n);
}

int32_t ref_ladder(const psa_schedule* s, double* temps, int32_t capacity, int32_t* levels) {
    return guarded([&] {
        const auto info = ladder({s->t0, s->t_min, s->rho, s->sweep_length});
        *levels = info.levels;
        for (int i = 0; i < info.levels && i < capacity; ++i) temps[i] = info.temperatures[i];
    });
}

int32_t ref_expected_evaluations(const psa_schedule* s, int32_t n_chains, uint64_t* out) {
    return guarded([&] { *out = expected_evaluations({s->t0, s->t_min, s->rho, s->sweep_length}, n_chains); });
}

int32_t ref_evaluate(const psa_objective* o, int32_t precision, const double* x, int32_t count,
                     double* out) {
    return guarded([&] {
        const auto f = make_objective(o);
        for (int i = 0; i < count; ++i) {
            std::vector<double> v(x + std::size_t(i) * o->dim, x + std::size_t(i + 1) * o->dim);
            out[i] = precision == PSA_F32 ? evaluate_single(f, v) : evaluate(f, v);
        }
    });
}

int32_t ref_reduce_min(const double* f, const int32_t* chain, int32_t count, int32_t* pos) {
    return guarded([&] {
        std::vector<Candidate> c;
        for (int i = 0; i < count; ++i) c.push_back({{double(i)}, f[i], chain[i]});
        const auto& w = reduce_min(c);
        *pos = int32_t(w.x[0]);
    });
}

// engine: 0 = v0, 1 = v1, 2 = v2
int32_t ref_run(int32_t engine, const psa_objective* o, const psa_engine_config* c,
                psa_run_result* out) {
    return guarded([&] {
        const auto f = make_objective(o);
        const auto cfg = make_config(o, c);
        RunResult r = engine == 0 ? run_sequential(f, cfg)
                      : engine == 1 ? run_asynchronous(f, cfg)
                                    : run_synchronous(f, cfg);
        fill_result(r, out);
    });
}

int32_t ref_hybrid_run(const psa_objective* o, const psa_engine_config* c, const psa_schedule* t,
                       const psa_nm_config* nm, psa_run_result* out) {
    return guarded([&] {
        const auto f = make_objective(o);
        const auto cfg = make_config(o, c);
        NelderMeadConfig n{nm->reflect, nm->expand, nm->contract, nm->shrink, nm->f_tol, nm->x_tol, nm->max_iters};
        RunResult r = hybrid_run(f, cfg, {t->t0, t->t_min, t->rho, t->sweep_length}, n);
        fill_result(r, out);
    });
}

int32_t ref_nelder_mead(const psa_objective* o, const double* x0, const psa_nm_config* nm,
                        psa_nm_result* out) {
    return guarded([&] {
        const auto f = make_objective(o);
        NelderMeadConfig n{nm->reflect, nm->expand, nm->contract, nm->shrink, nm->f_tol, nm->x_tol, nm->max_iters};
        const auto r = nelder_mead_minimize(f, std::vector<double>(x0, x0 + o->dim), n);
        if (out->x_best) std::memcpy(out->x_best, r.x_best.data(), sizeof(double) * r.x_best.size());
        out->f_best = r.f_best;
        out->iterations = r.iterations;
        out->evaluations = r.evaluations;
    });
}

} // extern "C"
