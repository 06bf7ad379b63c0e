// bridge.hpp — internal glue between the parsa:: C++ API and the C-ABI.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "parsa/engines.hpp"
#include "parsa/nelder_mead.hpp"
#include "parsa_b200.h"

namespace parsa::bridge {

// psa_status -> the reference's exception class, with the C-ABI's message
// (which is the reference's exact text for every reference-defined error).
[[noreturn]] inline void raise(psa_status st) {
    const std::string msg = psa_last_error();
    switch (st) {
    case PSA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PSA_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case PSA_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
    }
}

inline void check(psa_status st) {
    if (st != PSA_OK) raise(st);
}

// The device view of an objective.  Holds pointers into `f`, which must
// outlive it.  family = -1 when f has no device twin; the C-ABI then
// rejects it at the point where the reference would first evaluate it.
struct DeviceObjective {
    psa_objective c{};
    bool probed = false; // bound by probing the host functions (objectives.hpp rule 3)
};

inline DeviceObjective device_view(const ObjectiveFunction& f) {
    DeviceObjective o;
    o.c.id = f.id.c_str();
    o.c.family = device_binding(f, &o.probed, &o.c.param);
    o.c.dim = f.dim;
    o.c.lower = f.domain.lower.data();
    o.c.upper = f.domain.upper.data();
    return o;
}

// For a probed binding: the value the device reports at x must be the host
// function's own value there (double or single precision path).
inline void verify(const DeviceObjective& o, const ObjectiveFunction& f, const std::vector<double>& x, double fx,
                   const char* who) {
    if (!o.probed || x.size() != static_cast<std::size_t>(f.dim)) return;
    const double a = evaluate(f, x), b = evaluate_single(f, x);
    const auto same = [](double p, double q) { return std::memcmp(&p, &q, sizeof p) == 0; };
    if (!same(a, fx) && !same(b, fx))
        throw std::logic_error(std::string(who) + ": the device formula bound to '" + f.id +
                               "' disagrees with its host function at the returned point");
}

inline psa_schedule schedule_view(const AnnealSchedule& s) {
    psa_schedule c{};
    c.t0 = s.t0;
    c.t_min = s.t_min;
    c.rho = s.rho;
    c.sweep_length = s.sweep_length;
    return c;
}

inline psa_engine_config config_view(const EngineConfig& cfg) {
    psa_engine_config c{};
    c.n_chains = cfg.n_chains;
    c.start_mode = cfg.start_mode == StartMode::random_per_chain ? PSA_RANDOM_PER_CHAIN : PSA_SHARED_POINT;
    c.start_point = cfg.start_point.empty() ? nullptr : cfg.start_point.data();
    c.start_point_len = static_cast<int32_t>(cfg.start_point.size());
    c.precision = cfg.precision == Precision::f32 ? PSA_F32 : PSA_F64;
    c.seed = cfg.seed;
    c.workers = cfg.workers;
    c.schedule = schedule_view(cfg.schedule);
    return c;
}

inline psa_nm_config nm_view(const NelderMeadConfig& nm) {
    psa_nm_config c{};
    c.reflect = nm.reflect;
    c.expand = nm.expand;
    c.contract = nm.contract;
    c.shrink = nm.shrink;
    c.f_tol = nm.f_tol;
    c.x_tol = nm.x_tol;
    c.max_iters = nm.max_iters;
    return c;
}

// Caller-owned result buffers sized for `trace_rows` rows.
struct ResultBuffers {
    std::vector<double> best_x;
    std::vector<psa_trace_point> trace;
    psa_run_result c{};

    ResultBuffers(int dim, int trace_rows) : best_x(dim > 0 ? dim : 0), trace(trace_rows > 0 ? trace_rows : 0) {
        c.best_x = best_x.data();
        c.trace = trace.data();
        c.trace_capacity = static_cast<int32_t>(trace.size());
    }

    RunResult to_result() const {
        RunResult r;
        r.best_x = best_x;
        r.best_f = c.best_f;
        r.evaluations = c.evaluations;
        r.wall_time_s = c.wall_time_s;
        r.winning_chain = c.winning_chain;
        r.rng_draws = c.rng_draws;
        const int rows = c.trace_len < c.trace_capacity ? c.trace_len : c.trace_capacity;
        r.trace.reserve(rows);
        for (int i = 0; i < rows; ++i) r.trace.push_back(TracePoint{trace[i].level, trace[i].cumulative_evals, trace[i].best_f});
        if (c.has_phases) r.phases = PhaseBreakdown{c.sa_evaluations, c.refine_evaluations, c.sa_best_f};
        return r;
    }
};

// Number of ladder levels for a schedule that may be invalid: 0 lets the
// engine entry point report the schedule error in the reference's order.
inline int levels_or_zero(const AnnealSchedule& s) {
    const psa_schedule c = schedule_view(s);
    int32_t levels = 0;
    if (psa_ladder(&c, nullptr, 0, &levels) != PSA_OK) return 0;
    return levels;
}

} // namespace parsa::bridge
