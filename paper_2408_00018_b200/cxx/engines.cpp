// engines.cpp — parsa:: sa_core / engines / nelder_mead over the C-ABI.
//
// Every function that touches a chain is one C-ABI call into the device
// library (libparsa_b200.so); this file only converts between the
// reference's C++ types (engines.hpp, sa_core.hpp, nelder_mead.hpp) and the
// C structs, and maps psa_status codes back onto the reference's exception
// classes.  Host-only pieces (schedule validation, the ladder, the budget,
// reduce_min) go through the same C-ABI helpers the Python mirror uses, so
// there is one implementation of each.
//
// Reference: sa_core.cpp:8-79, engines.cpp:55-207, nelder_mead.cpp:30-136.
#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "bridge.hpp"
#include "parsa/engines.hpp"
#include "parsa/nelder_mead.hpp"
#include "parsa/sa_core.hpp"

namespace parsa {

// ---- sa_core ---------------------------------------------------------------

void AnnealSchedule::validate() const {
    const psa_schedule c = bridge::schedule_view(*this);
    bridge::check(psa_schedule_validate(&c));
}

LadderInfo ladder(const AnnealSchedule& sched) {
    const psa_schedule c = bridge::schedule_view(sched);
    int32_t levels = 0;
    bridge::check(psa_ladder(&c, nullptr, 0, &levels));
    LadderInfo info;
    info.levels = levels;
    info.temperatures.resize(levels);
    bridge::check(psa_ladder(&c, info.temperatures.data(), levels, &levels));
    return info;
}

std::uint64_t expected_evaluations(const AnnealSchedule& sched, int n_chains) {
    if (n_chains < 1) throw std::invalid_argument("expected_evaluations: need n_chains >= 1");
    const psa_schedule c = bridge::schedule_view(sched);
    std::uint64_t budget = 0;
    bridge::check(psa_expected_evaluations(&c, n_chains, &budget));
    return budget;
}

// sa_core.cpp:37-44 — the two proposal draws, host side (the API hands the
// caller a stream; device sweeps regenerate the same draws in-kernel)
std::vector<double> compute_neighbour(const std::vector<double>& x, const BoxDomain& domain,
                                      UniformStream& stream) {
    std::vector<double> y = x;
    const int d = stream.next_coordinate_index(domain.dim());
    const double u = stream.next_uniform();
    y[d] = domain.lower[d] + u * domain.width(d);
    return y;
}

// sa_core.cpp:46-55 — host form of the rule the device applies in
// metropolis_decide (csrc/engine.cuh); glibc exp/expf here, their bitwise
// restatements there.
bool metropolis_accept(double delta_e, double temperature, UniformStream& stream, Precision prec) {
    const double u = stream.next_uniform();
    if (delta_e <= 0) return true;
    if (prec == Precision::f32) {
        const float arg = -static_cast<float>(delta_e) / static_cast<float>(temperature);
        return static_cast<float>(u) <= std::exp(arg);
    }
    return u <= std::exp(-delta_e / temperature);
}

double chain_energy(const ObjectiveFunction& f, const std::vector<double>& x, Precision prec) {
    return prec == Precision::f32 ? evaluate_single(f, x) : evaluate(f, x);
}

void metropolis_sweep(ChainState& state, const ObjectiveFunction& f, double temperature, int n_steps,
                      Precision prec, std::uint64_t& eval_count) {
    if (n_steps <= 0) return;
    if (state.x.size() != static_cast<std::size_t>(f.dim))
        throw std::invalid_argument("metropolis_sweep: state dimension does not match the objective");
    const bridge::DeviceObjective o = bridge::device_view(f);
    const StreamKey& key = state.stream.key();
    std::uint64_t counter = state.stream.draws();
    bridge::check(psa_metropolis_sweep(&o.c, prec == Precision::f32 ? PSA_F32 : PSA_F64, state.x.data(),
                                       &state.energy, key.master_seed, key.chain_index, key.level_index,
                                       &counter, temperature, n_steps, &eval_count));
    state.stream.set_draws(counter);
}

// ---- engines ---------------------------------------------------------------

const Candidate& reduce_min(const std::vector<Candidate>& candidates) {
    if (candidates.empty()) throw std::invalid_argument("reduce_min: empty candidate list");
    std::vector<double> values(candidates.size());
    std::vector<int32_t> chains(candidates.size());
    for (std::size_t i = 0; i < candidates.size(); ++i) {
        values[i] = candidates[i].f_value;
        chains[i] = candidates[i].chain_index;
    }
    int32_t pos = 0;
    bridge::check(psa_reduce_min(values.data(), chains.data(), static_cast<int32_t>(candidates.size()), &pos));
    return candidates[static_cast<std::size_t>(pos)];
}

namespace {

using EngineEntry = psa_status (*)(const psa_objective*, const psa_engine_config*, psa_run_result*);

RunResult run_on_device(EngineEntry entry, const char* who, const ObjectiveFunction& f, const EngineConfig& cfg) {
    const bridge::DeviceObjective o = bridge::device_view(f);
    const psa_engine_config c = bridge::config_view(cfg);
    bridge::ResultBuffers out(f.dim, bridge::levels_or_zero(cfg.schedule));
    bridge::check(entry(&o.c, &c, &out.c));
    RunResult r = out.to_result();
    bridge::verify(o, f, r.best_x, r.best_f, who);
    return r;
}

} // namespace

RunResult run_sequential(const ObjectiveFunction& f, const EngineConfig& cfg) {
    return run_on_device(psa_run_sequential, "run_sequential", f, cfg);
}

RunResult run_asynchronous(const ObjectiveFunction& f, const EngineConfig& cfg) {
    return run_on_device(psa_run_asynchronous, "run_asynchronous", f, cfg);
}

RunResult run_synchronous(const ObjectiveFunction& f, const EngineConfig& cfg) {
    return run_on_device(psa_run_synchronous, "run_synchronous", f, cfg);
}

// ---- Nelder–Mead -----------------------------------------------------------

void NelderMeadConfig::validate() const {
    if (!(reflect > 0) || !(expand > 1) || !(contract > 0) || !(contract < 1) || !(shrink > 0) || !(shrink < 1))
        throw std::invalid_argument("nelder-mead: coefficient out of range");
}

NelderMeadResult nelder_mead_minimize(const ObjectiveFunction& f, const std::vector<double>& x_start,
                                      const NelderMeadConfig& cfg) {
    cfg.validate();
    if (!contains(f.domain, x_start)) throw std::invalid_argument("nelder_mead_minimize: infeasible start");
    const bridge::DeviceObjective o = bridge::device_view(f);
    const psa_nm_config c = bridge::nm_view(cfg);
    NelderMeadResult r;
    r.x_best.assign(f.dim, 0.0);
    psa_nm_result out{};
    out.x_best = r.x_best.data();
    bridge::check(psa_nelder_mead_minimize(&o.c, x_start.data(), &c, &out));
    r.f_best = out.f_best;
    r.iterations = out.iterations;
    r.evaluations = out.evaluations;
    bridge::verify(o, f, r.x_best, r.f_best, "nelder_mead_minimize");
    return r;
}

RunResult hybrid_run(const ObjectiveFunction& f, const EngineConfig& cfg, const AnnealSchedule& truncated_sched,
                     const NelderMeadConfig& nm_cfg) {
    const bridge::DeviceObjective o = bridge::device_view(f);
    const psa_engine_config c = bridge::config_view(cfg);
    const psa_schedule t = bridge::schedule_view(truncated_sched);
    const psa_nm_config nm = bridge::nm_view(nm_cfg);
    bridge::ResultBuffers out(f.dim, bridge::levels_or_zero(truncated_sched) + 1);
    bridge::check(psa_hybrid_run(&o.c, &c, &t, &nm, &out.c));
    RunResult r = out.to_result();
    bridge::verify(o, f, r.best_x, r.best_f, "hybrid_run");
    return r;
}

} // namespace parsa
