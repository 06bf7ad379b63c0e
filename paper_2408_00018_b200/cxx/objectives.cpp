// objectives.cpp — parsa::ObjectiveFunction plug-in, the 41-entry suite and
// its host evaluation pointers (C++ API layer over the C-ABI).
//
// Host code only: the formula templates of csrc/objectives.cuh (written
// __host__ __device__) are compiled here by g++ with PSA_HD=inline and
// -ffp-contract=off, i.e. the same operations the device runs.  The engines never call these host functions: each registry entry
// is bound to its device family (device_family_of) and the device runs the
// same template.  The host pointers exist because the reference plug-in
// exposes them to callers (objectives.hpp:31-39); being the same
// glibc-exact templates, f.eval_f64(x, n) equals the device's energy bit for
// bit.
//
// Reference: registry assembly objectives.cpp:286-469, helpers :471-551.
#include <algorithm>
#include <cstring>
#include <cmath>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <utility>

#include "objectives.cuh"
#include "parsa/objectives.hpp"
#include "parsa/rng.hpp"
#include "parsa_b200.h"

namespace parsa {
namespace {

using psa::fold;

// f = finish(fold_k term_k(x_k)) in index order — the separable families.
template <class R, template <class> class F>
R host_separable(const R* x, int n) {
    using Fam = F<R>;
    constexpr int A = Fam::kArrays;
    R acc[A];
    for (int a = 0; a < A; ++a) acc[a] = Fam::init(a, n);
    for (int k = 0; k < n; ++k) {
        R t[A];
        Fam::term(x[k], k, t);
        for (int a = 0; a < A; ++a) acc[a] = fold<R>(Fam::op(a), acc[a], t[a]);
    }
    return Fam::finish(acc, n);
}

template <class R>
struct PtrX {
    const R* p;
    R operator()(int k) const { return p[k]; }
};

template <class R, class Formula>
R host_full(const R* x, int n) {
    return Formula::eval(PtrX<R>{x}, n);
}

template <template <class> class F>
struct Sep {
    static double f64(const double* x, int n) { return host_separable<double, F>(x, n); }
    static float f32(const float* x, int n) { return host_separable<float, F>(x, n); }
};

template <template <class> class F>
struct Whole {
    static double f64(const double* x, int n) { return host_full<double, F<double>>(x, n); }
    static float f32(const float* x, int n) { return host_full<float, F<float>>(x, n); }
};

template <int M>
struct ShekelM {
    static double f64(const double* x, int n) { return host_full<double, psa::Shekel<double, M>>(x, n); }
    static float f32(const float* x, int n) { return host_full<float, psa::Shekel<float, M>>(x, n); }
};

struct FamilyEntry {
    double (*f64)(const double*, int);
    float (*f32)(const float*, int);
    int family;
};

// every formula with its device family (include/parsa_b200.h psa_family)
const FamilyEntry kFamilies[] = {
    {Sep<psa::Schwefel>::f64, Sep<psa::Schwefel>::f32, PSA_FN_SCHWEFEL},
    {Sep<psa::Ackley>::f64, Sep<psa::Ackley>::f32, PSA_FN_ACKLEY},
    {Whole<psa::Branin>::f64, Whole<psa::Branin>::f32, PSA_FN_BRANIN},
    {Sep<psa::CosineMixture>::f64, Sep<psa::CosineMixture>::f32, PSA_FN_COSINE_MIXTURE},
    {Whole<psa::DekkersAarts>::f64, Whole<psa::DekkersAarts>::f32, PSA_FN_DEKKERS_AARTS},
    {Whole<psa::Easom>::f64, Whole<psa::Easom>::f32, PSA_FN_EASOM},
    {Sep<psa::Exponential>::f64, Sep<psa::Exponential>::f32, PSA_FN_EXPONENTIAL},
    {Whole<psa::GoldsteinPrice>::f64, Whole<psa::GoldsteinPrice>::f32, PSA_FN_GOLDSTEIN_PRICE},
    {Sep<psa::Griewank>::f64, Sep<psa::Griewank>::f32, PSA_FN_GRIEWANK},
    {Whole<psa::Himmelblau>::f64, Whole<psa::Himmelblau>::f32, PSA_FN_HIMMELBLAU},
    {Whole<psa::LevyMontalvo>::f64, Whole<psa::LevyMontalvo>::f32, PSA_FN_LEVY_MONTALVO},
    {Whole<psa::ModLangerman>::f64, Whole<psa::ModLangerman>::f32, PSA_FN_MOD_LANGERMAN},
    {Sep<psa::Michalewicz>::f64, Sep<psa::Michalewicz>::f32, PSA_FN_MICHALEWICZ},
    {Sep<psa::Rastrigin>::f64, Sep<psa::Rastrigin>::f32, PSA_FN_RASTRIGIN},
    {Whole<psa::Rosenbrock>::f64, Whole<psa::Rosenbrock>::f32, PSA_FN_ROSENBROCK},
    {Sep<psa::Salomon>::f64, Sep<psa::Salomon>::f32, PSA_FN_SALOMON},
    {Whole<psa::SixHumpCamel>::f64, Whole<psa::SixHumpCamel>::f32, PSA_FN_SIX_HUMP_CAMEL},
    {Sep<psa::Shubert>::f64, Sep<psa::Shubert>::f32, PSA_FN_SHUBERT},
    {ShekelM<5>::f64, ShekelM<5>::f32, PSA_FN_SHEKEL5},
    {ShekelM<7>::f64, ShekelM<7>::f32, PSA_FN_SHEKEL7},
    {ShekelM<10>::f64, ShekelM<10>::f32, PSA_FN_SHEKEL10},
    {Whole<psa::ShekelFoxholes>::f64, Whole<psa::ShekelFoxholes>::f32, PSA_FN_SHEKEL_FOXHOLES},
    {Sep<psa::Sphere>::f64, Sep<psa::Sphere>::f32, PSA_FN_SPHERE},
};

const FamilyEntry& entry(int family) {
    for (const auto& e : kFamilies)
        if (e.family == family) return e;
    throw std::logic_error("parsa: unknown device family");
}

constexpr double kPi = 3.141592653589793238462643383279502884;

BoxDomain cube(int n, double lo, double hi) {
    return BoxDomain{std::vector<double>(n, lo), std::vector<double>(n, hi)};
}

ReferenceOptimum origin(int n, double f_star) {
    return ReferenceOptimum{f_star, {std::vector<double>(n, 0.0)}, true, true};
}

ReferenceOptimum points(double f_star, std::vector<std::vector<double>> m) {
    return ReferenceOptimum{f_star, std::move(m), true, false};
}

ReferenceOptimum value(double f_star) { return ReferenceOptimum{f_star, {}, false, false}; }

ObjectiveFunction entry_for(int family, std::string id, std::string name, int dim, BoxDomain box,
                            ReferenceOptimum ref) {
    const FamilyEntry& e = entry(family);
    ObjectiveFunction f;
    f.id = std::move(id);
    f.name = std::move(name);
    f.dim = dim;
    f.domain = std::move(box);
    f.eval_f64 = e.f64;
    f.eval_f32 = e.f32;
    f.reference = std::move(ref);
    return f; // device_family stays -1: inferred from eval_f64, so a caller
              // who swaps the pointer is not silently run as this formula
}

// The suite of the paper's appendix (objectives.cpp:337-469): ids, names,
// dimensions, boxes and published optima.
std::vector<ObjectiveFunction> make_suite() {
    std::vector<ObjectiveFunction> s;
    s.reserve(41);
    const std::pair<const char*, int> schwefel_dims[] = {{"a", 8},   {"b", 16},  {"c", 32}, {"d", 64},
                                                         {"e", 128}, {"f", 256}, {"g", 512}};
    for (const auto& [sfx, n] : schwefel_dims)
        s.push_back(entry_for(PSA_FN_SCHWEFEL, std::string("F0_") + sfx, "Schwefel (normalized)", n,
                              cube(n, -512, 512), points(-418.982887, {std::vector<double>(n, 420.968746)})));
    const std::pair<const char*, int> ackley_dims[] = {{"a", 30}, {"b", 100}, {"c", 200}, {"d", 400}};
    for (const auto& [sfx, n] : ackley_dims)
        s.push_back(entry_for(PSA_FN_ACKLEY, std::string("F1_") + sfx, "Ackley", n, cube(n, -30, 30), origin(n, 0.0)));
    s.push_back(entry_for(PSA_FN_BRANIN, "F2", "Branin", 2, cube(2, -20, 20),
                          points(0.397887, {{-kPi, 12.275}, {kPi, 2.275}, {9.425, 2.475}})));
    s.push_back(entry_for(PSA_FN_COSINE_MIXTURE, "F3_a", "Cosine mixture", 2, cube(2, -1, 1), origin(2, -0.2)));
    s.push_back(entry_for(PSA_FN_COSINE_MIXTURE, "F3_b", "Cosine mixture", 4, cube(4, -1, 1), origin(4, -0.4)));
    s.push_back(entry_for(PSA_FN_DEKKERS_AARTS, "F4", "Dekkers and Aarts", 2, cube(2, -20, 20),
                          points(-24776.518, {{0.0, -14.945}, {0.0, 14.945}})));
    s.push_back(entry_for(PSA_FN_EASOM, "F5", "Easom", 2, cube(2, -10, 10), points(-1.0, {{kPi, kPi}})));
    s.push_back(entry_for(PSA_FN_EXPONENTIAL, "F6", "Exponential", 4, cube(4, -1, 1), origin(4, -1.0)));
    s.push_back(entry_for(PSA_FN_GOLDSTEIN_PRICE, "F7", "Goldstein and Price", 2, cube(2, -2, 2),
                          points(3.0, {{0.0, -1.0}})));
    const std::pair<const char*, int> griewank_dims[] = {{"a", 100}, {"b", 200}, {"c", 400}};
    for (const auto& [sfx, n] : griewank_dims)
        s.push_back(entry_for(PSA_FN_GRIEWANK, std::string("F8_") + sfx, "Griewank", n, cube(n, -600, 600),
                              origin(n, 0.0)));
    s.push_back(entry_for(PSA_FN_HIMMELBLAU, "F9", "Himmelblau", 2, cube(2, -6, 6),
                          points(0.0, {{3.0, 2.0}, {-2.805118, 3.131312}, {-3.779310, -3.283186},
                                       {3.584428, -1.848126}})));
    const std::pair<const char*, int> levy_dims[] = {{"a", 2}, {"b", 5}, {"c", 10}};
    for (const auto& [sfx, n] : levy_dims)
        s.push_back(entry_for(PSA_FN_LEVY_MONTALVO, std::string("F10_") + sfx, "Levy and Montalvo", n,
                              cube(n, -10, 10), points(0.0, {std::vector<double>(n, -1.0)})));
    s.push_back(entry_for(PSA_FN_MOD_LANGERMAN, "F11_a", "Modified Langerman", 2, cube(2, 0, 10),
                          points(-1.080938, {{9.6810707, 0.6666515}})));
    s.push_back(entry_for(PSA_FN_MOD_LANGERMAN, "F11_b", "Modified Langerman", 5, cube(5, 0, 10),
                          points(-0.964999, {{8.074000, 8.777001, 3.467004, 1.863013, 6.707995}})));
    const std::tuple<const char*, int, double> mich[] = {{"a", 2, -1.8013}, {"b", 5, -4.6877}, {"c", 10, -9.6602}};
    for (const auto& [sfx, n, fs] : mich)
        s.push_back(entry_for(PSA_FN_MICHALEWICZ, std::string("F12_") + sfx, "Michalewicz", n, cube(n, 0, kPi),
                              value(fs)));
    s.push_back(entry_for(PSA_FN_RASTRIGIN, "F13_a", "Rastrigin", 100, cube(100, -5.12, 5.12), origin(100, 0.0)));
    s.push_back(entry_for(PSA_FN_RASTRIGIN, "F13_b", "Rastrigin", 400, cube(400, -5.12, 5.12), origin(400, 0.0)));
    s.push_back(entry_for(PSA_FN_ROSENBROCK, "F14", "Generalized Rosenbrock", 4, cube(4, -2.048, 2.048),
                          points(0.0, {{1.0, 1.0, 1.0, 1.0}})));
    s.push_back(entry_for(PSA_FN_SALOMON, "F15", "Salomon", 10, cube(10, -100, 100), origin(10, 0.0)));
    s.push_back(entry_for(PSA_FN_SIX_HUMP_CAMEL, "F16", "Six-Hump Camel Back", 2, BoxDomain{{-3, -2}, {3, 2}},
                          points(-1.0316, {{-0.0898, 0.7126}, {0.0898, -0.7126}})));
    // the 18 minimisers of the n=2 Shubert function (the appendix misprint
    // 4.850 is read as 4.8580, as in the reference)
    s.push_back(entry_for(
        PSA_FN_SHUBERT, "F17", "Shubert", 2, cube(2, -10, 10),
        points(-186.7309, {{-7.0835, 4.8580}, {-7.0835, -7.7083}, {-1.4251, -7.0835}, {5.4828, 4.8580},
                           {-1.4251, -0.8003}, {4.8580, 5.4828},   {-7.7083, -7.0835}, {-7.0835, -1.4251},
                           {-7.7083, -0.8003}, {-7.7083, 5.4828},  {-0.8003, -7.7083}, {-0.8003, -1.4251},
                           {-0.8003, 4.8580},  {-1.4251, 5.4828},  {5.4828, -7.7083},  {4.8580, -7.0835},
                           {5.4828, -1.4251},  {4.8580, -0.8003}})));
    const std::tuple<const char*, int, int, double> shekel[] = {
        {"a", PSA_FN_SHEKEL5, 5, -10.1532}, {"b", PSA_FN_SHEKEL7, 7, -10.4029}, {"c", PSA_FN_SHEKEL10, 10, -10.5364}};
    for (const auto& [sfx, fam, m, fs] : shekel)
        s.push_back(entry_for(fam, std::string("F18_") + sfx, "Shekel " + std::to_string(m), 4, cube(4, 0, 10),
                              points(fs, {{4.0, 4.0, 4.0, 4.0}})));
    s.push_back(entry_for(PSA_FN_SHEKEL_FOXHOLES, "F19_a", "Modified Shekel Foxholes", 2, cube(2, -5, 15),
                          points(-12.1190, {{8.024, 9.146}})));
    s.push_back(entry_for(PSA_FN_SHEKEL_FOXHOLES, "F19_b", "Modified Shekel Foxholes", 5, cube(5, -5, 15),
                          points(-10.4056, {{8.025, 9.152, 5.114, 7.621, 4.564}})));
    return s;
}

void check_size(int want, std::size_t got, const char* who) {
    if (static_cast<std::size_t>(want) == got) return;
    std::ostringstream m;
    m << who << ": expected dimension " << want << ", got " << got;
    throw std::invalid_argument(m.str());
}

} // namespace

std::vector<double> BoxDomain::center() const {
    std::vector<double> mid(lower.size());
    for (std::size_t k = 0; k < mid.size(); ++k) mid[k] = 0.5 * (lower[k] + upper[k]);
    return mid;
}

bool contains(const BoxDomain& domain, std::span<const double> x) {
    check_size(domain.dim(), x.size(), "contains");
    // a NaN coordinate fails neither comparison, as in objectives.cpp:490-496
    for (std::size_t k = 0; k < x.size(); ++k)
        if (x[k] < domain.lower[k] || x[k] > domain.upper[k]) return false;
    return true;
}

double evaluate(const ObjectiveFunction& f, std::span<const double> x) {
    check_size(f.dim, x.size(), "evaluate");
    return f.eval_f64(x.data(), f.dim);
}

double evaluate_single(const ObjectiveFunction& f, std::span<const double> x) {
    check_size(f.dim, x.size(), "evaluate_single");
    thread_local std::vector<float> xf;
    xf.assign(x.begin(), x.end()); // element-wise double -> float rounding
    return static_cast<double>(f.eval_f32(xf.data(), f.dim));
}

double location_error(const ObjectiveFunction& f, std::span<const double> x) {
    check_size(f.dim, x.size(), "location_error");
    if (!f.reference.location_known)
        throw std::invalid_argument("location_error: exact minimizer unknown for " + f.id);
    double nearest = std::numeric_limits<double>::infinity();
    for (const auto& m : f.reference.minimizers) {
        double dist2 = 0, norm2 = 0;
        for (int k = 0; k < f.dim; ++k) {
            const double d = x[k] - m[k];
            dist2 += d * d;
            norm2 += m[k] * m[k];
        }
        const double e = f.reference.location_at_origin ? std::sqrt(dist2) : std::sqrt(dist2) / std::sqrt(norm2);
        nearest = std::min(nearest, e);
    }
    return nearest;
}

const FoxholesData& foxholes_data() {
    static const FoxholesData data{PSA_FOX_ROWS, PSA_FOX_COLS, psa_fox_a, psa_fox_c};
    return data;
}

const std::vector<ObjectiveFunction>& registry() {
    static const std::vector<ObjectiveFunction> suite = make_suite();
    return suite;
}

const ObjectiveFunction& registry_get(const std::string& id) {
    const auto& reg = registry();
    const auto it = std::find_if(reg.begin(), reg.end(), [&](const ObjectiveFunction& f) { return f.id == id; });
    if (it != reg.end()) return *it;
    std::string msg = "unknown function id '" + id + "'; valid ids:";
    for (const auto& f : reg) msg += " " + f.id;
    throw std::out_of_range(msg);
}

namespace {

// Coordinates a formula reads regardless of n (objectives.cpp:43-114,
// 232-284), and the 10-column limit of the Langerman/Foxholes table.
bool family_fits(int family, int n) {
    switch (family) {
    case PSA_FN_BRANIN: case PSA_FN_DEKKERS_AARTS: case PSA_FN_EASOM: case PSA_FN_GOLDSTEIN_PRICE:
    case PSA_FN_HIMMELBLAU: case PSA_FN_SIX_HUMP_CAMEL: return n >= 2;
    case PSA_FN_SHEKEL5: case PSA_FN_SHEKEL7: case PSA_FN_SHEKEL10: return n >= 4;
    case PSA_FN_MOD_LANGERMAN: case PSA_FN_SHEKEL_FOXHOLES: return n <= 10;
    default: return true;
    }
}

template <class T>
bool same_bits(T a, T b) {
    return std::memcmp(&a, &b, sizeof(T)) == 0;
}

// Binding a host function to a device formula by probing.  The reference
// plug-in is an opaque host function pointer (objectives.hpp:31-39) that the
// engines call once per trial; a GPU engine cannot call it.  A descriptor
// that is not a registry formula is therefore matched against every device
// formula on kProbes points of its box (centre, both corners, the rest from
// a fixed Philox stream), in double AND single precision; a formula is
// accepted only if it reproduces the caller's function bit for bit on all
// of them.  Engines re-check every result they return against the host
// function (bridge::verify), so a coincidental match cannot go unnoticed.
constexpr int kProbes = 64;

int probe_family(const ObjectiveFunction& f, double* param) {
    const int n = f.dim;
    if (!f.eval_f64 || !f.eval_f32 || n < 1 || f.domain.dim() != n ||
        static_cast<int>(f.domain.upper.size()) != n)
        return -1;
    std::vector<std::vector<double>> pts;
    pts.reserve(kProbes);
    pts.push_back(f.domain.center());
    pts.push_back(f.domain.lower);
    pts.push_back(f.domain.upper);
    UniformStream u(StreamKey{0x5eed0b1dULL, static_cast<std::uint32_t>(n), 0u});
    while (static_cast<int>(pts.size()) < kProbes) {
        std::vector<double> x(n);
        for (int k = 0; k < n; ++k) x[k] = f.domain.lower[k] + u.next_uniform() * f.domain.width(k);
        pts.push_back(std::move(x));
    }
    std::vector<double> want64(pts.size());
    std::vector<float> want32(pts.size());
    std::vector<std::vector<float>> pts32(pts.size());
    for (std::size_t i = 0; i < pts.size(); ++i) {
        want64[i] = f.eval_f64(pts[i].data(), n);
        pts32[i].assign(pts[i].begin(), pts[i].end());
        want32[i] = f.eval_f32(pts32[i].data(), n);
    }
    // a constant function (the fixtures of test_engines.cpp:91-99 and
    // test_sa_core.cpp:140-160): one value everywhere, the single-precision
    // one its rounding
    bool constant = same_bits(want32[0], static_cast<float>(want64[0]));
    for (std::size_t i = 1; constant && i < pts.size(); ++i)
        constant = same_bits(want64[i], want64[0]) && same_bits(want32[i], want32[0]);
    if (constant) {
        if (param) *param = want64[0];
        return PSA_FN_CONSTANT;
    }
    for (const auto& e : kFamilies) {
        if (!family_fits(e.family, n)) continue;
        bool ok = true;
        for (std::size_t i = 0; ok && i < pts.size(); ++i)
            ok = same_bits(e.f64(pts[i].data(), n), want64[i]) && same_bits(e.f32(pts32[i].data(), n), want32[i]);
        if (ok) return e.family;
    }
    return -1;
}

} // namespace

int device_binding(const ObjectiveFunction& f, bool* probed, double* param) {
    if (probed) *probed = false;
    if (param) *param = f.device_param;
    if (f.device_family >= 0) return f.device_family < PSA_FN_COUNT ? f.device_family : -1;
    for (const auto& e : kFamilies)
        if (f.eval_f64 != nullptr && f.eval_f64 == e.f64 && f.eval_f32 == e.f32)
            return family_fits(e.family, f.dim) ? e.family : -1;
    const int fam = probe_family(f, param);
    if (probed) *probed = fam >= 0;
    return fam;
}

int device_family_of(const ObjectiveFunction& f) { return device_binding(f, nullptr); }

} // namespace parsa
