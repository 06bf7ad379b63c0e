// parsa/objectives.hpp — the cost-function plug-in and the benchmark suite.
//
// B200 drop-in for /root/reference/proj/include/parsa/objectives.hpp:1-73.
// The descriptor keeps the reference's shape (id, name, dim, box, a pair of
// host evaluation pointers, the known optimum) so caller code is unchanged.
//
// What differs is how an engine consumes it.  The reference engines call
// eval_f64/eval_f32 once per Metropolis trial on the CPU.  The B200 engines
// never call a host function per trial: they evaluate a compiled device
// twin of the formula (csrc/objectives.cuh), chosen as follows
// (device_family_of):
//   1. device_family, when the caller sets it explicitly;
//   2. a registry formula, recognised by its eval pointers (this also covers
//      copies with dim and domain overridden, the way the paper's configs
//      reach n = 100 and 500);
//   3. otherwise the host functions are probed: a device formula is bound
//      only if it reproduces both eval_f64 and eval_f32 bit for bit on 64
//      points of the box, and every engine result is then re-checked
//      against the host function (std::logic_error on a mismatch).
// A descriptor that matches no device formula is rejected with
// std::invalid_argument — there is no CPU fallback.  The registry's host
// pointers are real functions (the same glibc-exact templates compiled for
// the host), so f.eval_f64(x, n) and evaluate(f, x) work as before.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

namespace parsa {

// I = [lower_1, upper_1] x ... x [lower_n, upper_n]
struct BoxDomain {
    std::vector<double> lower;
    std::vector<double> upper;

    int dim() const { return static_cast<int>(lower.size()); }
    double width(int k) const { return upper[k] - lower[k]; }
    std::vector<double> center() const; // 0.5 * (lower + upper), per coordinate
};

// The published optimum, for error reporting.  location_at_origin selects
// absolute (instead of relative) location errors; location_known is false
// when no minimiser is published (Michalewicz).
struct ReferenceOptimum {
    double f_star = 0.0;
    std::vector<std::vector<double>> minimizers;
    bool location_known = false;
    bool location_at_origin = false;
};

struct ObjectiveFunction {
    std::string id;
    std::string name;
    int dim = 0;
    BoxDomain domain;
    double (*eval_f64)(const double* x, int n) = nullptr;
    float (*eval_f32)(const float* x, int n) = nullptr;
    ReferenceOptimum reference;
    // B200 addition: psa_family of the device twin (include/parsa_b200.h);
    // -1 = infer from eval_f64 (registry formulas), else explicit.
    int device_family = -1;
    // B200 addition: the family parameter (PSA_FN_CONSTANT's value); set by
    // probing when a host function is bound to the constant family.
    double device_param = 0.0;
};

// l_k <= x_k <= u_k for every k; std::invalid_argument on a size mismatch.
bool contains(const BoxDomain& domain, std::span<const double> x);

// f(x) in double precision (std::invalid_argument on a size mismatch).
double evaluate(const ObjectiveFunction& f, std::span<const double> x);

// f(x) with every coordinate rounded to float and float arithmetic
// throughout, widened back to double.
double evaluate_single(const ObjectiveFunction& f, std::span<const double> x);

// ||x - x*||_2 / ||x*||_2 to the nearest listed minimiser (plain distance
// when the optimum is at the origin); std::invalid_argument when unknown.
double location_error(const ObjectiveFunction& f, std::span<const double> x);

// The 30 x 10 table behind Modified Langerman (first 5 rows) and Modified
// Shekel Foxholes (all rows).
struct FoxholesData {
    int rows;
    int cols;
    const double (*a)[10];
    const double* c;
};
const FoxholesData& foxholes_data();

// The 41 suite entries F0_a ... F19_b, in id order.
const std::vector<ObjectiveFunction>& registry();

// Entry by id; std::out_of_range (listing every valid id) otherwise.
const ObjectiveFunction& registry_get(const std::string& id);

// B200 addition: the device family an engine will run for f, or -1 when f
// has no device twin.  device_binding also reports whether the family was
// found by probing (rule 3 above).
int device_family_of(const ObjectiveFunction& f);
int device_binding(const ObjectiveFunction& f, bool* probed, double* param = nullptr);

} // namespace parsa
