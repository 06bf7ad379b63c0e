// engine_fam_sep_a.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#ifndef PSA_EXPERIMENT_ONLY
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels sep_set<float, Ackley>(int);
template EngineKernels sep_set_generic<float, CosineMixture>(int);
template EngineKernels sep_set_generic<float, Exponential>(int);
template EngineKernels sep_set<double, Ackley>(int);
template EngineKernels sep_set_generic<double, CosineMixture>(int);
template EngineKernels sep_set_generic<double, Exponential>(int);

} // namespace psa
#endif
