// engine_fam_sep_b.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#ifndef PSA_EXPERIMENT_ONLY
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels sep_set<float, Griewank>(int);
template EngineKernels sep_set_generic<float, Michalewicz>(int);
template EngineKernels sep_set<float, Rastrigin>(int);
template EngineKernels sep_set<double, Griewank>(int);
template EngineKernels sep_set_generic<double, Michalewicz>(int);
template EngineKernels sep_set<double, Rastrigin>(int);

} // namespace psa
#endif
