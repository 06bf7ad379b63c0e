// engine_fam_sep_c.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#ifndef PSA_EXPERIMENT_ONLY
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels sep_set_generic<float, Salomon>(int);
template EngineKernels sep_set_generic<float, Shubert>(int);
template EngineKernels sep_set_generic<float, Sphere>(int);
template EngineKernels sep_set_generic<double, Salomon>(int);
template EngineKernels sep_set_generic<double, Shubert>(int);
template EngineKernels sep_set_generic<double, Sphere>(int);

} // namespace psa
#endif
