// engine_fam_full.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#ifndef PSA_EXPERIMENT_ONLY
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels full_set<float>(int);
template EngineKernels full_set<double>(int);

} // namespace psa
#endif
