// engine_fam_schwefel_f32.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels sep_set<float, Schwefel>(int);

} // namespace psa
