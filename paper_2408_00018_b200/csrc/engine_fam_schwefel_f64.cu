// engine_fam_schwefel_f64.cu — explicit instantiations of the engine kernel sets
// (engine_kernels.cuh) for one family group, compiled in parallel with the
// other groups.
#include "engine_kernels.cuh"

namespace psa {

template EngineKernels sep_set<double, Schwefel>(int);

} // namespace psa
