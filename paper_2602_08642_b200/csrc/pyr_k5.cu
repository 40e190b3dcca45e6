// Pyramid filter instantiations for k = 5 (compiled as its own TU for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(5, float, float)
SSB_INSTANTIATE_PYR(5, __nv_bfloat16, float)
SSB_INSTANTIATE_PYR(5, double, double)
}  // namespace ssb
