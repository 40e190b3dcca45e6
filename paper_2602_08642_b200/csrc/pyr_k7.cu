// Pyramid filter instantiations for k = 7 (compiled as its own TU for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(7, float, float)
SSB_INSTANTIATE_PYR(7, __nv_bfloat16, float)
SSB_INSTANTIATE_PYR(7, double, double)
}  // namespace ssb
