// Pyramid filter instantiations for k = 3 (compiled as its own TU for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(3, float, float)
SSB_INSTANTIATE_PYR(3, __nv_bfloat16, float)
SSB_INSTANTIATE_PYR(3, double, double)
}  // namespace ssb
