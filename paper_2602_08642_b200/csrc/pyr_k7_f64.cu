// Pyramid filter instantiations for k = 7, f64 logits (one TU per (k, logit
// dtype) for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(7, double, double)
}  // namespace ssb
