// Pyramid filter instantiations for k = 5, bf16 logits (one TU per (k, logit
// dtype) for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(5, __nv_bfloat16, float)
}  // namespace ssb
