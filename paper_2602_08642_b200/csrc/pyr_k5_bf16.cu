// Pyramid filter instantiations for k = 5, bf16 logits (one TU per (k, logit
// dtype) for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(5, __nv_bfloat16, float)
}  // namespace ssb

#ifdef SSB_ROLE_TIMING
// experiment build only: this TU's counters (tools/role_timing.py)
extern "C" int ssb_debug_role_cycles5b(unsigned long long* out8) { return ssb::role_cycles_read(out8); }
#endif
