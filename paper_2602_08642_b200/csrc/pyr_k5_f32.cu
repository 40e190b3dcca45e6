// Pyramid filter instantiations for k = 5, f32 logits (one TU per (k, logit
// dtype) for build parallelism).
#include "pyr_launch.cuh"

namespace ssb {
SSB_INSTANTIATE_PYR(5, float, float)
}  // namespace ssb

#ifdef SSB_ROLE_TIMING
// experiment build only (not in ssb_api.h): read and reset this TU's
// backward-kernel per-role cycle counters (tools/role_timing.py)
extern "C" int ssb_debug_role_cycles5(unsigned long long* out8) { return ssb::role_cycles_read(out8); }
#endif
