// Shared device helpers for libssb200 (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssb_api.h"

namespace ssb {

constexpr double kDemodFloor = 1e-3;  // pyramid.py:28 DEMOD_FLOOR

__host__ __device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// ---- logit storage -> compute type -------------------------------------
template <typename T>
__device__ __forceinline__ T ld_logit(const float* p) { return (T)__ldcs(p); }
template <typename T>
__device__ __forceinline__ T ld_logit(const double* p) { return (T)__ldcs(p); }
template <typename T>
__device__ __forceinline__ T ld_logit(const __nv_bfloat16* p) {
    unsigned short raw = __ldcs(reinterpret_cast<const unsigned short*>(p));
    return (T)__uint_as_float(((unsigned int)raw) << 16);
}

// ---- gradient store into the logit storage type --------------------------
__device__ __forceinline__ void st_glogit(float* p, float v, bool acc) {
    if (acc) v += *p;
    __stcs(p, v);
}
__device__ __forceinline__ void st_glogit(double* p, double v, bool acc) {
    if (acc) v += *p;
    __stcs(p, v);
}
__device__ __forceinline__ void st_glogit(__nv_bfloat16* p, float v, bool acc) {
    if (acc) v += __bfloat162float(*p);
    *p = __float2bfloat16_rn(v);
}

// ---- exponentials ---------------------------------------------------------
// fp32: MUFU.EX2-based fast exp (arguments are <= 0 after max subtraction, so
// the relative error is a few ulp where the weight matters); fp64: libdevice.
__device__ __forceinline__ float sexp(float x) { return __expf(x); }
__device__ __forceinline__ double sexp(double x) { return exp(x); }

template <typename T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }

template <typename T>
__device__ __forceinline__ T demod_clamp(T d) { return d > (T)kDemodFloor ? d : (T)kDemodFloor; }

// launch accounting (pyr_api.cu): every kernel launch is wrapped in
// SSB_LAUNCH(stream, kernel<<<...>>>(...)) so the bench can count launches and
// time individual kernels with CUDA events on their own stream.
void launch_begin(cudaStream_t s);
void launch_end(cudaStream_t s);

}  // namespace ssb

#define SSB_LAUNCH(stream, ...)          \
    do {                                 \
        ::ssb::launch_begin(stream);     \
        __VA_ARGS__;                     \
        ::ssb::launch_end(stream);       \
    } while (0)
