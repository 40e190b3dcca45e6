// Shared device helpers for libssb200 (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

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

// ---- shared-memory logit staging (TMA boxes keep the storage type)
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
// gradient of one logit into the storage type, streaming (written once)
__device__ __forceinline__ void st_gz(float* p, float v, bool acc) {
    if (acc) *p += v;
    else __stcs(p, v);
}
__device__ __forceinline__ void st_gz(__nv_bfloat16* p, float v, bool acc) {
    if (acc) v += __bfloat162float(*p);
    __stcs(reinterpret_cast<unsigned short*>(p), __bfloat16_as_ushort(__float2bfloat16_rn(v)));
}

// ---- packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 / FMUL2, one issue slot
// for two lanes of math; a scalar operand is broadcast by the hardware)
__device__ __forceinline__ unsigned long long f2_bits(float2 a) {
    return (unsigned long long)__float_as_uint(a.x) | ((unsigned long long)__float_as_uint(a.y) << 32);
}
__device__ __forceinline__ float2 bits_f2(unsigned long long d) {
    return make_float2(__uint_as_float((unsigned)d), __uint_as_float((unsigned)(d >> 32)));
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return bits_f2(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return bits_f2(d);
}
__device__ __forceinline__ float2 bcast2(float s) { return make_float2(s, s); }

// max / sum of a per-pixel register array as 4 independent chains (dependency
// depth N/4 + 2 instead of N: the softmax's serial tails)
template <int N>
__device__ __forceinline__ float max4(const float (&e)[N]) {
    float m[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = e[j < N ? j : N - 1];
#pragma unroll
    for (int t = 4; t < N; ++t) m[t & 3] = fmaxf(m[t & 3], e[t]);
    return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}
template <int N>
__device__ __forceinline__ float sum4(const float (&e)[N]) {
    float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < N; ++t) s[t & 3] += e[t];
    return (s[0] + s[1]) + (s[2] + s[3]);
}

// ---- exponentials ---------------------------------------------------------
// fp32: MUFU.EX2 with flush-to-zero (arguments are <= 0 after the max
// subtraction; weights below 2^-126 are irrelevant), the max subtraction folded
// into one FFMA: exp(l - m) = 2^(l*log2e - m*log2e).  fp64: libdevice exp.
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// softmax numerator: `mk` is prep_max(m) for the row max m
__device__ __forceinline__ float prep_max(float m) { return m * kLog2e; }
__device__ __forceinline__ double prep_max(double m) { return m; }
__device__ __forceinline__ float softmax_exp(float l, float mk) { return ex2_ftz(fmaf(l, kLog2e, -mk)); }
__device__ __forceinline__ double softmax_exp(double l, double mk) { return exp(l - mk); }
__device__ __forceinline__ float sexp(float x) { return ex2_ftz(x * kLog2e); }
__device__ __forceinline__ double sexp(double x) { return exp(x); }

// fp32 hot paths divide by reciprocal-multiply (MUFU.RCP, <= 2 ulp; exact for
// the power-of-two pooling counts); fp64 (the parity mode) keeps IEEE division
__device__ __forceinline__ float fdiv(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double fdiv(double a, double b) { return a / b; }
__device__ __forceinline__ float frcp(float b) { return __fdividef(1.0f, b); }
__device__ __forceinline__ double frcp(double b) { return 1.0 / b; }

__device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }

template <typename T>
__device__ __forceinline__ T demod_clamp(T d) { return d > (T)kDemodFloor ? d : (T)kDemodFloor; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and
// device (the attribute lives in the current device's context): `mask` is
// the call site's static, one bit per device; a race only repeats the
// idempotent call
inline void smem_attr_once(std::atomic<unsigned long long>& mask, const void* kern, int bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(mask.load(std::memory_order_relaxed) & bit)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        mask.fetch_or(bit);
    }
}

// launch accounting (pyr_api.cu): every kernel launch is wrapped in
// SSB_LAUNCH(stream, kernel<<<...>>>(...)) so the bench can count launches and
// time individual kernels with CUDA events on their own stream.
void launch_begin(cudaStream_t s);
void launch_end(cudaStream_t s);
void launch_debug_check(cudaStream_t s, const char* what);

}  // namespace ssb

#define SSB_LAUNCH(stream, ...)                    \
    do {                                           \
        ::ssb::launch_begin(stream);               \
        __VA_ARGS__;                               \
        ::ssb::launch_end(stream);                 \
        ::ssb::launch_debug_check(stream, #__VA_ARGS__); \
    } while (0)
