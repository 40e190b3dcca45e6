// Tonemap + loss epilogue, planar on device:
//   tonemap_array / tonemap_backward  tonemap.py:36-118 (log augment,
//     three-piece filmic curve, sRGB encode; chain rule incl. the saturation
//     mixing Jacobian and the log clamp)
//   spatial_loss / temporal_loss / combined_loss  losses.py:58-91
//   and their gradients as optimize.evaluate_step forms them
//   (optimize.py:219-231): the per-pixel max picks the branch (ties to the
//   spatial term), g_sp = [spatial wins] / N, g_tm = [temporal wins] * 1.25 / N.
// Images (B, 3, H, W); maps (B, H, W); per-frame loss scalars reduced in a
// fixed order (deterministic).  ssb_losses runs maps, sums and gradients in
// one pass; ssb_epilogue fuses tonemap -> losses -> gradient -> tonemap
// backward per pixel.  Compiled with -fmad=false (float64 parity; the float32
// vector kernels use explicit FMAs).
#include <math.h>
#include <string>

#include "common.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

constexpr double kLogFloor = 1e-8;      // tonemap.py:11 LOG_FLOOR
constexpr double kTemporalWeight = 1.25;  // losses.py:14 TEMPORAL_WEIGHT

struct Tmo {
    double exposure, contrast, saturation, toe, shoulder;
};

// float32: MUFU-based log / exp / pow (relative error ~1e-6, inside the fp32
// tolerance); float64: libdevice (the parity mode)
__device__ __forceinline__ float tm_log(float v) { return __logf(v); }
__device__ __forceinline__ double tm_log(double v) { return log(v); }
__device__ __forceinline__ float tm_exp(float v) { return __expf(v); }
__device__ __forceinline__ double tm_exp(double v) { return exp(v); }
__device__ __forceinline__ float tm_pow(float a, float b) { return exp2f(b * __log2f(a)); }
__device__ __forceinline__ double tm_pow(double a, double b) { return pow(a, b); }

template <typename T>
__device__ __forceinline__ T filmic(T x, T toe, T sh) {  // tonemap.py:45-57
    if (x < toe - (T)1) return (T)0.5 * toe * tm_exp(fmin((x + (T)1 - toe) / toe, (T)0));
    if (x >= (T)1 - sh) return (T)1 - (T)0.5 * sh * tm_exp(fmin(-(x + sh - (T)1) / sh, (T)0));
    return (T)0.5 * ((T)1 + x);
}
template <typename T>
__device__ __forceinline__ T filmic_d(T x, T toe, T sh) {  // tonemap.py:60-69
    if (x >= (T)1 - sh) return (T)0.5 * tm_exp(fmin(-(x + sh - (T)1) / sh, (T)0));
    if (x < toe - (T)1) return (T)0.5 * tm_exp(fmin((x + (T)1 - toe) / toe, (T)0));
    return (T)0.5;
}
template <typename T>
__device__ __forceinline__ T srgb(T v) {  // tonemap.py:72-78
    return v <= (T)0.0031308 ? v * (T)12.92 : (T)1.055 * tm_pow(fmax(v, (T)0), (T)1 / (T)2.4) - (T)0.055;
}
template <typename T>
__device__ __forceinline__ T srgb_d(T v) {  // tonemap.py:81-84
    return v <= (T)0.0031308 ? (T)12.92 : ((T)1.055 / (T)2.4) * tm_pow(fmax(v, (T)1e-300), (T)1 / (T)2.4 - (T)1);
}

// log-space augmentation of one pixel: x_c = contrast * (m + sat * (c_c - m) + exposure)
template <typename T>
__device__ __forceinline__ void log_augment(const T rad[3], const Tmo& p, T x[3]) {
    T c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = tm_log(fmax(rad[k], (T)kLogFloor));
    const T m = ((c[0] + c[1]) + c[2]) / (T)3;
#pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = (T)p.contrast * ((m + (T)p.saturation * (c[k] - m)) + (T)p.exposure);
}

template <typename T>
__global__ void k_tonemap(long long n, Tmo p, const T* __restrict__ rad, T* __restrict__ ldr) {
    const int b = blockIdx.y;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const T* r = rad + (long long)b * 3 * n + i;
        T v[3] = {r[0], r[n], r[2 * n]}, x[3];
        log_augment(v, p, x);
#pragma unroll
        for (int k = 0; k < 3; ++k) ldr[(long long)b * 3 * n + k * n + i] = srgb(filmic(x[k], (T)p.toe, (T)p.shoulder));
    }
}

template <typename T>
__global__ void k_tonemap_backward(long long n, Tmo p, const T* __restrict__ rad, const T* __restrict__ up,
                                   T* __restrict__ grad) {
    const int b = blockIdx.y;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long o = (long long)b * 3 * n + i;
        T v[3] = {rad[o], rad[o + n], rad[o + 2 * n]}, x[3], gx[3];
        log_augment(v, p, x);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T y = filmic(x[k], (T)p.toe, (T)p.shoulder);
            gx[k] = up[o + k * n] * srgb_d(y) * filmic_d(x[k], (T)p.toe, (T)p.shoulder);
        }
        const T gs = (gx[0] + gx[1]) + gx[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T gc = (T)p.contrast * ((T)p.saturation * gx[k] + ((T)1 - (T)p.saturation) / (T)3 * gs);
            grad[o + k * n] = v[k] > (T)kLogFloor ? gc / fmax(v[k], (T)kLogFloor) : (T)0;
        }
    }
}

// ---- float32, four pixels per thread (16-B loads / streaming stores):
// branch-free filmic pieces, reciprocals of toe / shoulder precomputed, MUFU
// log2 / exp2 (approx.ftz: relative error ~1e-6, inside the fp32 tolerance;
// inputs are >= the 1e-8 log floor, no denormals), explicit FMAs (the file is
// built with -fmad=false for the float64 parity kernels)
struct TmoF {
    float exposure, contrast, saturation, toe, shoulder, itoe, ish;
};

__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void filmic_f(float x, const TmoF& p, float& y, float& dy) {  // tonemap.py:45-69
    const bool lo = x < p.toe - 1.f, hi = x >= 1.f - p.shoulder;
    const float z = lo ? (x + 1.f - p.toe) * p.itoe : -(x + p.shoulder - 1.f) * p.ish;
    const float e = ex2_ftz(fminf(z, 0.f) * 1.4426950408889634f);
    y = lo ? 0.5f * p.toe * e : (hi ? __fmaf_rn(-0.5f * p.shoulder, e, 1.f) : __fmaf_rn(0.5f, x, 0.5f));
    dy = (lo || hi) ? 0.5f * e : 0.5f;
}

__device__ __forceinline__ void log_augment_f(const float rad[3], const TmoF& p, float x[3]) {
    float c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = lg2_ftz(fmaxf(rad[k], (float)kLogFloor)) * 0.6931471805599453f;
    const float m = ((c[0] + c[1]) + c[2]) * (1.f / 3.f);
#pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = p.contrast * (__fmaf_rn(p.saturation, c[k] - m, m) + p.exposure);
}

__device__ __forceinline__ float srgb_f(float v) {  // tonemap.py:72-78
    return v <= 0.0031308f ? v * 12.92f : __fmaf_rn(1.055f, ex2_ftz(lg2_ftz(v) * (1.f / 2.4f)), -0.055f);
}
__device__ __forceinline__ float srgb_d_f(float v) {  // tonemap.py:81-84
    return v <= 0.0031308f ? 12.92f : (1.055f / 2.4f) * ex2_ftz(lg2_ftz(v) * (1.f / 2.4f - 1.f));
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, const float v[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void unpack4(const float4 v, float o[4]) {
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
}

// n4 = H * W / 4 quads per plane; 32-bit offsets inside a frame (3 n < 2^31)
__global__ void __launch_bounds__(256) k_tonemap_f32v4(unsigned n4, TmoF p, const float* __restrict__ rad,
                                                       float* __restrict__ ldr) {
    const int b = blockIdx.y;
    const unsigned n = 4u * n4;
    const float* rb = rad + (size_t)b * 3 * n;
    float* lb = ldr + (size_t)b * 3 * n;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        float r[3][4], y[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c) unpack4(ld4(rb + c * n + 4 * i), r[c]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float v[3] = {r[0][j], r[1][j], r[2][j]};
            float x[3];
            log_augment_f(v, p, x);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float f, df;
                filmic_f(x[c], p, f, df);
                y[c][j] = srgb_f(f);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) st4(lb + c * n + 4 * i, y[c]);
    }
}

__global__ void __launch_bounds__(256) k_tonemap_backward_f32v4(unsigned n4, TmoF p, const float* __restrict__ rad,
                                                                const float* __restrict__ up,
                                                                float* __restrict__ grad) {
    const int b = blockIdx.y;
    const unsigned n = 4u * n4;
    const size_t fo = (size_t)b * 3 * n;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        float r[3][4], u[3][4], g[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            unpack4(ld4(rad + fo + c * n + 4 * i), r[c]);
            unpack4(ld4(up + fo + c * n + 4 * i), u[c]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float v[3] = {r[0][j], r[1][j], r[2][j]};
            float x[3], gx[3];
            log_augment_f(v, p, x);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float f, df;
                filmic_f(x[c], p, f, df);
                gx[c] = u[c][j] * srgb_d_f(f) * df;
            }
            const float gs = (gx[0] + gx[1]) + gx[2];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float gc = p.contrast * __fmaf_rn(p.saturation, gx[c], (1.f - p.saturation) * (1.f / 3.f) * gs);
                g[c][j] = v[c] > (float)kLogFloor ? __fdividef(gc, v[c]) : 0.f;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) st4(grad + fo + c * n + 4 * i, g[c]);
    }
}

__device__ __forceinline__ double lr_block_sum(double v) {
    __shared__ double sh[8];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    return v;
}

constexpr int kLossBlocks = 512;

// losses[b] = (spatial, temporal, combined) means
__global__ void k_loss_reduce(long long n, int has_temporal, int has_validity, const double* __restrict__ part,
                              double* __restrict__ losses) {
    const int b = blockIdx.x;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < kLossBlocks; k += blockDim.x)
        for (int j = 0; j < 4; ++j) v[j] += part[((long long)b * kLossBlocks + k) * 4 + j];
    for (int j = 0; j < 4; ++j) v[j] = lr_block_sum(v[j]);
    if (threadIdx.x == 0) {
        losses[3 * b + 0] = v[0] / (double)n;
        losses[3 * b + 1] = !has_temporal ? 0.0 : (has_validity ? v[1] / fmax(v[3], 1.0) : v[1] / (double)n);
        losses[3 * b + 2] = v[2] / (double)n;
    }
}

template <typename T>
__device__ __forceinline__ T sgn(T v) { return v > (T)0 ? (T)1 : (v < (T)0 ? (T)-1 : (T)0); }
// x / 3: IEEE division in float64 (bit-exact with numpy); float32 multiplies
// by the rounded reciprocal (<= 1 ulp, inside the fp32 tolerance)
__device__ __forceinline__ double div3(double x) { return x / 3.0; }
__device__ __forceinline__ float div3(float x) { return x * (1.f / 3.f); }

// Per-pixel maps (spatial / temporal / combined, losses.py:58-91),
// per-block partials of their sums (+ the valid count) and the gradients of
// the combined loss w.r.t. ldr1 and the warped ldr0 (optimize.py:219-231) in
// ONE pass over the inputs; V = 4
// pixels per iteration with 16-B loads (float32, n % 4 == 0, aligned planes)
template <typename T, int V>
struct Vec;
template <>
struct Vec<float, 4> {
    static __device__ __forceinline__ void ld(const float* p, float o[4]) { unpack4(ld4(p), o); }
    static __device__ __forceinline__ void st(float* p, const float v[4]) { st4(p, v); }
};
template <typename T>
struct Vec<T, 1> {
    static __device__ __forceinline__ void ld(const T* p, T o[1]) { o[0] = *p; }
    static __device__ __forceinline__ void st(T* p, const T v[1]) { *p = v[0]; }
};

template <typename T, int V>
__global__ void __launch_bounds__(256, 2) k_loss_fused(long long n, const T* __restrict__ out1, const T* __restrict__ ref,
                                                    const T* __restrict__ out0w, const T* __restrict__ refw,
                                                    const T* __restrict__ validity, const T* __restrict__ mask,
                                                    T* sp_map, T* tm_map, T* cb_map, double* part,
                                                    T* __restrict__ g1, T* __restrict__ g0w) {
    using VL = Vec<T, V>;
    const int b = blockIdx.y;
    const T inv_n = (T)1 / (T)n;
    double ssp = 0.0, stm = 0.0, scb = 0.0, scnt = 0.0;
    const long long nv = n / V;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        const long long o = (long long)b * 3 * n + V * i, pm = (long long)b * n + V * i;
        T a1[3][V], rf[3][V], a0[3][V], rw[3][V], val[V], w[V];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            VL::ld(out1 + o + k * n, a1[k]);
            VL::ld(ref + o + k * n, rf[k]);
            if (out0w) {
                VL::ld(out0w + o + k * n, a0[k]);
                VL::ld(refw + o + k * n, rw[k]);
            }
        }
        if (validity) VL::ld(validity + pm, val);
        if (mask) VL::ld(mask + pm, w);
        else
#pragma unroll
            for (int j = 0; j < V; ++j) w[j] = (T)1;
        T spv[V], tmv[V], cbv[V], cs[V], ct[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            T sp = (T)0, tm = (T)0;
#pragma unroll
            for (int k = 0; k < 3; ++k) sp = sp + fabs(a1[k][j] - rf[k][j]);
            sp = div3(sp) * w[j];
            if (out0w) {
#pragma unroll
                for (int k = 0; k < 3; ++k) tm = tm + fabs((a1[k][j] - a0[k][j]) - (rf[k][j] - rw[k][j]));
                tm = div3(tm);
                if (validity) {
                    const bool valid = val[j] >= (T)1;
                    tm = valid ? tm : (T)0;
                    scnt += valid ? 1.0 : 0.0;
                }
            }
            const T cb = fmax((T)kTemporalWeight * tm, sp);
            spv[j] = sp;
            tmv[j] = tm;
            cbv[j] = cb;
            ssp += (double)sp;
            stm += (double)tm;
            scb += (double)cb;
            // optimize.py:219-231 (ties to the spatial term); s * x / 3 ==
            // s * (x / 3) exactly for a sign s, so the /3 is hoisted
            const bool twins = (T)kTemporalWeight * tm > sp;
            const T gsp = twins ? (T)0 : inv_n, gtm = twins ? (T)kTemporalWeight / (T)n : (T)0;
            cs[j] = div3(gsp * w[j]);
            ct[j] = div3(gtm);
        }
        if (sp_map) VL::st(sp_map + pm, spv);
        if (tm_map) VL::st(tm_map + pm, tmv);
        if (cb_map) VL::st(cb_map + pm, cbv);
        if (g1) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T gv1[V], gv0[V];
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    T v = sgn(a1[k][j] - rf[k][j]) * cs[j];
                    if (out0w) {
                        const T st = sgn((a1[k][j] - a0[k][j]) - (rf[k][j] - rw[k][j]));
                        v = v + st * ct[j];
                        gv0[j] = -st * ct[j];
                    }
                    gv1[j] = v;
                }
                VL::st(g1 + o + k * n, gv1);
                if (g0w) VL::st(g0w + o + k * n, gv0);
            }
        }
    }
    // (reduced unconditionally: a shuffle under a branch the compiler cannot
    // prove uniform is emulated per active subset)
    ssp = lr_block_sum(ssp);
    stm = lr_block_sum(stm);
    scb = lr_block_sum(scb);
    scnt = lr_block_sum(scnt);
    {
        if (part && threadIdx.x == 0) {
            double* q = part + ((long long)b * kLossBlocks + blockIdx.x) * 4;
            q[0] = ssp;
            q[1] = stm;
            q[2] = scb;
            q[3] = scnt;
        }
    }
}

// The whole evaluate_step epilogue in ONE pass (optimize.py:219-231 with
// tonemap.py:36-118): tonemap the radiance, the three losses against the
// reference (+ the warped history), their gradient w.r.t. the LDR frame, and
// its chain through the tonemap to the radiance -- per pixel, so nothing but
// the inputs and the two gradients (and optionally the LDR frame) touches
// HBM.  float64 evaluates exactly the expressions of k_tonemap, k_loss_fused
// and k_tonemap_backward (bit-identical to the three-launch composition);
// float32 uses the fast pieces of the vector kernels.
template <typename T, int V>
__global__ void __launch_bounds__(256, 2) k_epilogue(long long n, Tmo p, TmoF pf, const T* __restrict__ rad,
                                                     const T* __restrict__ ref, const T* __restrict__ out0w,
                                                     const T* __restrict__ refw, const T* __restrict__ validity,
                                                     const T* __restrict__ mask, T* __restrict__ ldr_out,
                                                     double* part, T* __restrict__ grad, T* __restrict__ g0w) {
    using VL = Vec<T, V>;
    constexpr bool F32 = sizeof(T) == 4;
    const int b = blockIdx.y;
    const T inv_n = (T)1 / (T)n;
    double ssp = 0.0, stm = 0.0, scb = 0.0, scnt = 0.0;
    const long long nv = n / V;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        const long long o = (long long)b * 3 * n + V * i, pm = (long long)b * n + V * i;
        T rv[3][V], rf[3][V], a0[3][V], rw[3][V], val[V], w[V];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            VL::ld(rad + o + k * n, rv[k]);
            VL::ld(ref + o + k * n, rf[k]);
            if (out0w) {
                VL::ld(out0w + o + k * n, a0[k]);
                VL::ld(refw + o + k * n, rw[k]);
            }
        }
        if (validity) VL::ld(validity + pm, val);
        if (mask) VL::ld(mask + pm, w);
        else
#pragma unroll
            for (int j = 0; j < V; ++j) w[j] = (T)1;
        T a1[3][V], dfy[3][V], gout[3][V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            // tonemap (k_tonemap): x, filmic y, ldr = srgb(y); keep d ldr / dx
            const T v[3] = {rv[0][j], rv[1][j], rv[2][j]};
            T x[3];
            if constexpr (F32) log_augment_f(v, pf, x);
            else log_augment(v, p, x);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if constexpr (F32) {
                    float f, df;
                    filmic_f(x[k], pf, f, df);
                    a1[k][j] = srgb_f(f);
                    dfy[k][j] = srgb_d_f(f) * df;
                } else {
                    const T y = filmic(x[k], (T)p.toe, (T)p.shoulder);
                    a1[k][j] = srgb(y);
                    dfy[k][j] = srgb_d(y);  // (times filmic_d below, in k_tonemap_backward's order)
                }
            }
            // losses + their LDR gradient (k_loss_fused)
            T sp = (T)0, tm = (T)0;
#pragma unroll
            for (int k = 0; k < 3; ++k) sp = sp + fabs(a1[k][j] - rf[k][j]);
            sp = div3(sp) * w[j];
            if (out0w) {
#pragma unroll
                for (int k = 0; k < 3; ++k) tm = tm + fabs((a1[k][j] - a0[k][j]) - (rf[k][j] - rw[k][j]));
                tm = div3(tm);
                if (validity) {
                    const bool valid = val[j] >= (T)1;
                    tm = valid ? tm : (T)0;
                    scnt += valid ? 1.0 : 0.0;
                }
            }
            const T cb = fmax((T)kTemporalWeight * tm, sp);
            ssp += (double)sp;
            stm += (double)tm;
            scb += (double)cb;
            const bool twins = (T)kTemporalWeight * tm > sp;
            const T gsp = twins ? (T)0 : inv_n, gtm = twins ? (T)kTemporalWeight / (T)n : (T)0;
            const T cs = div3(gsp * w[j]), ct = div3(gtm);
            T gx[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T g1 = sgn(a1[k][j] - rf[k][j]) * cs;
                if (out0w) {
                    const T st = sgn((a1[k][j] - a0[k][j]) - (rf[k][j] - rw[k][j]));
                    g1 = g1 + st * ct;
                    gout[k][j] = -st * ct;
                }
                // tonemap backward (k_tonemap_backward)
                if constexpr (F32) gx[k] = g1 * dfy[k][j];
                else gx[k] = g1 * dfy[k][j] * filmic_d(x[k], (T)p.toe, (T)p.shoulder);
            }
            const T gs = (gx[0] + gx[1]) + gx[2];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if constexpr (F32) {
                    const float gc = pf.contrast * __fmaf_rn(pf.saturation, gx[k], (1.f - pf.saturation) * (1.f / 3.f) * gs);
                    dfy[k][j] = v[k] > (float)kLogFloor ? __fdividef(gc, v[k]) : 0.f;
                } else {
                    const T gc = (T)p.contrast * ((T)p.saturation * gx[k] + ((T)1 - (T)p.saturation) / (T)3 * gs);
                    dfy[k][j] = v[k] > (T)kLogFloor ? gc / fmax(v[k], (T)kLogFloor) : (T)0;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            VL::st(grad + o + k * n, dfy[k]);
            if (g0w) VL::st(g0w + o + k * n, gout[k]);
            if (ldr_out) VL::st(ldr_out + o + k * n, a1[k]);
        }
    }
    ssp = lr_block_sum(ssp);
    stm = lr_block_sum(stm);
    scb = lr_block_sum(scb);
    scnt = lr_block_sum(scnt);
    if (part && threadIdx.x == 0) {
        double* q = part + ((long long)b * kLossBlocks + blockIdx.x) * 4;
        q[0] = ssp;
        q[1] = stm;
        q[2] = scb;
        q[3] = scnt;
    }
}

template <typename T>
dim3 grid_for(long long n, int B) {
    long long g = (n + 255) / 256;
    return dim3((unsigned)(g < 2048 ? g : 2048), B);
}

}  // namespace ssb

using namespace ssb;

extern "C" {

static TmoF tmo_f(const Tmo& p) {
    return TmoF{(float)p.exposure, (float)p.contrast, (float)p.saturation, (float)p.toe, (float)p.shoulder,
                (float)(1.0 / p.toe), (float)(1.0 / p.shoulder)};
}

// the float32 vector kernels: whole quads per plane, 16-B aligned planes,
// 32-bit offsets inside a frame
static bool vec4_ok(long long n, int B, const void* a, const void* b = nullptr, const void* c = nullptr,
                    const void* d = nullptr, const void* e = nullptr, const void* f = nullptr,
                    const void* g = nullptr, const void* h = nullptr, const void* i = nullptr,
                    const void* j = nullptr) {
    (void)B;
    if (n % 4 != 0 || 3 * n >= (1ll << 31)) return false;
    for (const void* q : {a, b, c, d, e, f, g, h, i, j})
        if (q && (reinterpret_cast<size_t>(q) & 15)) return false;
    return true;
}

static int tmo_check(const double* tmo, Tmo* p) {
    if (!tmo) return SSB_EINVAL;
    *p = Tmo{tmo[0], tmo[1], tmo[2], tmo[3], tmo[4]};
    if (!(p->contrast > 0) || !(p->saturation > 0) || !(p->toe > 0 && p->toe < 1) ||
        !(p->shoulder > 0 && p->shoulder < 1))
        return SSB_EINVAL;
    return 0;
}

int ssb_tonemap(int dtype, int B, int H, int W, const double* tmo, const void* radiance, void* ldr,
                ssb_stream_t stream) {
    Tmo p;
    if (B <= 0 || H <= 0 || W <= 0 || !radiance || !ldr || tmo_check(tmo, &p)) {
        set_error("ssb_tonemap: invalid arguments (contrast, saturation > 0; toe, shoulder in (0, 1))");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)H * W;
    if (dtype == SSB_F64) SSB_LAUNCH(s, k_tonemap<double><<<grid_for<double>(n, B), 256, 0, s>>>(n, p, (const double*)radiance, (double*)ldr));
    else if (dtype == SSB_F32 && vec4_ok(n, B, radiance, ldr))
        SSB_LAUNCH(s, k_tonemap_f32v4<<<grid_for<float>(n / 4, B), 256, 0, s>>>((unsigned)(n / 4), tmo_f(p),
                                                                               (const float*)radiance, (float*)ldr));
    else if (dtype == SSB_F32) SSB_LAUNCH(s, k_tonemap<float><<<grid_for<float>(n, B), 256, 0, s>>>(n, p, (const float*)radiance, (float*)ldr));
    else {
        set_error("ssb_tonemap: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    return cuda_check("ssb_tonemap");
}

int ssb_tonemap_backward(int dtype, int B, int H, int W, const double* tmo, const void* radiance,
                         const void* upstream, void* grad, ssb_stream_t stream) {
    Tmo p;
    if (B <= 0 || H <= 0 || W <= 0 || !radiance || !upstream || !grad || tmo_check(tmo, &p)) {
        set_error("ssb_tonemap_backward: invalid arguments");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)H * W;
    if (dtype == SSB_F64)
        SSB_LAUNCH(s, k_tonemap_backward<double><<<grid_for<double>(n, B), 256, 0, s>>>(
                          n, p, (const double*)radiance, (const double*)upstream, (double*)grad));
    else if (dtype == SSB_F32 && vec4_ok(n, B, radiance, upstream, grad))
        SSB_LAUNCH(s, k_tonemap_backward_f32v4<<<grid_for<float>(n / 4, B), 256, 0, s>>>(
                          (unsigned)(n / 4), tmo_f(p), (const float*)radiance, (const float*)upstream, (float*)grad));
    else if (dtype == SSB_F32)
        SSB_LAUNCH(s, k_tonemap_backward<float><<<grid_for<float>(n, B), 256, 0, s>>>(
                          n, p, (const float*)radiance, (const float*)upstream, (float*)grad));
    else {
        set_error("ssb_tonemap_backward: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    return cuda_check("ssb_tonemap_backward");
}

int ssb_losses_workspace_bytes(int B, size_t* bytes) {
    if (B <= 0 || !bytes) {
        set_error("ssb_losses_workspace_bytes: invalid arguments");
        return SSB_EINVAL;
    }
    *bytes = (size_t)B * kLossBlocks * 4 * sizeof(double);
    return 0;
}

int ssb_losses(int dtype, int B, int H, int W, const void* ldr1, const void* ref, const void* ldr0_w,
               const void* ref_w, const void* validity, const void* mask, void* sp_map, void* tm_map,
               void* cb_map, double* losses, void* g_ldr1, void* g_ldr0_w, void* workspace,
               ssb_stream_t stream) {
    if (B <= 0 || H <= 0 || W <= 0 || !ldr1 || !ref || (!ldr0_w) != (!ref_w) || (validity && !ldr0_w) ||
        (losses && !workspace) || (g_ldr0_w && !ldr0_w)) {
        set_error("ssb_losses: invalid arguments");
        return SSB_EINVAL;
    }
    if (dtype != SSB_F32 && dtype != SSB_F64) {
        set_error("ssb_losses: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)H * W;
    const bool sums = losses != nullptr;
    auto run = [&](auto tag) {
        using T = decltype(tag);
        if (!(sums || sp_map || tm_map || cb_map || g_ldr1)) return;
        const bool v4 = sizeof(T) == 4 && vec4_ok(n, B, ldr1, ref, ldr0_w, ref_w, validity, mask, sp_map, tm_map,
                                                   cb_map, g_ldr1) &&
                        vec4_ok(n, B, g_ldr0_w);
        auto kern = v4 ? k_loss_fused<T, sizeof(T) == 4 ? 4 : 1> : k_loss_fused<T, 1>;
        SSB_LAUNCH(s, kern<<<dim3(kLossBlocks, B), 256, 0, s>>>(
                          n, (const T*)ldr1, (const T*)ref, (const T*)ldr0_w, (const T*)ref_w, (const T*)validity,
                          (const T*)mask, (T*)sp_map, (T*)tm_map, (T*)cb_map, sums ? (double*)workspace : nullptr,
                          (T*)g_ldr1, (T*)g_ldr0_w));
        if (sums)
            SSB_LAUNCH(s, k_loss_reduce<<<B, 256, 0, s>>>(n, ldr0_w != nullptr, validity != nullptr,
                                                          (const double*)workspace, losses));
    };
    if (dtype == SSB_F64) run(0.0);
    else run(0.0f);
    return cuda_check("ssb_losses");
}

int ssb_epilogue(int dtype, int B, int H, int W, const double* tmo, const void* radiance, const void* ref,
                 const void* ldr0_w, const void* ref_w, const void* validity, const void* mask, void* ldr,
                 double* losses, void* grad_radiance, void* g_ldr0_w, void* workspace, ssb_stream_t stream) {
    Tmo p;
    if (B <= 0 || H <= 0 || W <= 0 || !radiance || !ref || !grad_radiance || (!ldr0_w) != (!ref_w) ||
        (validity && !ldr0_w) || (losses && !workspace) || (g_ldr0_w && !ldr0_w) || tmo_check(tmo, &p)) {
        set_error("ssb_epilogue: invalid arguments");
        return SSB_EINVAL;
    }
    if (dtype != SSB_F32 && dtype != SSB_F64) {
        set_error("ssb_epilogue: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)H * W;
    auto run = [&](auto tag) {
        using T = decltype(tag);
        const bool v4 = sizeof(T) == 4 && vec4_ok(n, B, radiance, ref, ldr0_w, ref_w, validity, mask, ldr,
                                                   grad_radiance, g_ldr0_w);
        auto kern = v4 ? k_epilogue<T, sizeof(T) == 4 ? 4 : 1> : k_epilogue<T, 1>;
        SSB_LAUNCH(s, kern<<<dim3(kLossBlocks, B), 256, 0, s>>>(
                          n, p, tmo_f(p), (const T*)radiance, (const T*)ref, (const T*)ldr0_w, (const T*)ref_w,
                          (const T*)validity, (const T*)mask, (T*)ldr, losses ? (double*)workspace : nullptr,
                          (T*)grad_radiance, (T*)g_ldr0_w));
        if (losses)
            SSB_LAUNCH(s, k_loss_reduce<<<B, 256, 0, s>>>(n, ldr0_w != nullptr, validity != nullptr,
                                                          (const double*)workspace, losses));
    };
    if (dtype == SSB_F64) run(0.0);
    else run(0.0f);
    return cuda_check("ssb_epilogue");
}

}  // extern "C"
