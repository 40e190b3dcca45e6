// Tonemap + loss epilogue, planar on device:
//   tonemap_array / tonemap_backward  tonemap.py:36-118 (log augment,
//     three-piece filmic curve, sRGB encode; chain rule incl. the saturation
//     mixing Jacobian and the log clamp)
//   spatial_loss / temporal_loss / combined_loss  losses.py:58-91
//   and their gradients as optimize.evaluate_step forms them
//   (optimize.py:219-231): the per-pixel max picks the branch (ties to the
//   spatial term), g_sp = [spatial wins] / N, g_tm = [temporal wins] * 1.25 / N.
// Images (B, 3, H, W); maps (B, H, W); per-frame loss scalars reduced in a
// fixed order (deterministic).  Compiled with -fmad=false.
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

// per-pixel maps (spatial / temporal / combined) and per-block partials of
// their sums (+ the valid count): losses.py:58-91
template <typename T>
__global__ void __launch_bounds__(256) k_loss_maps(long long n, const T* __restrict__ out1, const T* __restrict__ ref,
                                                   const T* __restrict__ out0w, const T* __restrict__ refw,
                                                   const T* __restrict__ validity, const T* __restrict__ mask,
                                                   T* sp_map, T* tm_map, T* cb_map, double* part) {
    const int b = blockIdx.y;
    double ssp = 0.0, stm = 0.0, scb = 0.0, scnt = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long o = (long long)b * 3 * n + i, pm = (long long)b * n + i;
        T sp = (T)0, tm = (T)0;
#pragma unroll
        for (int k = 0; k < 3; ++k) sp = sp + fabs(out1[o + k * n] - ref[o + k * n]);
        sp = sp / (T)3 * (mask ? mask[pm] : (T)1);
        if (out0w) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                tm = tm + fabs((out1[o + k * n] - out0w[o + k * n]) - (ref[o + k * n] - refw[o + k * n]));
            tm = tm / (T)3;
            if (validity) {
                const bool valid = validity[pm] >= (T)1;
                tm = valid ? tm : (T)0;
                scnt += valid ? 1.0 : 0.0;
            }
        }
        const T cb = fmax((T)kTemporalWeight * tm, sp);
        if (sp_map) sp_map[pm] = sp;
        if (tm_map) tm_map[pm] = tm;
        if (cb_map) cb_map[pm] = cb;
        ssp += (double)sp;
        stm += (double)tm;
        scb += (double)cb;
    }
    ssp = lr_block_sum(ssp);
    stm = lr_block_sum(stm);
    scb = lr_block_sum(scb);
    scnt = lr_block_sum(scnt);
    if (threadIdx.x == 0) {
        double* q = part + ((long long)b * kLossBlocks + blockIdx.x) * 4;
        q[0] = ssp;
        q[1] = stm;
        q[2] = scb;
        q[3] = scnt;
    }
}

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

// gradients of the combined loss w.r.t. ldr1 and the warped ldr0
// (optimize.py:219-231)
template <typename T>
__global__ void k_loss_grads(long long n, const T* __restrict__ out1, const T* __restrict__ ref,
                             const T* __restrict__ out0w, const T* __restrict__ refw,
                             const T* __restrict__ validity, const T* __restrict__ mask, T* __restrict__ g1,
                             T* __restrict__ g0w) {
    const int b = blockIdx.y;
    const T inv_n = (T)1 / (T)n;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long o = (long long)b * 3 * n + i, pm = (long long)b * n + i;
        const T w = mask ? mask[pm] : (T)1;
        T sp = (T)0, tm = (T)0;
#pragma unroll
        for (int k = 0; k < 3; ++k) sp = sp + fabs(out1[o + k * n] - ref[o + k * n]);
        sp = sp / (T)3 * w;
        if (out0w) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                tm = tm + fabs((out1[o + k * n] - out0w[o + k * n]) - (ref[o + k * n] - refw[o + k * n]));
            tm = tm / (T)3;
            if (validity && !(validity[pm] >= (T)1)) tm = (T)0;
        }
        const bool twins = (T)kTemporalWeight * tm > sp;  // ties to the spatial term
        const T gsp = twins ? (T)0 : inv_n, gtm = twins ? (T)kTemporalWeight / (T)n : (T)0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const T s1 = sgn(out1[o + k * n] - ref[o + k * n]);
            T v = s1 * (gsp * w) / (T)3;
            if (out0w) {
                const T st = sgn((out1[o + k * n] - out0w[o + k * n]) - (ref[o + k * n] - refw[o + k * n]));
                v = v + st * gtm / (T)3;
                if (g0w) g0w[o + k * n] = -st * gtm / (T)3;
            }
            g1[o + k * n] = v;
        }
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
    auto run = [&](auto tag) {
        using T = decltype(tag);
        if (losses || sp_map || tm_map || cb_map) {
            SSB_LAUNCH(s, k_loss_maps<T><<<dim3(kLossBlocks, B), 256, 0, s>>>(
                              n, (const T*)ldr1, (const T*)ref, (const T*)ldr0_w, (const T*)ref_w, (const T*)validity,
                              (const T*)mask, (T*)sp_map, (T*)tm_map, (T*)cb_map, (double*)workspace));
            if (losses)
                SSB_LAUNCH(s, k_loss_reduce<<<B, 256, 0, s>>>(n, ldr0_w != nullptr, validity != nullptr,
                                                              (const double*)workspace, losses));
        }
        if (g_ldr1)
            SSB_LAUNCH(s, k_loss_grads<T><<<grid_for<T>(n, B), 256, 0, s>>>(
                              n, (const T*)ldr1, (const T*)ref, (const T*)ldr0_w, (const T*)ref_w, (const T*)validity,
                              (const T*)mask, (T*)g_ldr1, (T*)g_ldr0_w));
    };
    if (dtype == SSB_F64) run(0.0);
    else run(0.0f);
    return cuda_check("ssb_losses");
}

}  // extern "C"
