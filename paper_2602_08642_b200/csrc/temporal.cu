// Temporal path: bilinear backward warp of the
// previous frame and its transpose, planar on device.
//   warp_array    images.py:88-119   out(p) = sum_k w_k(p) prev(tap_k(p)), validity = sum_k w_k
//   warp_backward images.py:122-147  grad_prev = transpose (np.add.at scatter)
// The transpose is computed as a deterministic GATHER: every target pixel
// scans the sources that can reach it (|q - p| <= ceil(max|motion|) + 1) in
// the reference's own order (tap-major, then sources in raster order), so the
// float64 result reproduces np.add.at bit for bit and no atomics are used.
// Compiled with -fmad=false (products and sums rounded like numpy).
#include <math.h>
#include <string>

#include "common.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

// tap k = 2*dy + dx of pixel (x, y): weight (0 when outside the frame) and the
// clipped source coordinates, images.py:101-117 (same products, same order)
template <typename T>
__device__ __forceinline__ void warp_tap(int k, int x, int y, int W, int H, T mx, T my, T& w, int& ix,
                                         int& iy) {
    T x0, y0, fx, fy;
    if constexpr (sizeof(T) == 8) {  // the reference's formula, bit for bit
        const T sx = (T)x + mx, sy = (T)y + my;
        x0 = floor(sx);
        y0 = floor(sy);
        fx = sx - x0;
        fy = sy - y0;
    } else {  // float32: split off the integer pixel position first (x + mx
              // would round the fraction at ~1e-4 for x ~ 2000)
        const T fmx = floor(mx), fmy = floor(my);
        fx = mx - fmx;
        fy = my - fmy;
        x0 = (T)x + fmx;
        y0 = (T)y + fmy;
    }
    const int dy = k >> 1, dx = k & 1;
    const T wx = dx ? fx : (T)1 - fx, wy = dy ? fy : (T)1 - fy;
    const T wt = wx * wy;
    const T tx = x0 + (T)dx, ty = y0 + (T)dy;
    const bool inside = tx >= (T)0 && tx < (T)W && ty >= (T)0 && ty < (T)H;
    w = inside ? wt : (T)0;
    ix = (int)fmin(fmax(tx, (T)0), (T)(W - 1));
    iy = (int)fmin(fmax(ty, (T)0), (T)(H - 1));
}

template <typename T>
__global__ void k_warp(int C, int H, int W, const T* __restrict__ prev, const T* __restrict__ motion,
                       T* __restrict__ out, T* __restrict__ validity) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const long long hw = (long long)H * W, p = (long long)y * W + x;
    const T mx = motion[(b * 2 + 0) * hw + p], my = motion[(b * 2 + 1) * hw + p];
    T w[4];
    long long src[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int ix, iy;
        warp_tap(k, x, y, W, H, mx, my, w[k], ix, iy);
        src[k] = (long long)iy * W + ix;
    }
    for (int c = 0; c < C; ++c) {
        const T* pc = prev + ((long long)b * C + c) * hw;
        T acc = (T)0;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc = acc + w[k] * pc[src[k]];
        out[((long long)b * C + c) * hw + p] = acc;
    }
    if (validity) {
        T v = (T)0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v = v + w[k];
        validity[b * hw + p] = v;
    }
}

// per-frame max |motion| as ordered float bits (non-negative floats order like
// their bit patterns), for the gather window of the transpose
template <typename T>
__global__ void k_motion_absmax(long long n, const T* __restrict__ motion, unsigned long long* amax) {
    const int b = blockIdx.y;
    double m = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n;
         i += (long long)gridDim.x * blockDim.x) {
        const double v = fabs((double)motion[b * 2 * n + i]);
        m = v > m ? v : m;  // NaN motion is ignored (the reference warps it to weight 0 taps)
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(amax + b, (unsigned long long)__double_as_longlong(m));
}

template <typename T>
__global__ void k_warp_backward(int C, int H, int W, const T* __restrict__ gout,
                                const T* __restrict__ motion, const unsigned long long* __restrict__ amax,
                                T* __restrict__ gprev) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const long long hw = (long long)H * W;
    const double mm = __longlong_as_double((long long)amax[b]);
    // sources farther than ceil(max|m|) + 1 cannot land on this pixel
    const int MR = (int)fmin(ceil(mm) + 1.0, (double)(H > W ? H : W));
    const int qy0 = max(y - MR, 0), qy1 = min(y + MR, H - 1);
    const int qx0 = max(x - MR, 0), qx1 = min(x + MR, W - 1);
    constexpr int CMAX = 4;
    for (int c0 = 0; c0 < C; c0 += CMAX) {
        const int nc = min(CMAX, C - c0);
        T acc[CMAX];
#pragma unroll
        for (int c = 0; c < CMAX; ++c) acc[c] = (T)0;
        for (int k = 0; k < 4; ++k) {  // np.add.at order: tap-major, sources in raster order
            for (int qy = qy0; qy <= qy1; ++qy) {
                for (int qx = qx0; qx <= qx1; ++qx) {
                    const long long q = (long long)qy * W + qx;
                    const T mx = motion[(b * 2 + 0) * hw + q], my = motion[(b * 2 + 1) * hw + q];
                    T w;
                    int ix, iy;
                    warp_tap(k, qx, qy, W, H, mx, my, w, ix, iy);
                    if (ix != x || iy != y || w == (T)0) continue;
#pragma unroll
                    for (int c = 0; c < CMAX; ++c)
                        if (c < nc) acc[c] = acc[c] + w * gout[((long long)b * C + c0 + c) * hw + q];
                }
            }
        }
        for (int c = 0; c < nc; ++c) gprev[((long long)b * C + c0 + c) * hw + (long long)y * W + x] = acc[c];
    }
}

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_warp(int dtype, int B, int C, int H, int W, const void* prev, const void* motion, void* out,
             void* validity, ssb_stream_t stream) {
    if (B <= 0 || C <= 0 || H <= 0 || W <= 0 || !prev || !motion || !out) {
        set_error("ssb_warp: invalid arguments");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    if (dtype == SSB_F64)
        SSB_LAUNCH(s, k_warp<double><<<grid, block, 0, s>>>(C, H, W, (const double*)prev, (const double*)motion,
                                                          (double*)out, (double*)validity));
    else if (dtype == SSB_F32)
        SSB_LAUNCH(s, k_warp<float><<<grid, block, 0, s>>>(C, H, W, (const float*)prev, (const float*)motion,
                                                         (float*)out, (float*)validity));
    else {
        set_error("ssb_warp: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    return cuda_check("ssb_warp");
}

int ssb_warp_backward_workspace_bytes(int B, size_t* bytes) {
    if (B <= 0 || !bytes) {
        set_error("ssb_warp_backward_workspace_bytes: invalid arguments");
        return SSB_EINVAL;
    }
    *bytes = (size_t)B * sizeof(unsigned long long);
    return 0;
}

int ssb_warp_backward(int dtype, int B, int C, int H, int W, const void* grad_out, const void* motion,
                      void* grad_prev, void* workspace, ssb_stream_t stream) {
    if (B <= 0 || C <= 0 || H <= 0 || W <= 0 || !grad_out || !motion || !grad_prev || !workspace) {
        set_error("ssb_warp_backward: invalid arguments");
        return SSB_EINVAL;
    }
    if (dtype != SSB_F32 && dtype != SSB_F64) {
        set_error("ssb_warp_backward: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* amax = (unsigned long long*)workspace;
    cudaMemsetAsync(amax, 0, (size_t)B * sizeof(unsigned long long), s);
    const long long n = (long long)H * W;
    dim3 rgrid((unsigned)((2 * n + 255) / 256 < 1024 ? (2 * n + 255) / 256 : 1024), B);
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    if (dtype == SSB_F64) {
        SSB_LAUNCH(s, k_motion_absmax<double><<<rgrid, 256, 0, s>>>(n, (const double*)motion, amax));
        SSB_LAUNCH(s, k_warp_backward<double><<<grid, block, 0, s>>>(C, H, W, (const double*)grad_out,
                                                                   (const double*)motion, amax, (double*)grad_prev));
    } else {
        SSB_LAUNCH(s, k_motion_absmax<float><<<rgrid, 256, 0, s>>>(n, (const float*)motion, amax));
        SSB_LAUNCH(s, k_warp_backward<float><<<grid, block, 0, s>>>(C, H, W, (const float*)grad_out,
                                                                  (const float*)motion, amax, (float*)grad_prev));
    }
    return cuda_check("ssb_warp_backward");
}

}  // extern "C"
