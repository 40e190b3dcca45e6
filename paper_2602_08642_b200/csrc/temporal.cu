// Temporal path: bilinear backward warp of the
// previous frame and its transpose, planar on device.
//   warp_array    images.py:88-119   out(p) = sum_k w_k(p) prev(tap_k(p)), validity = sum_k w_k
//   warp_backward images.py:122-147  grad_prev = transpose (np.add.at scatter)
// The transpose is computed as a deterministic GATHER: every target pixel
// scans the sources that can reach it (|q - p| <= ceil(max|motion|) + 1,
// staged in shared memory per tile when max|motion| <= 5), in float64 in the
// reference's own order (tap-major, then sources in raster order) so the
// result reproduces np.add.at bit for bit; float32 in one raster pass.  No
// atomics: results are run-to-run identical.
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

// NC > 0: compile-time channel count (the 3-channel radiance path); NC = 0:
// any C.  32-bit offsets inside a frame (H*W*C < 2^31, checked on the host).
template <typename T, int NC>
__global__ void __launch_bounds__(256) k_warp(int C, int H, int W, const T* __restrict__ prev,
                                              const T* __restrict__ motion, T* __restrict__ out,
                                              T* __restrict__ validity) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const int cn = NC > 0 ? NC : C;
    const unsigned hw = (unsigned)H * (unsigned)W, p = (unsigned)y * (unsigned)W + (unsigned)x;
    const T* mb = motion + (size_t)b * 2 * hw;
    const T* pb = prev + (size_t)b * cn * hw;
    T* ob = out + (size_t)b * cn * hw;
    const T mx = __ldg(mb + p), my = __ldg(mb + hw + p);
    T w[4];
    unsigned src[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int ix, iy;
        warp_tap(k, x, y, W, H, mx, my, w[k], ix, iy);
        src[k] = (unsigned)iy * (unsigned)W + (unsigned)ix;
    }
#pragma unroll
    for (int c = 0; c < (NC > 0 ? NC : 1); ++c) {
        if (NC == 0) break;
        const T* pc = pb + c * hw;
        T acc = (T)0;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc = acc + w[k] * __ldg(pc + src[k]);
        ob[c * hw + p] = acc;
    }
    if (NC == 0) {
        for (int c = 0; c < cn; ++c) {
            const T* pc = pb + c * hw;
            T acc = (T)0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + w[k] * __ldg(pc + src[k]);
            ob[c * hw + p] = acc;
        }
    }
    if (validity) {
        T v = (T)0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v = v + w[k];
        validity[(size_t)b * hw + p] = v;
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

// Tiled transpose for |motion| <= WMAX: the CTA stages, for every source of
// its window (tile + MR halo), the integer floor offset, the fractions and
// the gradient, then every target scans its (2 MR + 1)^2 sources from shared
// memory.  EXACT (float64): one pass per tap, sources in raster order -- the
// np.add.at order; otherwise one pass over the sources (raster order, each
// source reaches a target through at most one tap): deterministic.
constexpr int WT_X = 32, WT_Y = 8, WMAX = 6;
constexpr int WWX = WT_X + 2 * WMAX, WWY = WT_Y + 2 * WMAX;

template <typename T, bool EXACT>
__global__ void __launch_bounds__(WT_X * WT_Y) k_warp_backward_tiled(
    int C, int H, int W, const T* __restrict__ gout, const T* __restrict__ motion,
    const unsigned long long* __restrict__ amax, T* __restrict__ gprev) {
    __shared__ int s_off[WWY * WWX];  // (x0 - qx + 128) | (y0 - qy + 128) << 8, or -1 (no source)
    __shared__ T s_fx[WWY * WWX], s_fy[WWY * WWX];
    __shared__ T s_g[3][WWY * WWX];
    const int b = blockIdx.z;
    const int tx0 = blockIdx.x * WT_X, ty0 = blockIdx.y * WT_Y;
    const int tid = threadIdx.y * WT_X + threadIdx.x;
    const double mm = __longlong_as_double((long long)amax[b]);
    const int MR = (int)ceil(mm) + 1;
    if (MR > WMAX) return;  // frame left to the general kernel (uniform per CTA)
    const int x = tx0 + threadIdx.x, y = ty0 + threadIdx.y;
    const unsigned hw = (unsigned)H * (unsigned)W;
    const T* mb = motion + (size_t)b * 2 * hw;
    const int wx0 = tx0 - MR, wy0 = ty0 - MR, wnx = WT_X + 2 * MR, wny = WT_Y + 2 * MR;
    // stage the window's floor offsets and fractions (channel independent),
    // with the window's offset range (sources only reach targets p with
    // p - q in [o_min, o_max + 1] per axis: the scan shrinks to that box)
    __shared__ int s_bb[4];
    if (tid < 4) s_bb[tid] = (tid & 1) ? -1000 : 1000;
    __syncthreads();
    int oxl = 1000, oxh = -1000, oyl = 1000, oyh = -1000;
    for (int i = tid; i < wnx * wny; i += WT_X * WT_Y) {
        const int qy = wy0 + i / wnx, qx = wx0 + i % wnx;
        int off = -1;
        T fx = (T)0, fy = (T)0;
        if (qx >= 0 && qx < W && qy >= 0 && qy < H) {
            const unsigned q = (unsigned)qy * (unsigned)W + (unsigned)qx;
            const T mx = mb[q], my = mb[hw + q];
            T x0, y0;
            if constexpr (sizeof(T) == 8) {
                const T sx = (T)qx + mx, sy = (T)qy + my;
                x0 = floor(sx);
                y0 = floor(sy);
                fx = sx - x0;
                fy = sy - y0;
            } else {
                const T fmx = floor(mx), fmy = floor(my);
                fx = mx - fmx;
                fy = my - fmy;
                x0 = (T)qx + fmx;
                y0 = (T)qy + fmy;
            }
            const T ox = x0 - (T)qx, oy = y0 - (T)qy;  // in [-MR, MR - 1]
            if (ox >= (T)-127 && ox <= (T)127 && oy >= (T)-127 && oy <= (T)127) {
                off = ((int)ox + 128) | (((int)oy + 128) << 8);
                oxl = min(oxl, (int)ox);
                oxh = max(oxh, (int)ox);
                oyl = min(oyl, (int)oy);
                oyh = max(oyh, (int)oy);
            }
        }
        s_off[i] = off;
        s_fx[i] = fx;
        s_fy[i] = fy;
    }
    atomicMin(&s_bb[0], oxl);
    atomicMax(&s_bb[1], oxh);
    atomicMin(&s_bb[2], oyl);
    atomicMax(&s_bb[3], oyh);
    for (int c0 = 0; c0 < C; c0 += 3) {
        const int nc = min(3, C - c0);
        __syncthreads();
        for (int i = tid; i < wnx * wny; i += WT_X * WT_Y) {
            const int qy = wy0 + i / wnx, qx = wx0 + i % wnx;
            const bool in = qx >= 0 && qx < W && qy >= 0 && qy < H;
            const unsigned q = in ? (unsigned)qy * (unsigned)W + (unsigned)qx : 0u;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                s_g[c][i] = (in && c < nc) ? gout[((size_t)b * C + c0 + c) * hw + q] : (T)0;
        }
        __syncthreads();
        if (x >= W || y >= H) continue;
        T acc[3] = {(T)0, (T)0, (T)0};
        // sources q with |q - p| <= MR, window-local index
        const int lx0 = threadIdx.x, ly0 = threadIdx.y;  // (x - MR) - wx0 = threadIdx.x
        // scan box: q - p in [-(o_max + 1), -o_min] per axis, within the MR window
        const int i0 = max(0, MR - s_bb[1] - 1), i1 = min(2 * MR, MR - s_bb[0]);
        const int j0 = max(0, MR - s_bb[3] - 1), j1 = min(2 * MR, MR - s_bb[2]);
        auto take = [&](int li, int kdx, int kdy, T fx, T fy) {
            const T wx = kdx ? fx : (T)1 - fx, wy = kdy ? fy : (T)1 - fy;
            const T wgt = wx * wy;
            if (wgt == (T)0) return;
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = acc[c] + wgt * s_g[c][li];
        };
        if constexpr (EXACT) {
            for (int k = 0; k < 4; ++k) {
                const int kdy = k >> 1, kdx = k & 1;
                for (int j = j0; j <= j1; ++j) {
                    const int qy = y - MR + j;
                    if (qy < 0 || qy >= H) continue;
                    for (int i = i0; i <= i1; ++i) {
                        const int qx = x - MR + i;
                        if (qx < 0 || qx >= W) continue;
                        const int li = (ly0 + j) * wnx + lx0 + i;
                        const int off = s_off[li];
                        if (off < 0) continue;
                        // tap k of q lands on (qx + ox + kdx, qy + oy + kdy)
                        if (qx + (off & 255) - 128 + kdx != x || qy + (off >> 8) - 128 + kdy != y) continue;
                        take(li, kdx, kdy, s_fx[li], s_fy[li]);
                    }
                }
            }
        } else {
            for (int j = j0; j <= j1; ++j) {
                for (int i = i0; i <= i1; ++i) {
                    const int li = (ly0 + j) * wnx + lx0 + i;
                    const int off = s_off[li];
                    if (off < 0) continue;
                    const int kdx = x - (x - MR + i) - ((off & 255) - 128);
                    const int kdy = y - (y - MR + j) - ((off >> 8) - 128);
                    if ((unsigned)kdx > 1u || (unsigned)kdy > 1u) continue;
                    take(li, kdx, kdy, s_fx[li], s_fy[li]);
                }
            }
        }
        for (int c = 0; c < nc; ++c) gprev[((size_t)b * C + c0 + c) * hw + (unsigned)y * (unsigned)W + x] = acc[c];
    }
}

// general transpose (any |motion|; frames whose max |motion| exceeds WMAX - 1)
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
    if ((int)ceil(mm) + 1 <= WMAX) return;  // handled by the tiled kernel
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
    if ((long long)H * W * C >= (1ll << 31)) {
        set_error("ssb_warp: H*W*C must be < 2^31 per frame");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    if (dtype == SSB_F64) {
        auto* pr = (const double*)prev;
        auto* mo = (const double*)motion;
        if (C == 3) SSB_LAUNCH(s, k_warp<double, 3><<<grid, block, 0, s>>>(C, H, W, pr, mo, (double*)out, (double*)validity));
        else SSB_LAUNCH(s, k_warp<double, 0><<<grid, block, 0, s>>>(C, H, W, pr, mo, (double*)out, (double*)validity));
    } else if (dtype == SSB_F32) {
        auto* pr = (const float*)prev;
        auto* mo = (const float*)motion;
        if (C == 3) SSB_LAUNCH(s, k_warp<float, 3><<<grid, block, 0, s>>>(C, H, W, pr, mo, (float*)out, (float*)validity));
        else SSB_LAUNCH(s, k_warp<float, 0><<<grid, block, 0, s>>>(C, H, W, pr, mo, (float*)out, (float*)validity));
    } else {
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
    dim3 tgrid((W + WT_X - 1) / WT_X, (H + WT_Y - 1) / WT_Y, B);
    if (dtype == SSB_F64) {
        SSB_LAUNCH(s, k_motion_absmax<double><<<rgrid, 256, 0, s>>>(n, (const double*)motion, amax));
        SSB_LAUNCH(s, k_warp_backward_tiled<double, true><<<tgrid, dim3(WT_X, WT_Y), 0, s>>>(
                          C, H, W, (const double*)grad_out, (const double*)motion, amax, (double*)grad_prev));
        SSB_LAUNCH(s, k_warp_backward<double><<<grid, block, 0, s>>>(C, H, W, (const double*)grad_out,
                                                                   (const double*)motion, amax, (double*)grad_prev));
    } else {
        SSB_LAUNCH(s, k_motion_absmax<float><<<rgrid, 256, 0, s>>>(n, (const float*)motion, amax));
        SSB_LAUNCH(s, k_warp_backward_tiled<float, false><<<tgrid, dim3(WT_X, WT_Y), 0, s>>>(
                          C, H, W, (const float*)grad_out, (const float*)motion, amax, (float*)grad_prev));
        SSB_LAUNCH(s, k_warp_backward<float><<<grid, block, 0, s>>>(C, H, W, (const float*)grad_out,
                                                                  (const float*)motion, amax, (float*)grad_prev));
    }
    return cuda_check("ssb_warp_backward");
}

}  // extern "C"
