// Temporal path: bilinear backward warp of the
// previous frame and its transpose, planar on device.
//   warp_array    images.py:88-119   out(p) = sum_k w_k(p) prev(tap_k(p)), validity = sum_k w_k
//   warp_backward images.py:122-147  grad_prev = transpose (np.add.at scatter)
// The transpose is computed as a deterministic GATHER.  float64: every target
// pixel scans the sources that can reach it (|q - p| <= ceil(max|motion|) + 1,
// staged in shared memory per tile when max|motion| <= 5) in the reference's
// own order (tap-major, then sources in raster order), so the result
// reproduces np.add.at bit for bit.  float32 with max|motion| <= 3: per-cell
// landing bit masks, per-cell tap sums, then 4 cells per target, in a fixed
// order (general scan beyond).  No floating-point atomics: results are
// run-to-run identical.  Compiled with -fmad=false (products and sums rounded
// like numpy; the float32 kernels use explicit FMAs where they want them).
#include <math.h>
#include <climits>
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

// float32, 3 channels: the CTA stages prev over its tile + a 4-pixel halo
// (coalesced rows) and gathers the taps from shared memory; a tap outside the
// staged window (|motion| > 3) falls back to a global load, per thread.
constexpr int WF_X = 32, WF_Y = 16, WF_WX = WF_X + 8, WF_WY = WF_Y + 8;

__global__ void __launch_bounds__(256) k_warp_staged(int H, int W, const float* __restrict__ prev,
                                                     const float* __restrict__ motion, float* __restrict__ out,
                                                     float* __restrict__ validity) {
    constexpr int NWIN = WF_WY * WF_WX;
    __shared__ float4 s_p[NWIN];  // channel-interleaved: one 16-B load per tap
    const int b = blockIdx.z, tid = threadIdx.x;
    const int tx0 = blockIdx.x * WF_X, ty0 = blockIdx.y * WF_Y;
    const int wx0 = tx0 - 4, wy0 = ty0 - 4;
    const unsigned hw = (unsigned)H * (unsigned)W;
    const float* mb = motion + (size_t)b * 2 * hw;
    const float* pb = prev + (size_t)b * 3 * hw;
    constexpr int NIT = (NWIN + 255) / 256;
    float pv[NIT][3];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {  // every load issued before the stores
        const int i = tid + it * 256;
        const int wj = i / WF_WX, wi = i - wj * WF_WX;
        const int qx = wx0 + wi, qy = wy0 + wj;
        const bool in = i < NWIN && qx >= 0 && qx < W && qy >= 0 && qy < H;
        const unsigned q = in ? (unsigned)qy * (unsigned)W + (unsigned)qx : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) pv[it][c] = in ? __ldg(pb + c * hw + q) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int i = tid + it * 256;
        if (i < NWIN) s_p[i] = make_float4(pv[it][0], pv[it][1], pv[it][2], 0.f);
    }
    __syncthreads();
    const int lx = tid & 31;
#pragma unroll
    for (int h = 0; h < WF_Y / 8; ++h) {
        const int x = tx0 + lx, y = ty0 + (tid >> 5) + 8 * h;
        if (x >= W || y >= H) continue;
        const unsigned p = (unsigned)y * (unsigned)W + (unsigned)x;
        const float mx = __ldg(mb + p), my = __ldg(mb + hw + p);
        // warp_tap's four taps, sharing the floor / fraction / clamp work:
        // x0 = x + floor(mx) (float32 split, images.py:101-117), taps x0 and
        // x0 + 1, weight 0 outside the frame, clamped source indices
        const float fmx = floorf(mx), fmy = floorf(my);
        const float fx = mx - fmx, fy = my - fmy;
        const float tx = (float)x + fmx, ty = (float)y + fmy;
        float wxs[2], wys[2];
        int ixs[2], iys[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            const float ux = tx + (float)d, uy = ty + (float)d;
            wxs[d] = (ux >= 0.f && ux < (float)W) ? (d ? fx : 1.f - fx) : 0.f;
            wys[d] = (uy >= 0.f && uy < (float)H) ? (d ? fy : 1.f - fy) : 0.f;
            ixs[d] = (int)fminf(fmaxf(ux, 0.f), (float)(W - 1));
            iys[d] = (int)fminf(fmaxf(uy, 0.f), (float)(H - 1));
        }
        float w[4], v[4][3];
        const bool inwin = ixs[0] - wx0 >= 0 && ixs[1] - wx0 < WF_WX && iys[0] - wy0 >= 0 && iys[1] - wy0 < WF_WY;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int dx = k & 1, dy = k >> 1;
            // (NaN motion: both tap weights of an axis are 0 -- the
            // comparisons fail -- and the clamped index is 0)
            w[k] = wxs[dx] * wys[dy];
            if (inwin) {
                const float4 t = s_p[(iys[dy] - wy0) * WF_WX + ixs[dx] - wx0];
                v[k][0] = t.x;
                v[k][1] = t.y;
                v[k][2] = t.z;
            } else {
                const unsigned src = (unsigned)iys[dy] * (unsigned)W + (unsigned)ixs[dx];
#pragma unroll
                for (int c = 0; c < 3; ++c) v[k][c] = __ldg(pb + c * hw + src);
            }
        }
        float* ob = out + (size_t)b * 3 * hw;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = __fmaf_rn(w[k], v[k][c], acc);
            __stcs(ob + c * hw + p, acc);
        }
        if (validity) {
            float vs = 0.f;
#pragma unroll
            for (int k = 0; k < 4; ++k) vs = vs + w[k];
            __stcs(validity + (size_t)b * hw + p, vs);
        }
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
        // non-finite motion is ignored: the reference gives its taps weight 0
        // (images.py:111-116: inf/NaN positions are never `inside`)
        m = (v > m && v < (double)INFINITY) ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(amax + b, (unsigned long long)__double_as_longlong(m));
}

// float32: max over the bit patterns of |m| (inf / NaN ignored), 16-B loads when
// the frame stride allows; stored as the double bits k_motion_absmax writes
__global__ void k_motion_absmax_f32(long long n2, const float* __restrict__ motion, unsigned long long* amax) {
    const int b = blockIdx.y;
    const float* mb = motion + (size_t)b * n2;
    unsigned m = 0u;
    auto take = [&](float v) {
        const unsigned a = __float_as_uint(v) & 0x7fffffffu;
        m = max(m, a >= 0x7f800000u ? 0u : a);  // inf / NaN: weight-0 taps, ignored
    };
    const long long stride = (long long)gridDim.x * blockDim.x;
    if (((reinterpret_cast<size_t>(mb)) & 15) == 0) {
        const long long n4 = n2 >> 2;
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcs(reinterpret_cast<const float4*>(mb) + i);
            take(v.x);
            take(v.y);
            take(v.z);
            take(v.w);
        }
        for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) take(mb[i]);
    } else {
        for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) take(mb[i]);
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m)
        atomicMax(amax + b, (unsigned long long)__double_as_longlong((double)__uint_as_float(m)));
}

// Float64 tiled transpose for |motion| <= WMAX - 1: the CTA stages, for every
// source of its window (tile + MR halo), the integer floor offset, the
// fractions and the gradient, then every target scans its (2 MR + 1)^2
// sources from shared memory, one pass per tap, sources in raster order --
// the np.add.at order (bit-exact).
constexpr int WT_X = 32, WT_Y = 8, WMAX = 6;
constexpr int SCAN_MR = 16;  // per-pixel source scans up to this radius; beyond: k_warp_backward_seg
constexpr int WM_MR = 4;  // float32 frames with MR <= WM_MR: k_warp_backward_mask
constexpr int WWX = WT_X + 2 * WMAX, WWY = WT_Y + 2 * WMAX;

template <typename T>
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
        for (int c = 0; c < nc; ++c) gprev[((size_t)b * C + c0 + c) * hw + (unsigned)y * (unsigned)W + x] = acc[c];
    }
}

// float32 transpose for max|motion| <= 3 (MR <= 4): instead of scanning
// every candidate source per target, each source of the window marks its
// tap-0 landing cell t0 = q + o (o = floor offset) in a per-cell bit mask
// (native shared atomicOr, order independent), then target p visits, tap by
// tap, the set bits of cell p - k in ascending order -- ~4 hits instead of
// ~25 candidates, deterministic.  Masks: NWD = 1 word per cell when
// max|motion| <= 2 (o in [-2, 2]^2, bit (oy + 2) * 5 + ox + 2), NWD = 2 when
// <= 3 (o in [-3, 3]^2, word oy > 0, bit ((oy + 3) & 3) * 8 + ox + 3).  The
// sources keep their four tap weights; a bit decodes to the source's window
// offset through a small table.  Larger motion runs the general per-target
// scan in the same kernel (one launch either way).
constexpr int WM_X = 32, WM_Y = 16;                 // tile
constexpr int WM_WX = WM_X + 7, WM_WY = WM_Y + 7;   // sources q - p in [-4, 3] per axis
constexpr int WM_MX = WM_X + 1, WM_MY = WM_Y + 1;   // landing cells t0 in [tile - 1, tile)

template <typename T>
__device__ void warp_backward_scan(int C, int H, int W, int b, int x, int y, int MR, const T* __restrict__ gout,
                                   const T* __restrict__ motion, T* __restrict__ gprev);

struct MaskSmem {
    static constexpr int NWIN = WM_WY * WM_WX, NCELL = WM_MY * WM_MX;
    float4 src[NWIN];      // per window source: fx, fy, g0, g1
    float src2[NWIN];      //                    g2
    float4 acc[4][NCELL];  // per landing cell and tap k: sum over its sources of w_k * g
    unsigned m[2][NCELL];
    int lut[64];           // bit -> window offset of the source from its cell
};

// Two gathers instead of one scatter: (1) every landing cell sums, per tap k,
// w_k * g over the sources that land on it (its mask bits, ascending); (2)
// every target adds the 4 cells p - k.  The cell walk is the only
// data-dependent loop, once per cell instead of once per (target, tap).
template <int NWD>
__device__ __forceinline__ void warp_bwd_mask_body(MaskSmem& sm, int C, int H, int W, int b, int tx0, int ty0,
                                                   const float* __restrict__ gout, const float* __restrict__ motion,
                                                   float* __restrict__ gprev) {
    constexpr int NWIN = MaskSmem::NWIN, NCELL = MaskSmem::NCELL, OB = NWD == 1 ? 2 : 3;  // |o| bound
    const int tid = threadIdx.x, lx = tid & 31, ly0 = tid >> 5;
    const int wx0 = tx0 - 4, wy0 = ty0 - 4;  // window origin; cell origin is tile - 1
    const unsigned hw = (unsigned)H * (unsigned)W;
    const float* mb = motion + (size_t)b * 2 * hw;
    for (int i = tid; i < NWD * NCELL; i += 256) (&sm.m[0][0])[i] = 0u;
    if (tid < 32 * NWD) {
        int oy, ox;
        if (NWD == 1) {
            oy = tid / 5 - 2;
            ox = tid % 5 - 2;
        } else {
            oy = ((tid & 31) >> 3) + (tid >= 32 ? 1 : -3);
            ox = (tid & 7) - 3;
        }
        sm.lut[tid] = (3 - oy) * WM_WX + (3 - ox);
    }
    __syncthreads();
    for (int c0 = 0; c0 < C; c0 += 3) {
        const int nc = min(3, C - c0);
        if (c0 > 0) __syncthreads();
        // (0) stage the window: landing masks (first group), fractions, gradient;
        // every load of the thread's window items is issued before any use
        constexpr int NIT = (NWIN + 255) / 256;
        const float* gp = gout + ((size_t)b * C + c0) * hw;  // 32-bit offsets below (C*H*W < 2^31)
        float mv[NIT][2], gv[NIT][3];
        bool inw[NIT];
        // window coordinates of item tid + 256 it, advanced incrementally
        constexpr int DJ = 256 / WM_WX, DI = 256 - DJ * WM_WX;
        int wjs[NIT], wis[NIT];
        wjs[0] = tid / WM_WX;
        wis[0] = tid - wjs[0] * WM_WX;
#pragma unroll
        for (int it = 1; it < NIT; ++it) {
            wjs[it] = wjs[it - 1] + DJ;
            wis[it] = wis[it - 1] + DI;
            if (wis[it] >= WM_WX) {
                wis[it] -= WM_WX;
                ++wjs[it];
            }
        }
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int i = tid + it * 256;
            const int wj = wjs[it], wi = wis[it];
            const int qx = wx0 + wi, qy = wy0 + wj;
            inw[it] = i < NWIN && qx >= 0 && qx < W && qy >= 0 && qy < H;  // others never land
            const unsigned q = inw[it] ? (unsigned)qy * (unsigned)W + (unsigned)qx : 0u;
            mv[it][0] = inw[it] ? __ldg(mb + q) : 0.f;
            mv[it][1] = inw[it] ? __ldg(mb + hw + q) : 0.f;
#pragma unroll
            for (int c = 0; c < 3; ++c) gv[it][c] = (inw[it] && c < nc) ? __ldg(gp + (c * hw + q)) : 0.f;
        }
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            if (!inw[it]) continue;
            const int i = tid + it * 256;
            const int wj = wjs[it], wi = wis[it];
            const float mx = mv[it][0], my = mv[it][1];
            const float fmx = floorf(mx), fmy = floorf(my);
            if (c0 == 0 && fmx >= (float)-OB && fmx <= (float)OB && fmy >= (float)-OB && fmy <= (float)OB) {
                const int ox = (int)fmx, oy = (int)fmy;  // (false for NaN motion)
                const int u = wi - 3 + ox, v = wj - 3 + oy;  // cell of t0 = q + o
                if (u >= 0 && u < WM_MX && v >= 0 && v < WM_MY) {
                    if (NWD == 1) atomicOr(&sm.m[0][v * WM_MX + u], 1u << ((oy + 2) * 5 + ox + 2));
                    else atomicOr(&sm.m[oy > 0][v * WM_MX + u], 1u << (((oy + 3) & 3) * 8 + ox + 3));
                }
            }
            sm.src[i] = make_float4(mx - fmx, my - fmy, gv[it][0], gv[it][1]);
            sm.src2[i] = gv[it][2];
        }
        __syncthreads();
        // (1) per landing cell and tap: sum of w_k * g over its sources, in bit order
        for (int cell = tid; cell < NCELL; cell += 256) {
            const int v = cell / WM_MX, u = cell - v * WM_MX;
            const int wc = v * WM_WX + u;
            float a[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int c = 0; c < 3; ++c) a[k][c] = 0.f;
#pragma unroll
            for (int wd = 0; wd < NWD; ++wd) {
                unsigned m = sm.m[wd][cell];
                while (m) {
                    const int bit = __ffs(m) - 1;
                    m &= m - 1;
                    const int li = wc + sm.lut[wd * 32 + bit];  // source q = t0 - o
                    const float4 t = sm.src[li];
                    const float g[3] = {t.z, t.w, sm.src2[li]};
                    // images.py:101-117: w = wx * wy per tap (dx, dy)
                    const float wk[4] = {(1.f - t.x) * (1.f - t.y), t.x * (1.f - t.y), (1.f - t.x) * t.y, t.x * t.y};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int c = 0; c < 3; ++c) a[k][c] = __fmaf_rn(wk[k], g[c], a[k][c]);  // (float32 path)
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sm.acc[k][cell] = make_float4(a[k][0], a[k][1], a[k][2], 0.f);
        }
        __syncthreads();
        // (2) targets: the 4 cells p - k, tap-major
#pragma unroll
        for (int h = 0; h < WM_Y / 8; ++h) {
            const int ly = ly0 + 8 * h, x = tx0 + lx, y = ty0 + ly;
            if (x >= W || y >= H) continue;
            float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 t = sm.acc[k][(ly + 1 - (k >> 1)) * WM_MX + lx + 1 - (k & 1)];
                acc[0] = acc[0] + t.x;
                acc[1] = acc[1] + t.y;
                acc[2] = acc[2] + t.z;
            }
            float* op = gprev + ((size_t)b * C + c0) * hw + ((unsigned)y * (unsigned)W + x);
            for (int c = 0; c < nc; ++c) __stcs(op + c * hw, acc[c]);
        }
    }
}

__global__ void __launch_bounds__(256) k_warp_backward_mask(int C, int H, int W, const float* __restrict__ gout,
                                                            const float* __restrict__ motion,
                                                            const unsigned long long* __restrict__ amax,
                                                            float* __restrict__ gprev) {
    extern __shared__ __align__(16) unsigned char smem_mask[];
    MaskSmem& sm = *reinterpret_cast<MaskSmem*>(smem_mask);
    const int b = blockIdx.z;
    const int tx0 = blockIdx.x * WM_X, ty0 = blockIdx.y * WM_Y;
    const double mm = __longlong_as_double((long long)amax[b]);
    if (mm <= 2.0) {
        warp_bwd_mask_body<1>(sm, C, H, W, b, tx0, ty0, gout, motion, gprev);
    } else if (mm <= 3.0) {
        warp_bwd_mask_body<2>(sm, C, H, W, b, tx0, ty0, gout, motion, gprev);
    } else {  // larger motion: general scan up to SCAN_MR (beyond: k_warp_backward_seg)
        const int MR = (int)ceil(mm) + 1;
        if (MR > SCAN_MR) return;
        for (int h = 0; h < WM_Y / 8; ++h) {
            const int x = tx0 + (threadIdx.x & 31), y = ty0 + (threadIdx.x >> 5) + 8 * h;
            if (x < W && y < H) warp_backward_scan<float>(C, H, W, b, x, y, MR, gout, motion, gprev);
        }
    }
}

// general transpose (any |motion|): target (x, y) scans every source within
// MR, np.add.at order (tap-major, sources in raster order)
template <typename T>
__device__ void warp_backward_scan(int C, int H, int W, int b, int x, int y, int MR, const T* __restrict__ gout,
                                   const T* __restrict__ motion, T* __restrict__ gprev) {
    const long long hw = (long long)H * W;
    const int qy0 = max(y - MR, 0), qy1 = min(y + MR, H - 1);
    const int qx0 = max(x - MR, 0), qx1 = min(x + MR, W - 1);
    constexpr int CMAX = 4;
    for (int c0 = 0; c0 < C; c0 += CMAX) {
        const int nc = min(CMAX, C - c0);
        T acc[CMAX];
#pragma unroll
        for (int c = 0; c < CMAX; ++c) acc[c] = (T)0;
        for (int k = 0; k < 4; ++k) {
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

// float64 frames whose max |motion| exceeds WMAX - 1 (up to SCAN_MR: beyond,
// k_warp_backward_seg)
template <typename T>
__global__ void k_warp_backward(int C, int H, int W, const T* __restrict__ gout,
                                const T* __restrict__ motion, const unsigned long long* __restrict__ amax,
                                T* __restrict__ gprev) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const double mm = __longlong_as_double((long long)amax[b]);
    if ((int)ceil(mm) + 1 <= WMAX) return;  // handled by the tiled kernel
    // sources farther than ceil(max|m|) + 1 cannot land on this pixel
    const int MR = (int)ceil(mm) + 1;
    if (MR > SCAN_MR) return;  // large motion: k_warp_backward_seg
    warp_backward_scan<T>(C, H, W, b, x, y, MR, gout, motion, gprev);
}

// Large motion (max |motion| + 1 > SCAN_MR), any dtype: O(HW) candidates
// instead of a (2 MR + 1)^2 scan per pixel (one outlier vector no longer turns
// every pixel's scan frame-wide).  Sources are taken in segments of SEG
// pixels of one row; k_warp_seg_bbox records the bounding box of each
// segment's in-frame, non-zero-weight landing cells; every 32 x 8 target tile
// then walks the segments in raster order (chunks of 256 tested at once and
// compacted in order), stages each intersecting segment's landings for tap k
// in shared memory and adds the matching ones -- tap-major, sources in raster
// order: the np.add.at order of images.py:140-146 (float64 bit-exact).
constexpr int SEG = 32;

template <typename T>
__global__ void __launch_bounds__(256) k_warp_seg_bbox(int H, int W, const T* __restrict__ motion,
                                                       const unsigned long long* __restrict__ amax,
                                                       int4* __restrict__ bbox, int nseg) {
    const int b = blockIdx.y;
    const double mm = __longlong_as_double((long long)amax[b]);
    if ((int)ceil(mm) + 1 <= SCAN_MR) return;
    const int wid = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (wid >= H * nseg) return;  // warp-uniform
    const int y = wid / nseg, sx = (wid - y * nseg) * SEG + lane;
    int x0 = INT_MAX, x1 = INT_MIN, y0 = INT_MAX, y1 = INT_MIN;
    if (sx < W) {
        const long long hw = (long long)H * W, q = (long long)y * W + sx;
        const T mx = motion[(b * 2 + 0) * hw + q], my = motion[(b * 2 + 1) * hw + q];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            T w;
            int ix, iy;
            warp_tap(k, sx, y, W, H, mx, my, w, ix, iy);
            if (w != (T)0) {
                x0 = min(x0, ix);
                x1 = max(x1, ix);
                y0 = min(y0, iy);
                y1 = max(y1, iy);
            }
        }
    }
    x0 = __reduce_min_sync(0xffffffffu, x0);
    x1 = __reduce_max_sync(0xffffffffu, x1);
    y0 = __reduce_min_sync(0xffffffffu, y0);
    y1 = __reduce_max_sync(0xffffffffu, y1);
    if (lane == 0) bbox[(long long)b * H * nseg + wid] = make_int4(x0, x1, y0, y1);
}

template <typename T>
__global__ void __launch_bounds__(256) k_warp_backward_seg(int C, int H, int W, const T* __restrict__ gout,
                                                           const T* __restrict__ motion,
                                                           const int4* __restrict__ bbox, int nseg,
                                                           const unsigned long long* __restrict__ amax,
                                                           T* __restrict__ gprev) {
    const int b = blockIdx.z;
    const double mm = __longlong_as_double((long long)amax[b]);
    if ((int)ceil(mm) + 1 <= SCAN_MR) return;  // block-uniform
    constexpr int CG = 4;
    __shared__ int s_cand[256];
    __shared__ int s_wc[8];
    __shared__ int s_ix[SEG], s_iy[SEG];
    __shared__ T s_w[SEG];
    __shared__ T s_gv[CG][SEG];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx0 = blockIdx.x * 32, ty0 = blockIdx.y * 8;
    const int x = tx0 + lane, y = ty0 + warp;
    const long long hw = (long long)H * W;
    const long long total = (long long)H * nseg;
    const int4* bb = bbox + (long long)b * total;
    for (int c0 = 0; c0 < C; c0 += CG) {
        const int nc = min(CG, C - c0);
        T acc[CG];
#pragma unroll
        for (int c = 0; c < CG; ++c) acc[c] = (T)0;
        for (int k = 0; k < 4; ++k) {
            for (long long s0 = 0; s0 < total; s0 += 256) {
                // segments of this chunk whose landing box meets the tile, in order
                bool hit = false;
                if (s0 + tid < total) {
                    const int4 r = bb[s0 + tid];
                    hit = r.x <= tx0 + 31 && r.y >= tx0 && r.z <= ty0 + 7 && r.w >= ty0;
                }
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (lane == 0) s_wc[warp] = __popc(m);
                __syncthreads();
                int off = 0, n = 0;
#pragma unroll
                for (int w2 = 0; w2 < 8; ++w2) {
                    off += w2 < warp ? s_wc[w2] : 0;
                    n += s_wc[w2];
                }
                if (hit) s_cand[off + __popc(m & ((1u << lane) - 1u))] = (int)(s0 + tid);
                __syncthreads();
                for (int j = 0; j < n; ++j) {
                    const int seg = s_cand[j];
                    const int sy = seg / nseg, sx = (seg - sy * nseg) * SEG + tid;
                    if (tid < SEG) {
                        T w = (T)0;
                        int ix = -1, iy = -1;
                        if (sx < W) {
                            const long long q = (long long)sy * W + sx;
                            warp_tap(k, sx, sy, W, H, motion[(b * 2 + 0) * hw + q], motion[(b * 2 + 1) * hw + q], w,
                                     ix, iy);
                            if (w != (T)0)
                                for (int c = 0; c < nc; ++c) s_gv[c][tid] = gout[((long long)b * C + c0 + c) * hw + q];
                        }
                        s_w[tid] = w;
                        s_ix[tid] = ix;
                        s_iy[tid] = iy;
                    }
                    __syncthreads();
                    if (x < W && y < H) {
                        for (int jj = 0; jj < SEG; ++jj) {
                            if (s_w[jj] != (T)0 && s_ix[jj] == x && s_iy[jj] == y) {
#pragma unroll
                                for (int c = 0; c < CG; ++c)
                                    if (c < nc) acc[c] = acc[c] + s_w[jj] * s_gv[c][jj];
                            }
                        }
                    }
                    __syncthreads();
                }
            }
        }
        if (x < W && y < H)
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
        dim3 sgrid((W + WF_X - 1) / WF_X, (H + WF_Y - 1) / WF_Y, B);
        if (C == 3) SSB_LAUNCH(s, k_warp_staged<<<sgrid, 256, 0, s>>>(H, W, pr, mo, (float*)out, (float*)validity));
        else SSB_LAUNCH(s, k_warp<float, 0><<<grid, block, 0, s>>>(C, H, W, pr, mo, (float*)out, (float*)validity));
    } else {
        set_error("ssb_warp: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    return cuda_check("ssb_warp");
}

int ssb_warp_backward_workspace_bytes(int B, int H, int W, size_t* bytes) {
    if (B <= 0 || H <= 0 || W <= 0 || !bytes) {
        set_error("ssb_warp_backward_workspace_bytes: invalid arguments");
        return SSB_EINVAL;
    }
    // per frame: max |motion| (8 B), then the segment landing boxes (16 B
    // each) of the large-motion path
    const size_t nseg = (size_t)(W + SEG - 1) / SEG;
    *bytes = (((size_t)B * sizeof(unsigned long long) + 15) & ~(size_t)15) + (size_t)B * H * nseg * sizeof(int4);
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
    if ((long long)H * W * C >= (1ll << 31)) {
        set_error("ssb_warp_backward: H*W*C must be < 2^31 per frame");
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
        SSB_LAUNCH(s, k_warp_backward_tiled<double><<<tgrid, dim3(WT_X, WT_Y), 0, s>>>(
                          C, H, W, (const double*)grad_out, (const double*)motion, amax, (double*)grad_prev));
        SSB_LAUNCH(s, k_warp_backward<double><<<grid, block, 0, s>>>(C, H, W, (const double*)grad_out,
                                                                   (const double*)motion, amax, (double*)grad_prev));
    } else {
        const long long b4 = (2 * n + 1023) / 1024;
        SSB_LAUNCH(s, k_motion_absmax_f32<<<dim3((unsigned)(b4 < 296 ? b4 : 296), B), 256, 0, s>>>(
                          2 * n, (const float*)motion, amax));
        dim3 mgrid((W + WM_X - 1) / WM_X, (H + WM_Y - 1) / WM_Y, B);
        static std::atomic<unsigned long long> attr_mask{0};
        smem_attr_once(attr_mask, (const void*)k_warp_backward_mask, (int)sizeof(MaskSmem));
        SSB_LAUNCH(s, k_warp_backward_mask<<<mgrid, 256, sizeof(MaskSmem), s>>>(C, H, W, (const float*)grad_out,
                                                                 (const float*)motion, amax, (float*)grad_prev));
    }
    // large motion (frames with max |motion| + 1 > SCAN_MR; the kernels exit
    // at once for the others)
    const int nseg = (W + SEG - 1) / SEG;
    int4* bbox = (int4*)((char*)workspace + (((size_t)B * sizeof(unsigned long long) + 15) & ~(size_t)15));
    dim3 bgrid((unsigned)(((long long)H * nseg + 7) / 8), B);
    if (dtype == SSB_F64) {
        SSB_LAUNCH(s, k_warp_seg_bbox<double><<<bgrid, 256, 0, s>>>(H, W, (const double*)motion, amax, bbox, nseg));
        SSB_LAUNCH(s, k_warp_backward_seg<double><<<grid, 256, 0, s>>>(C, H, W, (const double*)grad_out,
                                                                     (const double*)motion, bbox, nseg, amax,
                                                                     (double*)grad_prev));
    } else {
        SSB_LAUNCH(s, k_warp_seg_bbox<float><<<bgrid, 256, 0, s>>>(H, W, (const float*)motion, amax, bbox, nseg));
        SSB_LAUNCH(s, k_warp_backward_seg<float><<<grid, 256, 0, s>>>(C, H, W, (const float*)grad_out,
                                                                    (const float*)motion, bbox, nseg, amax,
                                                                    (float*)grad_prev));
    }
    return cuda_check("ssb_warp_backward");
}

}  // extern "C"
