// Estimator backward to the density scores, the
// sampler half of optimize.evaluate_step (optimize.py:244-251):
//   g_spp   = sum_f sum_c g_input[f, c] * grad_density[f, c]     (per pixel)
//   g_spp   = gaussian_filter(g_spp, sigma, mode="nearest")      (if sigma > 0)
//   w       = softmax(scores)                                    (frame-global)
//   g_score = (7/8 * budget * N) * w * (g_spp - sum(w * g_spp))  (density.py:49-52)
// gaussian_filter is scipy.ndimage's (1.18.x): separable 1-D correlations,
// axis 0 then axis 1, weights exp(-x^2 / (2 sigma^2)) on |x| <= int(4 sigma +
// 0.5) normalised to sum 1, edge replication; the symmetric-kernel sum order
// x_i w0 + sum_{j = r..1} (x_{i-j} + x_{i+j}) w_j is kept.  Arithmetic in float64 (a
// few bytes per pixel; the reductions are deterministic two-level trees).
#include <math.h>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

constexpr int kSgThreads = 256, kSgBlocks = 128;  // reduction partials per frame
constexpr int kMaxBlurRadius = 64;

struct BlurWeights {
    double w[kMaxBlurRadius + 1];  // w[0] centre, w[j] = weight at +-j
    int r;
};

// block-wide reduction for 256-thread blocks of any shape (linear thread id)
__device__ __forceinline__ double sg_block_reduce(double v, bool is_max) {
    __shared__ double sh[kSgThreads / 32];
    const int t = threadIdx.y * blockDim.x + threadIdx.x;
    for (int o = 16; o > 0; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, u) : v + u;
    }
    if ((t & 31) == 0) sh[t >> 5] = v;
    __syncthreads();
    if (t < 32) {
        v = t < kSgThreads / 32 ? sh[t] : (is_max ? -INFINITY : 0.0);
        for (int o = 16; o > 0; o >>= 1) {
            const double u = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmax(v, u) : v + u;
        }
    }
    __syncthreads();
    return v;
}

// g_spp[b, p] = sum_f ((g0 d0 + g1 d1) + g2 d2) ..., frames added in order
template <typename T>
__global__ void k_score_dot(int F, int C, long long n, const T* __restrict__ gin, const T* __restrict__ gd,
                            double* __restrict__ gspp) {
    const int b = blockIdx.y;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        double tot = 0.0;
        for (int f = 0; f < F; ++f) {
            const long long base = ((long long)(b * F + f) * C) * n + p;
            double s = (double)gin[base] * (double)gd[base];
            for (int c = 1; c < C; ++c) s = s + (double)gin[base + c * n] * (double)gd[base + c * n];
            tot = f == 0 ? s : tot + s;
        }
        gspp[(long long)b * n + p] = tot;
    }
}

// 1-D correlation along y (axis 0) or x (axis 1), edge replication
__global__ void k_blur_axis(int H, int W, int axis, BlurWeights bw, const double* __restrict__ in,
                            double* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const double* p = in + (long long)b * H * W;
    auto at = [&](int yy, int xx) { return p[(long long)clampi(yy, 0, H - 1) * W + clampi(xx, 0, W - 1)]; };
    double s = at(y, x) * bw.w[0];
    for (int j = bw.r; j >= 1; --j) {  // scipy's symmetric loop runs from the far taps inwards
        const double a = axis == 0 ? at(y - j, x) : at(y, x - j);
        const double c = axis == 0 ? at(y + j, x) : at(y, x + j);
        s = s + (a + c) * bw.w[j];
    }
    out[(long long)b * H * W + (long long)y * W + x] = s;
}

template <typename T>
__global__ void k_sg_partial_max(long long n, const T* __restrict__ scores, double* pmax) {
    const int b = blockIdx.y;
    double m = -INFINITY;
    for (long long i = (long long)blockIdx.x * kSgThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kSgThreads)
        m = fmax(m, (double)scores[(long long)b * n + i]);
    m = sg_block_reduce(m, true);
    if (threadIdx.x == 0) pmax[b * kSgBlocks + blockIdx.x] = m;
}

__device__ __forceinline__ double sg_frame(const double* part, int b, bool is_max) {
    double v = is_max ? -INFINITY : 0.0;
    for (int k = 0; k < kSgBlocks; ++k) v = is_max ? fmax(v, part[b * kSgBlocks + k]) : v + part[b * kSgBlocks + k];
    return v;
}

// partial sums of e = exp(s - max) and of e * g
template <typename T>
__global__ void k_sg_partial_sums(long long n, const T* __restrict__ scores, const double* __restrict__ g,
                                  const double* pmax, double* psum, double* pdot) {
    const int b = blockIdx.y;
    const double m = sg_frame(pmax, b, true);
    double se = 0.0, sd = 0.0;
    for (long long i = (long long)blockIdx.x * kSgThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kSgThreads) {
        const double e = exp((double)scores[(long long)b * n + i] - m);
        se += e;
        sd += e * g[(long long)b * n + i];
    }
    se = sg_block_reduce(se, false);
    sd = sg_block_reduce(sd, false);
    if (threadIdx.x == 0) {
        psum[b * kSgBlocks + blockIdx.x] = se;
        pdot[b * kSgBlocks + blockIdx.x] = sd;
    }
}

template <typename T>
__global__ void k_sg_apply(long long n, const T* __restrict__ scores, const double* __restrict__ g,
                           const double* pmax, const double* psum, const double* pdot, double total,
                           T* __restrict__ out) {
    const int b = blockIdx.y;
    __shared__ double sm, ss, inner;
    if (threadIdx.x == 0) {
        sm = sg_frame(pmax, b, true);
        ss = sg_frame(psum, b, false);
        inner = sg_frame(pdot, b, false) / ss;  // sum(w * g)
    }
    __syncthreads();
    for (long long i = (long long)blockIdx.x * kSgThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kSgThreads) {
        const double w = exp((double)scores[(long long)b * n + i] - sm) / ss;
        out[(long long)b * n + i] = (T)(total * (w * (g[(long long)b * n + i] - inner)));
    }
}


// ---- fused path (blur radius <= 16): dot + score max, tiled 2-D blur + the
// softmax partial sums, per-frame reduction, apply -- three passes over the
// pixels instead of six
constexpr int SG_TX = 32, SG_TY = 8, SG_RMAX = 16;
constexpr int kDotBlocks = 1024;  // dot + max pass: blocks per frame

template <typename T>
__device__ __forceinline__ double sg_exp(T s, double m) {
    if constexpr (sizeof(T) == 8) return exp(s - m);
    else return (double)__expf((float)((double)s - m));  // float32 path: 2-ulp exp
}

// float32 inputs compute the per-pixel dot and the blur in float32 (the
// reductions stay float64); float64 inputs keep float64 throughout
template <typename T>
using acc_t = typename std::conditional<sizeof(T) == 8, double, float>::type;

template <typename T>
__global__ void k_score_dot_max(int F, int C, long long n, const T* __restrict__ gin, const T* __restrict__ gd,
                                const T* __restrict__ scores, acc_t<T>* __restrict__ gspp, double* pmax) {
    using A = acc_t<T>;
    const int b = blockIdx.y;
    double m = -INFINITY;
    for (long long p = (long long)blockIdx.x * kSgThreads + threadIdx.x; p < n; p += (long long)gridDim.x * kSgThreads) {
        A tot = (A)0;
        for (int f = 0; f < F; ++f) {
            const long long base = ((long long)(b * F + f) * C) * n + p;
            A s = (A)gin[base] * (A)gd[base];
            for (int c = 1; c < C; ++c) s = s + (A)gin[base + c * n] * (A)gd[base + c * n];
            tot = f == 0 ? s : tot + s;
        }
        gspp[(long long)b * n + p] = tot;
        m = fmax(m, (double)scores[(long long)b * n + p]);
    }
    m = sg_block_reduce(m, true);
    if (threadIdx.x == 0) pmax[b * kDotBlocks + blockIdx.x] = m;
}

// float32, four pixels per thread (16-B loads; n % 4 == 0, aligned planes):
// the same per-pixel float sums as k_score_dot_max
__global__ void __launch_bounds__(kSgThreads) k_score_dot_max_f32v4(int F, int C, unsigned n4,
                                                                    const float* __restrict__ gin,
                                                                    const float* __restrict__ gd,
                                                                    const float* __restrict__ scores,
                                                                    float* __restrict__ gspp, double* pmax) {
    const int b = blockIdx.y;
    const unsigned n = 4u * n4;
    const float4* sc4 = reinterpret_cast<const float4*>(scores + (size_t)b * n);
    float4* out4 = reinterpret_cast<float4*>(gspp + (size_t)b * n);
    float m = -INFINITY;
    for (unsigned p = blockIdx.x * kSgThreads + threadIdx.x; p < n4; p += gridDim.x * kSgThreads) {
        float tot[4] = {0.f, 0.f, 0.f, 0.f};
        for (int f = 0; f < F; ++f) {
            const float4* g4 = reinterpret_cast<const float4*>(gin + ((size_t)(b * F + f) * C) * n) + p;
            const float4* d4 = reinterpret_cast<const float4*>(gd + ((size_t)(b * F + f) * C) * n) + p;
            float4 gg = __ldcs(g4), dd = __ldcs(d4);
            float sv[4] = {gg.x * dd.x, gg.y * dd.y, gg.z * dd.z, gg.w * dd.w};
            for (int c = 1; c < C; ++c) {
                gg = __ldcs(g4 + (size_t)c * n4);
                dd = __ldcs(d4 + (size_t)c * n4);
                sv[0] = sv[0] + gg.x * dd.x;
                sv[1] = sv[1] + gg.y * dd.y;
                sv[2] = sv[2] + gg.z * dd.z;
                sv[3] = sv[3] + gg.w * dd.w;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) tot[j] = f == 0 ? sv[j] : tot[j] + sv[j];
        }
        out4[p] = make_float4(tot[0], tot[1], tot[2], tot[3]);
        const float4 s4 = __ldg(sc4 + p);
        m = fmaxf(m, fmaxf(fmaxf(s4.x, s4.y), fmaxf(s4.z, s4.w)));
    }
    const double md = sg_block_reduce((double)m, true);
    if (threadIdx.x == 0) pmax[b * kDotBlocks + blockIdx.x] = md;
}

__global__ void k_max_reduce(const double* __restrict__ pmax, double* __restrict__ fmaxv) {
    const int b = blockIdx.x;
    double m = -INFINITY;
    for (int k = threadIdx.x; k < kDotBlocks; k += kSgThreads) m = fmax(m, pmax[b * kDotBlocks + k]);
    m = sg_block_reduce(m, true);
    if (threadIdx.x == 0) fmaxv[b] = m;
}

// blur (axis 0 then axis 1, scipy order) of one 32 x 8 tile from shared
// memory; writes the blurred g and the block's partial sums of e and e * g
template <typename T>
__global__ void __launch_bounds__(SG_TX * SG_TY) k_blur_sums(int H, int W, BlurWeights bw,
                                                             const acc_t<T>* __restrict__ g0,
                                                             const T* __restrict__ scores,
                                                             const double* __restrict__ pmax,
                                                             acc_t<T>* __restrict__ g1, double* __restrict__ pse,
                                                             double* __restrict__ psd) {
    using A = acc_t<T>;
    __shared__ A s_in[(SG_TY + 2 * SG_RMAX) * (SG_TX + 2 * SG_RMAX)];
    __shared__ A s_v[SG_TY * (SG_TX + 2 * SG_RMAX)];
    __shared__ A s_w[SG_RMAX + 1];
    __shared__ double s_m;
    const int b = blockIdx.z, r = bw.r;
    const int x0 = blockIdx.x * SG_TX, y0 = blockIdx.y * SG_TY;
    const int tid = threadIdx.y * SG_TX + threadIdx.x;
    const int nx = SG_TX + 2 * r, ny = SG_TY + 2 * r;
    const A* gb = g0 + (long long)b * H * W;
    if (tid == 0) s_m = pmax[b];  // per-frame max (k_max_reduce)
    if (tid <= r) s_w[tid] = (A)bw.w[tid];
    for (int i = tid; i < nx * ny; i += SG_TX * SG_TY) {
        const int yy = clampi(y0 - r + i / nx, 0, H - 1), xx = clampi(x0 - r + i % nx, 0, W - 1);
        s_in[i] = gb[(long long)yy * W + xx];
    }
    __syncthreads();
    for (int i = tid; i < SG_TY * nx; i += SG_TX * SG_TY) {  // axis 0
        const int ty = i / nx, tx = i % nx;
        const A* c = s_in + (ty + r) * nx + tx;
        A v = c[0] * s_w[0];
        for (int j = r; j >= 1; --j) v = v + (c[-j * nx] + c[j * nx]) * s_w[j];
        s_v[ty * nx + tx] = v;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    double se = 0.0, sd = 0.0;
    if (x < W && y < H) {
        const A* c = s_v + threadIdx.y * nx + threadIdx.x + r;
        A v = c[0] * s_w[0];  // axis 1
        for (int j = r; j >= 1; --j) v = v + (c[-j] + c[j]) * s_w[j];
        const long long o = (long long)b * H * W + (long long)y * W + x;
        g1[o] = v;
        const double e = sg_exp(scores[o], s_m);
        se = e;
        sd = e * (double)v;
    }
    se = sg_block_reduce(se, false);
    sd = sg_block_reduce(sd, false);
    if (tid == 0) {  // (the reduced value lives in thread 0)
        const long long k = ((long long)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        pse[k] = se;
        psd[k] = sd;
    }
}

// acc + x * y: float64 rounds the product (scipy's order; the file is built
// with -fmad=false), float32 fuses it
__device__ __forceinline__ double madd(double x, double y, double acc) { return acc + x * y; }
__device__ __forceinline__ float madd(float x, float y, float acc) { return __fmaf_rn(x, y, acc); }

// compile-time radius R, float32: 64 x 16 tile per CTA, register-blocked --
// the vertical pass gives each thread 4 consecutive rows of one column (4 + 2R
// shared loads for 4 outputs), the horizontal pass 4 consecutive columns of
// one row (16-B shared loads); every output keeps scipy's sum order
// (x_i w0 + sum_{j = R..1} (x_{i-j} + x_{i+j}) w_j)
constexpr int SB_TX = 64, SB_TY = 16;

template <int R>
struct BlurTile {
    static constexpr int NX = SB_TX + 2 * R, NY = SB_TY + 2 * R, NWIN = NX * NY;
    static constexpr int NXP = (NX + 3) & ~3;      // 16-B row pitch of the vertical-pass output
    static constexpr int VOFF = (NWIN + 3) & ~3;   // s_v offset (16-B aligned)
    static constexpr int NB = 4 + 2 * R, NV4 = (NB + 3) / 4;
    static constexpr size_t BYTES = (size_t)(VOFF + SB_TY * NXP) * sizeof(float);
};

template <typename T, int R>
__global__ void __launch_bounds__(256) k_blur_sums_r(int H, int W, BlurWeights bw, const acc_t<T>* __restrict__ g0,
                                                     const T* __restrict__ scores, const double* __restrict__ pmax,
                                                     acc_t<T>* __restrict__ g1, double* __restrict__ pse,
                                                     double* __restrict__ psd) {
    static_assert(sizeof(T) == 4, "float32 path");
    using TT = BlurTile<R>;
    constexpr int NX = TT::NX, NWIN = TT::NWIN, NXP = TT::NXP, NB = TT::NB;
    extern __shared__ __align__(16) unsigned char smem_blur[];
    float* s_in = reinterpret_cast<float*>(smem_blur);  // [NY][NX]
    float* s_v = s_in + TT::VOFF;                        // [SB_TY][NXP]
    const int b = blockIdx.z, tid = threadIdx.x;
    const int x0 = blockIdx.x * SB_TX, y0 = blockIdx.y * SB_TY;
    const float* gb = g0 + (size_t)b * H * W;
    float w[R + 1];
#pragma unroll
    for (int j = 0; j <= R; ++j) w[j] = (float)bw.w[j];
    const double m = pmax[b];
    constexpr int NIT = (NWIN + 255) / 256;
    float v[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {  // every load issued before the stores
        const int i = tid + it * 256;
        const int wy = i / NX, wx = i - wy * NX;
        const int yy = clampi(y0 - R + wy, 0, H - 1), xx = clampi(x0 - R + wx, 0, W - 1);
        v[it] = i < NWIN ? gb[(size_t)yy * W + xx] : 0.f;
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it)
        if (tid + it * 256 < NWIN) s_in[tid + it * 256] = v[it];
    __syncthreads();
    for (int i = tid; i < (SB_TY / 4) * NX; i += 256) {  // axis 0: rows 4 q4 .. 4 q4 + 3 of column tx
        const int q4 = i / NX, tx = i - q4 * NX;
        const float* c = s_in + 4 * q4 * NX + tx;  // window row 0 = output row 4 q4 - R
        float col[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) col[k] = c[k * NX];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float a = col[q + R] * w[0];
#pragma unroll
            for (int j = R; j >= 1; --j) a = madd(col[q + R - j] + col[q + R + j], w[j], a);
            s_v[(4 * q4 + q) * NXP + tx] = a;
        }
    }
    __syncthreads();
    // axis 1: row ty, columns 4 lq .. 4 lq + 3
    const int ty = tid >> 4, lq = tid & 15, y = y0 + ty, xq = x0 + 4 * lq;
    double se = 0.0, sd = 0.0;
    if (y < H && xq < W) {
        float row[4 * TT::NV4];
        const float4* r4 = reinterpret_cast<const float4*>(s_v + ty * NXP + 4 * lq);
#pragma unroll
        for (int k = 0; k < TT::NV4; ++k) {
            const float4 t = r4[k];
            row[4 * k] = t.x;
            row[4 * k + 1] = t.y;
            row[4 * k + 2] = t.z;
            row[4 * k + 3] = t.w;
        }
        float out[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float a = row[q + R] * w[0];
#pragma unroll
            for (int j = R; j >= 1; --j) a = madd(row[q + R - j] + row[q + R + j], w[j], a);
            out[q] = a;
        }
        const size_t o = (size_t)b * H * W + (size_t)y * W + xq;
        float sc[4];
        const bool vec = (W & 3) == 0 && xq + 3 < W && (reinterpret_cast<size_t>(scores) & 15) == 0 &&
                         (reinterpret_cast<size_t>(g1) & 15) == 0;
        if (vec) {
            const float4 s4 = __ldg(reinterpret_cast<const float4*>(scores + o));
            sc[0] = s4.x;
            sc[1] = s4.y;
            sc[2] = s4.z;
            sc[3] = s4.w;
            *reinterpret_cast<float4*>(g1 + o) = make_float4(out[0], out[1], out[2], out[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (xq + q >= W) break;
            if (!vec) {
                sc[q] = scores[o + q];
                g1[o + q] = out[q];
            }
            const double e = sg_exp(sc[q], m);
            se += e;
            sd += e * (double)out[q];
        }
    }
    se = sg_block_reduce(se, false);
    sd = sg_block_reduce(sd, false);
    if (tid == 0) {
        const long long k = ((long long)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        pse[k] = se;
        psd[k] = sd;
    }
}

template <typename T, int R>
size_t blur_r_smem() {
    return BlurTile<R>::BYTES;
}

// per-frame totals of the tile partials (fixed order: deterministic)
__global__ void k_sums_reduce(int nblk, const double* __restrict__ pse, const double* __restrict__ psd,
                              double* __restrict__ tot) {
    const int b = blockIdx.x;
    double se = 0.0, sd = 0.0;
    for (int k = threadIdx.x; k < nblk; k += kSgThreads) {
        se += pse[(long long)b * nblk + k];
        sd += psd[(long long)b * nblk + k];
    }
    se = sg_block_reduce(se, false);
    sd = sg_block_reduce(sd, false);
    if (threadIdx.x == 0) {
        tot[2 * b] = se;
        tot[2 * b + 1] = sd;
    }
}

template <typename T>
__global__ void k_sg_apply_tot(long long n, const T* __restrict__ scores, const acc_t<T>* __restrict__ g,
                               const double* pmax, const double* __restrict__ tot, double total, T* __restrict__ out) {
    const int b = blockIdx.y;
    __shared__ double sm, ss, inner;
    if (threadIdx.x == 0) {
        sm = pmax[b];
        ss = tot[2 * b];
        inner = tot[2 * b + 1] / ss;  // sum(w * g)
    }
    __syncthreads();
    for (long long i = (long long)blockIdx.x * kSgThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kSgThreads) {
        const double w = sg_exp(scores[(long long)b * n + i], sm) / ss;
        out[(long long)b * n + i] = (T)(total * (w * ((double)g[(long long)b * n + i] - inner)));
    }
}

// float32 apply, four pixels per thread; w = e * (1 / sum e) (<= 1 ulp of
// float64 off the division, far below the float32 output rounding)
__global__ void __launch_bounds__(kSgThreads) k_sg_apply_f32v4(unsigned n4, const float* __restrict__ scores,
                                                               const float* __restrict__ g, const double* pmax,
                                                               const double* __restrict__ tot, double total,
                                                               float* __restrict__ out) {
    const int b = blockIdx.y;
    const unsigned n = 4u * n4;
    const double sm = pmax[b], rs = 1.0 / tot[2 * b], inner = tot[2 * b + 1] / tot[2 * b];
    const float4* s4 = reinterpret_cast<const float4*>(scores + (size_t)b * n);
    const float4* g4 = reinterpret_cast<const float4*>(g + (size_t)b * n);
    float4* o4 = reinterpret_cast<float4*>(out + (size_t)b * n);
    for (unsigned i = blockIdx.x * kSgThreads + threadIdx.x; i < n4; i += gridDim.x * kSgThreads) {
        const float4 sv = __ldcs(s4 + i), gv = __ldcs(g4 + i);
        const float ss[4] = {sv.x, sv.y, sv.z, sv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w};
        float r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = (float)(total * ((sg_exp(ss[j], sm) * rs) * ((double)gg[j] - inner)));
        __stcs(o4 + i, make_float4(r[0], r[1], r[2], r[3]));
    }
}

template <typename T, int R>
bool launch_blur_r(int r, dim3 grid, int H, int W, const BlurWeights& bw, const acc_t<T>* g0, const T* sc,
                   const double* fmx, acc_t<T>* g1, double* pse, double* psd, cudaStream_t s) {
    if constexpr (R > SG_RMAX) {
        return false;
    } else {
        if (r != R) return launch_blur_r<T, R + 1>(r, grid, H, W, bw, g0, sc, fmx, g1, pse, psd, s);
        static std::atomic<unsigned long long> attr_mask{0};
        smem_attr_once(attr_mask, (const void*)k_blur_sums_r<T, R>, (int)blur_r_smem<T, R>());
        SSB_LAUNCH(s, k_blur_sums_r<T, R><<<grid, 256, blur_r_smem<T, R>(), s>>>(H, W, bw, g0, sc, fmx, g1, pse, psd));
        return true;
    }
}

template <typename T>
int score_grad_fused(int B, int F, int C, int H, int W, const T* gin, const T* gd, const T* sc, double total,
                     const BlurWeights& bw, T* out, char* ws, cudaStream_t s) {
    const long long n = (long long)H * W;
    using A = acc_t<T>;
    A* g0 = (A*)ws;
    A* g1 = g0 + (size_t)B * n;
    // f32: the radius-templated 64 x 16 tiles; f64 (parity mode): 32 x 8
    constexpr bool RT = sizeof(T) == 4;
    dim3 tgrid = RT ? dim3((W + SB_TX - 1) / SB_TX, (H + SB_TY - 1) / SB_TY, B)
                    : dim3((W + SG_TX - 1) / SG_TX, (H + SG_TY - 1) / SG_TY, B);
    const int nblk = tgrid.x * tgrid.y;
    double* pmax = (double*)(ws + 2 * (size_t)B * n * sizeof(double));  // B x kDotBlocks
    double* fmx = pmax + (size_t)B * kDotBlocks;  // B
    double* pse = fmx + B;
    double* psd = pse + (size_t)B * nblk;
    double* tot = psd + (size_t)B * nblk;
    bool v4 = false;
    if constexpr (RT) {
        v4 = n % 4 == 0 && 3 * n < (1ll << 31);
        for (const void* q : {(const void*)gin, (const void*)gd, (const void*)sc, (const void*)out})
            if (reinterpret_cast<size_t>(q) & 15) v4 = false;
    }
    if (v4)
        SSB_LAUNCH(s, k_score_dot_max_f32v4<<<dim3(kDotBlocks, B), kSgThreads, 0, s>>>(
                          F, C, (unsigned)(n / 4), (const float*)gin, (const float*)gd, (const float*)sc,
                          (float*)g0, pmax));
    else
        SSB_LAUNCH(s, k_score_dot_max<T><<<dim3(kDotBlocks, B), kSgThreads, 0, s>>>(F, C, n, gin, gd, sc, g0, pmax));
    SSB_LAUNCH(s, k_max_reduce<<<B, kSgThreads, 0, s>>>(pmax, fmx));
    if constexpr (RT) {
        if (!launch_blur_r<T, 0>(bw.r, tgrid, H, W, bw, g0, sc, fmx, g1, pse, psd, s)) return SSB_EUNSUPPORTED;
    } else {
        SSB_LAUNCH(s, k_blur_sums<T><<<tgrid, dim3(SG_TX, SG_TY), 0, s>>>(H, W, bw, g0, sc, fmx, g1, pse, psd));
    }
    SSB_LAUNCH(s, k_sums_reduce<<<B, kSgThreads, 0, s>>>(nblk, pse, psd, tot));
    const unsigned ag = (unsigned)((n + kSgThreads - 1) / kSgThreads < 4096 ? (n + kSgThreads - 1) / kSgThreads : 4096);
    if (v4)
        SSB_LAUNCH(s, k_sg_apply_f32v4<<<dim3((ag + 3) / 4, B), kSgThreads, 0, s>>>(
                          (unsigned)(n / 4), (const float*)sc, (const float*)g1, fmx, tot, total, (float*)out));
    else
        SSB_LAUNCH(s, k_sg_apply_tot<T><<<dim3(ag, B), kSgThreads, 0, s>>>(n, sc, g1, fmx, tot, total, out));
    return 0;
}

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_score_grad_workspace_bytes(int B, int H, int W, size_t* bytes) {
    if (B <= 0 || H <= 0 || W <= 0 || !bytes) {
        set_error("ssb_score_grad_workspace_bytes: invalid arguments");
        return SSB_EINVAL;
    }
    const size_t n = (size_t)H * W;
    const size_t nblk = (size_t)((W + SG_TX - 1) / SG_TX) * ((H + SG_TY - 1) / SG_TY);
    *bytes = (2 * (size_t)B * n + (size_t)B * (kDotBlocks > 3 * kSgBlocks ? kDotBlocks : 3 * kSgBlocks) +
              (size_t)B + 2 * (size_t)B * nblk + 2 * (size_t)B) * sizeof(double);
    return 0;
}

int ssb_score_grad(int dtype, int B, int F, int C, int H, int W, const void* g_input,
                   const void* grad_density, const void* scores, double budget, double sigma,
                   void* g_scores, void* workspace, ssb_stream_t stream) {
    if (B <= 0 || F <= 0 || C <= 0 || H <= 0 || W <= 0 || !g_input || !grad_density || !scores ||
        !g_scores || !workspace || !(sigma >= 0.0)) {
        set_error("ssb_score_grad: invalid arguments");
        return SSB_EINVAL;
    }
    if (dtype != SSB_F32 && dtype != SSB_F64) {
        set_error("ssb_score_grad: dtype must be f32 or f64");
        return SSB_EUNSUPPORTED;
    }
    BlurWeights bw{};
    if (sigma > 0.0) {
        bw.r = (int)(4.0 * sigma + 0.5);  // scipy truncate = 4.0
        if (bw.r > kMaxBlurRadius) {
            set_error("ssb_score_grad: blur radius above 64");
            return SSB_EUNSUPPORTED;
        }
        std::vector<double> phi(2 * bw.r + 1);
        double tot = 0.0;
        for (int i = -bw.r; i <= bw.r; ++i) {
            phi[i + bw.r] = exp(-0.5 / (sigma * sigma) * (double)(i * i));
            tot += phi[i + bw.r];
        }
        for (int j = 0; j <= bw.r; ++j) bw.w[j] = phi[bw.r + j] / tot;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = (long long)H * W;
    if (bw.r <= SG_RMAX) {
        if (sigma == 0.0) {
            bw.r = 0;
            bw.w[0] = 1.0;  // identity "blur": the tile pass only forms the sums
        }
        const double tot = (7.0 / 8.0) * budget * (double)n;
        if (dtype == SSB_F64)
            score_grad_fused<double>(B, F, C, H, W, (const double*)g_input, (const double*)grad_density,
                                     (const double*)scores, tot, bw, (double*)g_scores, (char*)workspace, s);
        else
            score_grad_fused<float>(B, F, C, H, W, (const float*)g_input, (const float*)grad_density,
                                    (const float*)scores, tot, bw, (float*)g_scores, (char*)workspace, s);
        return cuda_check("ssb_score_grad");
    }
    double* g0 = (double*)workspace;
    double* g1 = g0 + (size_t)B * n;
    double* pmax = g1 + (size_t)B * n;
    double* psum = pmax + (size_t)B * kSgBlocks;
    double* pdot = psum + (size_t)B * kSgBlocks;
    const double total = (7.0 / 8.0) * budget * (double)n;
    dim3 pgrid((unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), B);
    dim3 block2(32, 8), grid2((W + 31) / 32, (H + 7) / 8, B);
    dim3 rgrid(kSgBlocks, B);
    const double* g = g0;
    if (dtype == SSB_F64)
        SSB_LAUNCH(s, k_score_dot<double><<<pgrid, 256, 0, s>>>(F, C, n, (const double*)g_input,
                                                              (const double*)grad_density, g0));
    else
        SSB_LAUNCH(s, k_score_dot<float><<<pgrid, 256, 0, s>>>(F, C, n, (const float*)g_input,
                                                             (const float*)grad_density, g0));
    if (sigma > 0.0) {
        SSB_LAUNCH(s, k_blur_axis<<<grid2, block2, 0, s>>>(H, W, 0, bw, g0, g1));
        SSB_LAUNCH(s, k_blur_axis<<<grid2, block2, 0, s>>>(H, W, 1, bw, g1, g0));
    }
    if (dtype == SSB_F64) {
        const double* sc = (const double*)scores;
        SSB_LAUNCH(s, k_sg_partial_max<double><<<rgrid, kSgThreads, 0, s>>>(n, sc, pmax));
        SSB_LAUNCH(s, k_sg_partial_sums<double><<<rgrid, kSgThreads, 0, s>>>(n, sc, g, pmax, psum, pdot));
        SSB_LAUNCH(s, k_sg_apply<double><<<rgrid, kSgThreads, 0, s>>>(n, sc, g, pmax, psum, pdot, total,
                                                                    (double*)g_scores));
    } else {
        const float* sc = (const float*)scores;
        SSB_LAUNCH(s, k_sg_partial_max<float><<<rgrid, kSgThreads, 0, s>>>(n, sc, pmax));
        SSB_LAUNCH(s, k_sg_partial_sums<float><<<rgrid, kSgThreads, 0, s>>>(n, sc, g, pmax, psum, pdot));
        SSB_LAUNCH(s, k_sg_apply<float><<<rgrid, kSgThreads, 0, s>>>(n, sc, g, pmax, psum, pdot, total,
                                                                   (float*)g_scores));
    }
    return cuda_check("ssb_score_grad");
}

}  // extern "C"
