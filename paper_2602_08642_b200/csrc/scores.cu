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

__device__ __forceinline__ double sg_block_reduce(double v, bool is_max) {
    __shared__ double sh[kSgThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, t) : v + t;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < kSgThreads / 32 ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.0);
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmax(v, t) : v + t;
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

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_score_grad_workspace_bytes(int B, int H, int W, size_t* bytes) {
    if (B <= 0 || H <= 0 || W <= 0 || !bytes) {
        set_error("ssb_score_grad_workspace_bytes: invalid arguments");
        return SSB_EINVAL;
    }
    const size_t n = (size_t)H * W;
    *bytes = 2 * (size_t)B * n * sizeof(double) + 3 * (size_t)B * kSgBlocks * sizeof(double);
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
