// Surface primitives of the reference's pyramid module, planar on device:
// normalize_kernels (softmax over channels), gather5 (k x k), upsample2 and
// _avgpool2 (pyramid.py:93-115, 140-149, 173-187, 216-241).  These back the
// compat layer's one-off calls; the fused filter path does not use them.
#include <string>

#include "pyr_kernels.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

template <typename T>
__global__ void k_softmax_channels(int C, int H, int W, int active, const T* __restrict__ in,
                                   T* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const long long hw = (long long)H * W;
    const T* p = in + b * C * hw + (long long)y * W + x;
    T* q = out + b * C * hw + (long long)y * W + x;
    T m = p[0];
    for (int c = 1; c < active; ++c) m = tmax(m, p[c * hw]);
    T s = (T)0;
    for (int c = 0; c < active; ++c) s += sexp(p[c * hw] - m);
    for (int c = 0; c < C; ++c) q[c * hw] = c < active ? sexp(p[c * hw] - m) / s : (T)0;
}

template <typename T>
__global__ void k_gather(int C, int H, int W, int K, const T* __restrict__ img,
                         const T* __restrict__ wts, T* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const int R = K / 2;
    const long long hw = (long long)H * W;
    for (int c = 0; c < C; ++c) {
        const T* ip = img + (b * C + c) * hw;
        T acc = (T)0;
        for (int t = 0; t < K * K; ++t) {
            const int dy = t / K - R, dx = t % K - R;
            const int yy = clampi(y + dy, 0, H - 1), xx = clampi(x + dx, 0, W - 1);
            acc += wts[(b * K * K + t) * hw + (long long)y * W + x] * ip[(long long)yy * W + xx];
        }
        out[(b * C + c) * hw + (long long)y * W + x] = acc;
    }
}

template <typename T>
__global__ void k_upsample2(int C, int Hc, int Wc, int Hf, int Wf, const T* __restrict__ coarse,
                            const T* __restrict__ wts, T* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= Wf || y >= Hf) return;
    const long long hwf = (long long)Hf * Wf, hwc = (long long)Hc * Wc;
    const int iy[2] = {min(y >> 1, Hc - 1), min((y + 1) >> 1, Hc - 1)};
    const int ix[2] = {min(x >> 1, Wc - 1), min((x + 1) >> 1, Wc - 1)};
    for (int c = 0; c < C; ++c) {
        const T* cp = coarse + (b * C + c) * hwc;
        T acc = (T)0;
        for (int t = 0; t < 4; ++t)
            acc += wts[(b * 4 + t) * hwf + (long long)y * Wf + x] * cp[iy[t >> 1] * Wc + ix[t & 1]];
        out[(b * C + c) * hwf + (long long)y * Wf + x] = acc;
    }
}

template <typename T>
static int prim_softmax(int B, int C, int H, int W, int active, const void* in, void* out,
                        cudaStream_t s) {
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    SSB_LAUNCH(s, k_softmax_channels<T><<<grid, block, 0, s>>>(C, H, W, active, (const T*)in, (T*)out));
    return cuda_check("ssb_softmax_channels");
}

}  // namespace ssb

using namespace ssb;

static int check_dims(int dtype, int B, int C, int H, int W) {
    if (dtype != SSB_F32 && dtype != SSB_F64) {
        set_error("dtype must be SSB_F32 or SSB_F64");
        return SSB_EUNSUPPORTED;
    }
    if (B < 1 || C < 1 || H < 1 || W < 1) {
        set_error("dimensions must be >= 1");
        return SSB_EINVAL;
    }
    return SSB_OK;
}

extern "C" {

int ssb_softmax_channels(int dtype, int B, int C, int H, int W, int active, const void* logits,
                         void* weights, ssb_stream_t stream) {
    int rc = check_dims(dtype, B, C, H, W);
    if (rc) return rc;
    if (active < 1 || active > C || !logits || !weights) {
        set_error("ssb_softmax_channels: need 1 <= active <= C and non-null buffers");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SSB_F32 ? prim_softmax<float>(B, C, H, W, active, logits, weights, s)
                            : prim_softmax<double>(B, C, H, W, active, logits, weights, s);
}

int ssb_gather(int dtype, int B, int C, int H, int W, int ksize, const void* image,
               const void* weights, void* out, ssb_stream_t stream) {
    int rc = check_dims(dtype, B, C, H, W);
    if (rc) return rc;
    if (ksize < 1 || (ksize & 1) == 0 || !image || !weights || !out) {
        set_error("ssb_gather: ksize must be odd and buffers non-null");
        return SSB_EINVAL;
    }
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SSB_F32)
        SSB_LAUNCH(s, k_gather<float><<<grid, block, 0, s>>>(C, H, W, ksize, (const float*)image,
                                               (const float*)weights, (float*)out));
    else
        SSB_LAUNCH(s, k_gather<double><<<grid, block, 0, s>>>(C, H, W, ksize, (const double*)image,
                                                (const double*)weights, (double*)out));
    return cuda_check("ssb_gather");
}

int ssb_upsample2(int dtype, int B, int C, int Hc, int Wc, int Hf, int Wf, const void* coarse,
                  const void* weights, void* out, ssb_stream_t stream) {
    int rc = check_dims(dtype, B, C, Hf, Wf);
    if (rc) return rc;
    if (Hc < 1 || Wc < 1 || !coarse || !weights || !out) {
        set_error("ssb_upsample2: bad coarse dims or null buffer");
        return SSB_EINVAL;
    }
    dim3 block(32, 8), grid((Wf + 31) / 32, (Hf + 7) / 8, B);
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SSB_F32)
        SSB_LAUNCH(s, k_upsample2<float><<<grid, block, 0, s>>>(C, Hc, Wc, Hf, Wf, (const float*)coarse,
                                                  (const float*)weights, (float*)out));
    else
        SSB_LAUNCH(s, k_upsample2<double><<<grid, block, 0, s>>>(C, Hc, Wc, Hf, Wf, (const double*)coarse,
                                                   (const double*)weights, (double*)out));
    return cuda_check("ssb_upsample2");
}

int ssb_avgpool2(int dtype, int B, int C, int H, int W, const void* in, void* out,
                 ssb_stream_t stream) {
    int rc = check_dims(dtype, B, C, H, W);
    if (rc) return rc;
    if (!in || !out) {
        set_error("ssb_avgpool2: null buffer");
        return SSB_EINVAL;
    }
    const long long hw = (long long)H * W;
    const long long hwc = (long long)((H + 1) / 2) * ((W + 1) / 2);
    cudaStream_t s = (cudaStream_t)stream;
    dim3 block(32, 8), grid(((W + 1) / 2 + 31) / 32, ((H + 1) / 2 + 7) / 8, B);
    if (dtype == SSB_F32)
        SSB_LAUNCH(s, k_pool2<float><<<grid, block, 0, s>>>(C, H, W, (const float*)in, C * hw, hw, nullptr,
                                              (float*)out, C * hwc, hwc));
    else
        SSB_LAUNCH(s, k_pool2<double><<<grid, block, 0, s>>>(C, H, W, (const double*)in, C * hw, hw, nullptr,
                                               (double*)out, C * hwc, hwc));
    return cuda_check("ssb_avgpool2");
}

}  // extern "C"
