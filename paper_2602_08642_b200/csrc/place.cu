// Sample placement: counter-based uniforms, frame-global density softmax,
// stochastic-rounding allocation, estimator core and the fused inference path.
//
// Reference: pkg/src/sparse_sampler/rng.py:21-63, density.py:43-65,196-233,
// estimators.py:70-149.  All decision arithmetic is IEEE float64 and this TU
// is compiled with -fmad=false so that elementwise results (floor/frac, u,
// u < frac, the estimator formulas) are bit-identical to numpy's.
#include <string>

#include "common.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

// ---------------------------------------------------------------- RNG
constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kM1;
    z = (z ^ (z >> 27)) * kM2;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t key_hash(uint64_t seed, uint64_t frame, uint64_t x, uint64_t y,
                                             uint64_t stream) {
    uint64_t h = mix64(seed + kGold);
    h = mix64(h ^ (frame * kGold + kGold));
    h = mix64(h ^ (x * kGold + kGold));
    h = mix64(h ^ (y * kGold + kGold));
    h = mix64(h ^ (stream * kGold + kGold));
    return h;
}

__device__ __forceinline__ double key_uniform(uint64_t seed, uint64_t frame, uint64_t x,
                                              uint64_t y, uint64_t stream) {
    return (double)(key_hash(seed, frame, x, y, stream) >> 11) * 0x1.0p-53;
}

__global__ void k_uniform_grid(uint64_t seed, int64_t frame0, const int64_t* frames, int H, int W,
                               uint64_t stream, double* u) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= W || y >= H) return;
    const uint64_t f = (uint64_t)(frames ? frames[b] : frame0 + b);
    u[((long long)b * H + y) * W + x] = key_uniform(seed, f, (uint64_t)x, (uint64_t)y, stream);
}

// ---------------------------------------------------------------- estimator math
constexpr double kGateFloor = 1e-4;
constexpr double kLogitClamp = 1e-6;

__device__ __forceinline__ double clipd(double v, double lo, double hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

__device__ __forceinline__ double gumbel_gate(double u, double frac, double temp) {
    const double pc = clipd(frac, kLogitClamp, 1.0 - kLogitClamp);
    const double uc = clipd(u, kLogitClamp, 1.0 - kLogitClamp);
    const double z = (((log(pc) - log1p(-pc)) + log(uc)) - log1p(-uc)) / temp;
    return 1.0 / (1.0 + exp(-z));
}

__device__ __forceinline__ bool take_rule(int rule, double u, double frac, double temp) {
    if (rule == SSB_RULE_STOCHASTIC) return u < frac;
    if (rule == SSB_RULE_RELAXED) return (frac > 0.0) && (u >= 1.0 - frac);
    return gumbel_gate(u, frac, temp) > kGateFloor;
}

struct CoreOut {
    double noisy[3], grad[3], contrib[3];
    bool drawn;
};

// stochastic_core for one pixel (estimators.py:90-133)
__device__ __forceinline__ CoreOut core_pixel(int variant, double spp, double frac, double u,
                                              const double* bsum, const double* hold, double lam,
                                              double temp, double floor_) {
    CoreOut o;
    const double s = spp > floor_ ? spp : floor_;
    if (variant == SSB_VAR_STOCHASTIC) {
        o.drawn = u < frac;
        for (int c = 0; c < 3; ++c) {
            o.contrib[c] = o.drawn ? hold[c] : 0.0;
            o.noisy[c] = (bsum[c] + o.contrib[c]) / s;
            o.grad[c] = -o.noisy[c] / s;
        }
    } else if (variant == SSB_VAR_RELAXED) {
        const double raw = frac > 0.0 ? (u + frac - 1.0) / frac : 0.0;
        const double ramp = clipd(lam * raw, 0.0, 1.0);
        const double gain = 2.0 * lam / (2.0 * lam - 1.0);
        o.drawn = (frac > 0.0) && (u >= 1.0 - frac);
        const bool linear = o.drawn && (ramp < 1.0);
        const double slope = linear ? lam * (1.0 - u) / (frac * frac) : 0.0;
        const double gr = gain * ramp, gs = gain * slope;
        for (int c = 0; c < 3; ++c) {
            o.contrib[c] = o.drawn ? hold[c] * gr : 0.0;
            o.noisy[c] = (bsum[c] + o.contrib[c]) / s;
            o.grad[c] = (hold[c] * gs - o.noisy[c]) / s;
        }
    } else if (variant == SSB_VAR_STRAIGHT_THROUGH) {
        const bool taken = u < frac;
        o.drawn = frac > 0.0;
        for (int c = 0; c < 3; ++c) {
            o.contrib[c] = taken ? hold[c] : 0.0;
            o.noisy[c] = (bsum[c] + o.contrib[c]) / s;
            o.grad[c] = ((o.drawn ? hold[c] : 0.0) - o.noisy[c]) / s;
        }
    } else {
        const double gate = gumbel_gate(u, frac, temp);
        o.drawn = gate > kGateFloor;
        const double pc = clipd(frac, kLogitClamp, 1.0 - kLogitClamp);
        const double dgate = (frac > kLogitClamp && frac < 1.0 - kLogitClamp)
                                 ? gate * (1.0 - gate) / (temp * pc * (1.0 - pc))
                                 : 0.0;
        for (int c = 0; c < 3; ++c) {
            o.contrib[c] = o.drawn ? hold[c] * gate : 0.0;
            o.noisy[c] = (bsum[c] + o.contrib[c]) / s;
            o.grad[c] = ((o.drawn ? hold[c] * dgate : 0.0) - o.noisy[c]) / s;
        }
    }
    return o;
}

__global__ void k_stochastic_core(ssb_estimate_desc d, long long n, const double* spp,
                                  const double* frac, const double* u, const double* bsum,
                                  const double* hold, double* noisy, double* grad,
                                  double* contrib, uint8_t* drawn) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    CoreOut o = core_pixel(d.variant, spp[i], frac[i], u[i], bsum + 3 * i, hold + 3 * i, d.lam,
                           d.gumbel_temp, d.density_floor);
    for (int c = 0; c < 3; ++c) {
        if (noisy) noisy[3 * i + c] = o.noisy[c];
        if (grad) grad[3 * i + c] = o.grad[c];
        if (contrib) contrib[3 * i + c] = o.contrib[c];
    }
    if (drawn) drawn[i] = o.drawn;
}

// _stochastic_estimate with the SampleBank read (banks.py:61-73) fused
__global__ void k_estimate(ssb_estimate_desc d, int H, int W, const double* spp,
                           const int64_t* base, const double* frac, const double* u,
                           const double* samples, double* noisy, double* grad, double* contrib,
                           int64_t* used, float* noisy32) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long hw = (long long)H * W;
    const long long n = hw * d.B;
    if (i >= n) return;
    const int S = d.capacity;
    const int64_t bi = base[i];
    const int idx = (int)(bi < S - 1 ? bi : S - 1);
    const double* sp = samples + i * S * 3;
    double bs[3] = {0.0, 0.0, 0.0}, ho[3];
    for (int j = 0; j < idx; ++j)
        for (int c = 0; c < 3; ++c) bs[c] += sp[j * 3 + c];
    for (int c = 0; c < 3; ++c) ho[c] = sp[idx * 3 + c];
    CoreOut o = core_pixel(d.variant, spp[i], frac[i], u[i], bs, ho, d.lam, d.gumbel_temp,
                           d.density_floor);
    const long long b = i / hw, p = i - b * hw;
    for (int c = 0; c < 3; ++c) {
        const double nv = o.noisy[c] > 0.0 ? o.noisy[c] : 0.0;
        if (noisy) noisy[3 * i + c] = nv;
        if (grad) grad[3 * i + c] = o.grad[c];
        if (contrib) contrib[3 * i + c] = o.contrib[c];
        if (noisy32) noisy32[(b * 3 + c) * hw + p] = (float)nv;
    }
    if (used) used[i] = (int64_t)idx + (o.drawn ? 1 : 0);
}

// ---------------------------------------------------------------- allocation
__global__ void k_allocate(ssb_alloc_desc d, const double* spp, const int64_t* rank,
                           int64_t* base, double* frac, double* u, uint8_t* taken) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= d.W || y >= d.H) return;
    const long long i = ((long long)b * d.H + y) * d.W + x;
    const long long frame = d.frame0 + b;
    const double s = spp[i];
    const double fl = floor(s);
    const double fr = s - fl;
    double uv;
    if (d.dithered) {
        const int t = d.mask_size;
        const int sy = (int)((frame * 7) % t), sx = (int)((frame * 13) % t);
        uv = ((double)rank[((y + sy) % t) * t + (x + sx) % t] + 0.5) / (double)(t * t);
    } else {
        uv = key_uniform(d.seed, (uint64_t)frame, (uint64_t)x, (uint64_t)y, 0);
    }
    if (base) base[i] = (int64_t)fl;
    if (frac) frac[i] = fr;
    if (u) u[i] = uv;
    if (taken) taken[i] = take_rule(d.rule, uv, fr, d.gumbel_temp);
}

// ---------------------------------------------------------------- frame-global softmax
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 1024;  // partials per frame

__device__ __forceinline__ double block_reduce(double v, bool is_max) {
    __shared__ double sh[kRedThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, w) : v + w;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < kRedThreads / 32 ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.0);
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmax(v, w) : v + w;
        }
    }
    __syncthreads();
    return v;
}

template <typename TS>
__global__ void k_partial_max(long long n, const TS* scores, double* pmax) {
    const int b = blockIdx.y;
    const TS* p = scores + (long long)b * n;
    double m = -INFINITY;
    for (long long i = (long long)blockIdx.x * kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads)
        m = fmax(m, (double)p[i]);
    m = block_reduce(m, true);
    if (threadIdx.x == 0) pmax[b * kRedBlocks + blockIdx.x] = m;
}

// the frame's max / sum of the block partials, once per frame: out[2b] = max,
// out[2b+1] = sum (when psum given).  Each thread folds a strided subset in
// order, then a fixed shuffle tree (deterministic; launched with kRedThreads)
__global__ void k_frame_stats(const double* pmax, const double* psum, double* out, int nblk) {
    const int b = blockIdx.x;
    const bool is_max = psum == nullptr;
    const double* src = (is_max ? pmax : psum) + (size_t)b * kRedBlocks;
    double v = is_max ? -INFINITY : 0.0;
    for (int k = threadIdx.x; k < nblk; k += blockDim.x) v = is_max ? fmax(v, src[k]) : v + src[k];
    v = block_reduce(v, is_max);
    if (threadIdx.x == 0) out[2 * b + (is_max ? 0 : 1)] = v;
}

template <typename TS>
__global__ void k_partial_sum(long long n, const TS* scores, const double* fstat, double* psum) {
    const int b = blockIdx.y;
    const double m = fstat[2 * b];
    const TS* p = scores + (long long)b * n;
    double s = 0.0;
#pragma unroll 4
    for (long long i = (long long)blockIdx.x * kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads)
        s += exp((double)p[i] - m);
    s = block_reduce(s, false);
    if (threadIdx.x == 0) psum[b * kRedBlocks + blockIdx.x] = s;
}


// spp = budget/8 + (7/8 * budget * N) * (e / sum)   (density.py:63-64)
__global__ void k_density_apply(long long n, const double* scores, const double* fstat, double budget,
                                double* spp) {
    const int b = blockIdx.y;
    const double sm = fstat[2 * b], ss = fstat[2 * b + 1];
    const double adaptive = (1.0 - 0.125) * budget * (double)n;
    for (long long i = (long long)blockIdx.x * kRedThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kRedThreads) {
        const double e = exp(scores[(long long)b * n + i] - sm);
        spp[(long long)b * n + i] = 0.125 * budget + adaptive * (e / ss);
    }
}

// fused inference placement: scores f32 -> spp -> counts/mask -> noisy f32
__global__ void k_place_fused(ssb_place_desc d, const float* scores, const double* fstat, const float* bank,
                              float* noisy, float* spp_out, uint8_t* taken_out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= d.W || y >= d.H) return;
    const double sm = fstat[2 * b], ss = fstat[2 * b + 1];
    const long long hw = (long long)d.H * d.W, p = (long long)y * d.W + x;
    const double adaptive = (1.0 - 0.125) * d.budget * (double)hw;
    const double e = exp((double)scores[b * hw + p] - sm);
    const double spp = 0.125 * d.budget + adaptive * (e / ss);
    const double fl = floor(spp);
    const double fr = spp - fl;
    const double uv = key_uniform(d.seed, (uint64_t)(d.frame0 + b), (uint64_t)x, (uint64_t)y, 0);
    const bool taken = uv < fr;
    const int S = d.capacity;
    const int idx = (int)(fl < (double)(S - 1) ? fl : (double)(S - 1));
    const double sden = spp > 1e-8 ? spp : 1e-8;
    const double rs = 1.0 / sden;  // one division; the float32 result rounds the same to ~1 ulp
    const float* bp = bank + (long long)b * S * 3 * hw + p;
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int j = 0; j < idx; ++j) acc += (double)bp[(j * 3 + c) * hw];
        if (taken) acc += (double)bp[(idx * 3 + c) * hw];
        const double nv = acc * rs;
        noisy[(b * 3 + c) * hw + p] = (float)(nv > 0.0 ? nv : 0.0);
    }
    if (spp_out) spp_out[b * hw + p] = (float)spp;
    if (taken_out) taken_out[b * hw + p] = taken;
}

// partial maxima -> frame max -> partial sums of exp(s - max) -> frame sum
// (fstat[2b] = max, fstat[2b+1] = sum)
template <typename TS>
static void launch_reductions(int B, long long n, const TS* scores, double* pmax, double* psum,
                              double* fstat, cudaStream_t s) {
    // ~8 values per thread, 1..kRedBlocks blocks per frame (small frames: few blocks)
    long long nb = (n + kRedThreads * 8 - 1) / (kRedThreads * 8);
    nb = nb < 1 ? 1 : (nb > kRedBlocks ? kRedBlocks : nb);
    dim3 grid((unsigned)nb, B), sgrid(B, (unsigned)nb);  // (k_frame_stats reads nb from gridDim.y)
    SSB_LAUNCH(s, k_partial_max<TS><<<grid, kRedThreads, 0, s>>>(n, scores, pmax));
    SSB_LAUNCH(s, k_frame_stats<<<dim3(B, 1), kRedThreads, 0, s>>>(pmax, nullptr, fstat, (int)nb));
    SSB_LAUNCH(s, k_partial_sum<TS><<<grid, kRedThreads, 0, s>>>(n, scores, fstat, psum));
    SSB_LAUNCH(s, k_frame_stats<<<dim3(B, 1), kRedThreads, 0, s>>>(pmax, psum, fstat, (int)nb));
    (void)sgrid;
}

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_uniform_grid(uint64_t seed, int64_t frame0, const int64_t* frames, int B, int H, int W,
                     uint64_t stream_id, double* u, ssb_stream_t stream) {
    if (B < 1 || H < 1 || W < 1 || !u) {
        set_error("ssb_uniform_grid: bad dimensions or null output");
        return SSB_EINVAL;
    }
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8, B);
    SSB_LAUNCH((cudaStream_t)stream, k_uniform_grid<<<grid, block, 0, (cudaStream_t)stream>>>(seed, frame0, frames, H, W, stream_id, u));
    return cuda_check("ssb_uniform_grid");
}

int ssb_density_workspace_bytes(int B, int H, int W, size_t* bytes) {
    if (B < 1 || H < 1 || W < 1 || !bytes) {
        set_error("ssb_density_workspace_bytes: bad arguments");
        return SSB_EINVAL;
    }
    *bytes = ((size_t)2 * B * kRedBlocks + 2 * (size_t)B) * sizeof(double);
    return SSB_OK;
}

int ssb_normalize_density(int B, int H, int W, const double* scores, double budget, double* spp,
                          void* workspace, ssb_stream_t stream) {
    if (B < 1 || H < 1 || W < 1 || !scores || !spp || !workspace) {
        set_error("ssb_normalize_density: bad arguments");
        return SSB_EINVAL;
    }
    if (!(budget > 0.0)) {
        set_error("budget must be positive");
        return SSB_EINVAL;
    }
    const long long n = (long long)H * W;
    double* pmax = (double*)workspace;
    double* psum = pmax + (size_t)B * kRedBlocks;
    double* fstat = psum + (size_t)B * kRedBlocks;
    cudaStream_t s = (cudaStream_t)stream;
    launch_reductions<double>(B, n, scores, pmax, psum, fstat, s);
    SSB_LAUNCH(s, k_density_apply<<<dim3(kRedBlocks, B), kRedThreads, 0, s>>>(n, scores, fstat, budget, spp));
    return cuda_check("ssb_normalize_density");
}

int ssb_allocate(const ssb_alloc_desc* d, const double* spp, const int64_t* rank, int64_t* base,
                 double* frac, double* u, uint8_t* taken, ssb_stream_t stream) {
    if (!d || !spp || d->B < 1 || d->H < 1 || d->W < 1) {
        set_error("ssb_allocate: bad arguments");
        return SSB_EINVAL;
    }
    if (d->rule < SSB_RULE_STOCHASTIC || d->rule > SSB_RULE_GUMBEL) {
        set_error("unknown take rule");
        return SSB_EINVAL;
    }
    if (d->dithered && (!rank || d->mask_size < 1)) {
        set_error("dithered allocation requires a mask");
        return SSB_EINVAL;
    }
    dim3 block(32, 8), grid((d->W + 31) / 32, (d->H + 7) / 8, d->B);
    SSB_LAUNCH((cudaStream_t)stream, k_allocate<<<grid, block, 0, (cudaStream_t)stream>>>(*d, spp, rank, base, frac, u, taken));
    return cuda_check("ssb_allocate");
}

static int check_est(const ssb_estimate_desc* d) {
    if (!d || d->B < 1 || d->H < 1 || d->W < 1) {
        set_error("bad estimator descriptor");
        return SSB_EINVAL;
    }
    if (d->variant < SSB_VAR_STOCHASTIC || d->variant > SSB_VAR_GUMBEL) {
        set_error("not a stochastic variant");
        return SSB_EINVAL;
    }
    return SSB_OK;
}

int ssb_stochastic_core(const ssb_estimate_desc* d, const double* spp, const double* frac,
                        const double* u, const double* base_sum, const double* holdout,
                        double* noisy, double* grad, double* contrib, uint8_t* drawn,
                        ssb_stream_t stream) {
    int rc = check_est(d);
    if (rc) return rc;
    if (!spp || !frac || !u || !base_sum || !holdout) {
        set_error("ssb_stochastic_core: null input");
        return SSB_EINVAL;
    }
    const long long n = (long long)d->B * d->H * d->W;
    SSB_LAUNCH((cudaStream_t)stream, k_stochastic_core<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        *d, n, spp, frac, u, base_sum, holdout, noisy, grad, contrib, drawn));
    return cuda_check("ssb_stochastic_core");
}

int ssb_estimate(const ssb_estimate_desc* d, const double* spp, const int64_t* base,
                 const double* frac, const double* u, const double* samples, double* noisy,
                 double* grad, double* contrib, int64_t* used, float* noisy32,
                 ssb_stream_t stream) {
    int rc = check_est(d);
    if (rc) return rc;
    if (!spp || !base || !frac || !u || !samples || d->capacity < 1) {
        set_error("ssb_estimate: null input or empty bank");
        return SSB_EINVAL;
    }
    const long long n = (long long)d->B * d->H * d->W;
    SSB_LAUNCH((cudaStream_t)stream, k_estimate<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        *d, d->H, d->W, spp, base, frac, u, samples, noisy, grad, contrib, used, noisy32));
    return cuda_check("ssb_estimate");
}

int ssb_place_fused(const ssb_place_desc* d, const float* scores, const float* bank, float* noisy,
                    float* spp_out, uint8_t* taken_out, void* workspace, ssb_stream_t stream) {
    if (!d || !scores || !bank || !noisy || !workspace || d->B < 1 || d->H < 1 || d->W < 1 ||
        d->capacity < 1) {
        set_error("ssb_place_fused: bad arguments");
        return SSB_EINVAL;
    }
    if (d->variant != SSB_VAR_STOCHASTIC) {
        set_error("ssb_place_fused: only the stochastic variant is fused");
        return SSB_EUNSUPPORTED;
    }
    if (!(d->budget > 0.0)) {
        set_error("budget must be positive");
        return SSB_EINVAL;
    }
    const long long n = (long long)d->H * d->W;
    double* pmax = (double*)workspace;
    double* psum = pmax + (size_t)d->B * kRedBlocks;
    double* fstat = psum + (size_t)d->B * kRedBlocks;
    cudaStream_t s = (cudaStream_t)stream;
    launch_reductions<float>(d->B, n, scores, pmax, psum, fstat, s);
    dim3 block(32, 8), grid((d->W + 31) / 32, (d->H + 7) / 8, d->B);
    SSB_LAUNCH(s, k_place_fused<<<grid, block, 0, s>>>(*d, scores, fstat, bank, noisy, spp_out, taken_out));
    return cuda_check("ssb_place_fused");
}

}  // extern "C"
