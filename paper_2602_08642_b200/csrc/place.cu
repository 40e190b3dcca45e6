// Sample placement: counter-based uniforms, frame-global density softmax,
// stochastic-rounding allocation, estimator core and the fused inference path.
//
// Reference: pkg/src/sparse_sampler/rng.py:21-63, density.py:43-65,196-233,
// estimators.py:70-149.  All decision arithmetic is IEEE float64 and this TU
// is compiled with -fmad=false so that elementwise results (floor/frac, u,
// u < frac, the estimator formulas) are bit-identical to numpy's.
#include <string>
#include <type_traits>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

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

// one variate (rng.pixel_uniform): a single thread, no grid
__global__ void k_uniform_at(uint64_t seed, int64_t frame, int64_t x, int64_t y, uint64_t stream, double* u) {
    *u = key_uniform(seed, (uint64_t)frame, (uint64_t)x, (uint64_t)y, stream);
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

// ---------------------------------------------------------------- fused placement
// Two launches per call (SURVEY.md 8(a) a1-a6 on the inference/training path):
//  k_place_partials: per block of the frame, the (max, sum exp(v - max)) pair
//    of its scores -- each thread folds its elements (max pass, then sum pass
//    over the same L1-resident values), pairs combine in a fixed shuffle /
//    warp order (deterministic);
//  k_place: every CTA first folds the frame's partial pairs in the same fixed
//    order (identical (m, S) in every CTA, no finish launch), then places 4
//    horizontally adjacent pixels per thread: spp, floor/frac, the counter hash
//    (the per-frame prefix of key_hash hoisted), the exact integer decision,
//    the bank read (S = 2 specialised) and the estimator.
constexpr int kPlThreads = 256;
constexpr int kPlParts = 512;  // max partial pairs per frame

// partial pairs per frame of `units` score groups (float4s, or scalars):
// ~4 groups per thread, but at least 128 pairs where the frame has a group
// per thread for them (small frames: the pass spreads over the SMs)
__host__ __device__ inline int place_nparts(long long units) {
    long long np = (units + kPlThreads * 4 - 1) / (kPlThreads * 4);
    const long long lo = units / kPlThreads < 128 ? units / kPlThreads : 128;
    np = np < lo ? lo : np;
    return (int)(np < 1 ? 1 : (np > kPlParts ? kPlParts : np));
}

// exp(d) for d <= 0 in float64, ~3 ulp (the frame softmax's terms; not the
// compat normalize_density, which keeps libdevice exp): d = (64 n + j) ln2/64
// + r with |r| <= ln2/128 (Cody-Waite split, the high part with 20 trailing
// zero bits so k * hi is exact), e^r by a degree-5 polynomial (truncation
// r^6/720 < 3.5e-17), times 2^(j/64) from a 64-entry table (correctly rounded,
// generated with mpmath) and 2^n on the exponent bits.  d < -700 -> 0: such
// terms are < 1e-304 of the frame maximum's.
__device__ const double kExp2Tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

__device__ __forceinline__ void load_exp_table(double* t2) {
    if (threadIdx.x < 64) t2[threadIdx.x] = kExp2Tab[threadIdx.x];
}

__device__ __forceinline__ double exp_neg(double d, const double* t2) {
    if (!(d >= -700.0)) return 0.0;
    const double kf = rint(d * 0x1.71547652b82fep+6);  // round(d * 64 / ln2)
    const int k = (int)kf;
    const double r = fma(-kf, 0x1.473de6af278edp-40, fma(-kf, 0x1.62e42fef00000p-7, d));
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double v = t2[k & 63] * p;
    return __longlong_as_double(__double_as_longlong(v) + ((long long)(k >> 6) << 52));
}

template <bool VEC>
__global__ void __launch_bounds__(kPlThreads) k_place_partials(long long n, const float* __restrict__ scores,
                                                              double* __restrict__ parts, int nparts, int W,
                                                              uint64_t seed, int64_t frame0, uint64_t* __restrict__ hx) {
    __shared__ double t2[64];
    {
        // the frame's column hashes for k_place (key_hash's first two rounds)
        const int bb = blockIdx.y;
        const uint64_t hf = mix64(mix64(seed + kGold) ^ ((uint64_t)(frame0 + bb) * kGold + kGold));
        for (int x = blockIdx.x * kPlThreads + threadIdx.x; x < W; x += nparts * kPlThreads)
            hx[(long long)bb * W + x] = mix64(hf ^ ((uint64_t)x * kGold + kGold));
    }
    __shared__ double bm;
    load_exp_table(t2);
    const int b = blockIdx.y;
    const float* p = scores + (long long)b * n;
    const long long t0 = (long long)blockIdx.x * kPlThreads + threadIdx.x, step = (long long)nparts * kPlThreads;
    // pass 1: the block's max (a float32 value), broadcast
    float mf = -INFINITY;
    if constexpr (VEC) {
        const float4* p4 = reinterpret_cast<const float4*>(p);
        for (long long g = t0; g < (n >> 2); g += step) {
            const float4 v = __ldg(p4 + g);
            mf = fmaxf(fmaxf(mf, fmaxf(v.x, v.y)), fmaxf(v.z, v.w));
        }
    } else {
        for (long long i = t0; i < n; i += step) mf = fmaxf(mf, p[i]);
    }
    const double mb = block_reduce((double)mf, true);
    if (threadIdx.x == 0) bm = mb;
    __syncthreads();
    const double m = bm;
    // pass 2: sum of exp(v - max) over the same (L1-resident) values, four chains
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (VEC) {
        const float4* p4 = reinterpret_cast<const float4*>(p);
        for (long long g = t0; g < (n >> 2); g += step) {
            const float4 v = __ldg(p4 + g);
            s4[0] += exp_neg((double)v.x - m, t2);
            s4[1] += exp_neg((double)v.y - m, t2);
            s4[2] += exp_neg((double)v.z - m, t2);
            s4[3] += exp_neg((double)v.w - m, t2);
        }
    } else {
        for (long long i = t0; i < n; i += step) s4[0] += exp_neg((double)p[i] - m, t2);
    }
    const double sb = block_reduce((s4[0] + s4[1]) + (s4[2] + s4[3]), false);
    if (threadIdx.x == 0) {
        parts[2 * ((long long)b * kPlParts + blockIdx.x)] = m;
        parts[2 * ((long long)b * kPlParts + blockIdx.x) + 1] = sb;
    }
}

struct PlaceArgs {
    int B, H, W, S, variant, nparts;
    uint64_t seed;
    int64_t frame0;
    double budget, lam, temp, floor_;
    float gainf;  // relaxed fast path: (float)(2 lam / (2 lam - 1))
    const uint64_t* hx;  // (B, W) column hashes mix64(prefix(seed, frame) ^ key(x)), from k_place_partials
    const float* scores;
    const float* bank;
    const double* stat;
    float *noisy, *grad, *spp;
    uint8_t *taken, *drawn;
};

// one pixel: the allocation decision and the estimator outputs (pending:
// the float32 fast path could not decide it and the caller runs it again
// with the float64 path -- compacted across the warp, see k_place)
struct PlacePx {
    float noisy[3], grad[3], spp;
    uint8_t taken, drawn;
    bool pending;
};

template <int VAR, bool S2, bool DEFER = false>
__device__ __forceinline__ PlacePx place_px(const PlaceArgs& a, double m, double ssum, double uni, double adaptive,
                                            uint64_t h1, int y, float score, const float* bp, long long hw,
                                            const double* t2) {
    PlacePx o;
    o.pending = false;
    // key_hash with the (seed, frame) prefix and the column step hoisted
    // (h1 = mix64(prefix ^ key(x)), from the per-frame column table):
    // rng.py:43-48
    uint64_t h = mix64(h1 ^ ((uint64_t)y * kGold + kGold));
    h = mix64(h ^ kGold);  // stream STREAM_ALLOC = 0
    const double k53 = (double)(h >> 11);  // u = k53 * 2^-53 exactly
    const int S = S2 ? 2 : a.S;
    if constexpr (VAR == SSB_VAR_STOCHASTIC || VAR == SSB_VAR_RELAXED || VAR == SSB_VAR_STRAIGHT_THROUGH) {
        // float32 fast path with a rigorous bound on |spp32 - spp64|.  The
        // exponent x = (score - max) log2 e is carried as x_hi + x_lo (TwoSum
        // of the difference, split product with the float log2 e and its
        // residual), e32 = ex2.approx(x_hi) (1 + ln2 x_lo): the relative error
        // is the MUFU's (<= 2^-22) plus a few float32 roundings, < 5e-7, and
        // the constants / product / sum add ~2e-7 spp: err = 1.5e-6 spp + 1e-7
        // (3x margin).  Where the floor or the decision u < frac could come out
        // differently within err (~3e-6 of the pixels), the float64 path below
        // decides instead.  (This TU is built with -fmad=false: TwoSum exact.)
        const float mf = (float)m;  // the max of float32 scores: exact
        // TwoSum(score, -mf): dh + tl == score - mf exactly
        const float dh = score - mf;
        const float bb = dh - score, ab = dh - bb;
        const float tl = (score - ab) + (-mf - bb);
        constexpr float kL2eLo = 1.925963033500011e-08f;  // log2(e) - (float)log2(e)
        const float xh = dh * kLog2e;
        const float xl = fmaf(dh, kLog2e, -xh) + (tl * kLog2e + dh * kL2eLo);
        const float e32 = ex2_ftz(xh) * fmaf(0.6931471805599453f, xl, 1.0f);
        const float spp32 = fmaf((float)adaptive, e32, (float)uni);
        const float fl32 = floorf(spp32), fr32 = spp32 - fl32;
        const float err = fmaf(1.5e-6f, spp32, 1e-7f);
        const float u32 = (float)(h >> 11) * 0x1.0p-53f;  // |u32 - u| <= 6e-8
        // relaxed (estimators.py:101-113): drawn = u >= 1 - frac; the values
        // take the fast path where they depend on spp alone -- not drawn
        // (contrib 0) or the ramp clipped at 1 (contrib = hold * gain); the
        // linear part of the ramp (~frac / lam of the pixels, its value
        // sensitive to frac) and every ambiguous decision go to float64
        bool relaxed_fast = false, rdrawn = false;
        if constexpr (VAR == SSB_VAR_RELAXED) {
            const float lamf = (float)a.lam;
            const float dd = (u32 + fr32) - 1.0f;  // u - (1 - frac)
            const float md = err + 2e-7f;
            rdrawn = dd > 0.0f;
            relaxed_fast = fr32 > err && fr32 < 1.0f - err && fabsf(dd) > md && spp32 < 8388608.0f &&
                           (!rdrawn || fmaf(lamf, dd, -fr32) > (lamf + 1.0f) * md + 1e-6f);
        }
        if constexpr (VAR == SSB_VAR_RELAXED) {
            if (relaxed_fast) {
                o.taken = o.drawn = rdrawn;
                o.spp = a.spp ? (float)(uni + adaptive * exp_neg((double)score - m, t2)) : spp32;  // (optional output)
                const int idx = (int)(fl32 < (float)(S - 1) ? fl32 : (float)(S - 1));
                const float sden = spp32 > (float)a.floor_ ? spp32 : (float)a.floor_;
                const float rs = __frcp_rn(sden);  // == 1.0f / sden (both correctly rounded)
                const float gain = a.gainf;  // 2 lam / (2 lam - 1), rounded once on the host
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float acc = 0.0f;
                    if (S2) {
                        if (idx == 1) acc = bp[(0 * 3 + c) * hw];
                    } else {
                        for (int j = 0; j < idx; ++j) acc += bp[(j * 3 + c) * hw];
                    }
                    if (rdrawn) acc += bp[(idx * 3 + c) * hw] * gain;
                    const float nv = acc * rs;
                    o.noisy[c] = nv > 0.0f ? nv : 0.0f;
                    o.grad[c] = -nv * rs;
                }
                return o;
            }
            if constexpr (DEFER) {
                o.pending = true;
                return o;
            }
        } else if (fr32 > err && fr32 < 1.0f - err && fabsf(u32 - fr32) > err + 1e-7f && spp32 < 8388608.0f) {
            // stochastic; straight-through (estimators.py:114-121): the same
            // take decision, drawn = frac > 0 (here always), and the gradient
            // (hold - noisy) / s
            constexpr bool ST = VAR == SSB_VAR_STRAIGHT_THROUGH;
            const bool tk = u32 < fr32;
            o.taken = tk;
            o.drawn = ST ? 1 : tk;
            o.spp = a.spp ? (float)(uni + adaptive * exp_neg((double)score - m, t2)) : spp32;  // (optional output)
            const int idx = (int)(fl32 < (float)(S - 1) ? fl32 : (float)(S - 1));
            const float sden = spp32 > (float)a.floor_ ? spp32 : (float)a.floor_;
            const float rs = __frcp_rn(sden);  // == 1.0f / sden (both correctly rounded)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float acc = 0.0f;
                if (S2) {
                    if (idx == 1) acc = bp[(0 * 3 + c) * hw];
                } else {
                    for (int j = 0; j < idx; ++j) acc += bp[(j * 3 + c) * hw];
                }
                const float hold = (ST || tk) ? bp[(idx * 3 + c) * hw] : 0.0f;  // (stochastic: read if taken)
                if (tk) acc += hold;
                const float nv = acc * rs;
                o.noisy[c] = nv > 0.0f ? nv : 0.0f;
                o.grad[c] = ST ? (hold - nv) * rs : -nv * rs;
            }
            return o;
        }
    }
    const double e = exp_neg((double)score - m, t2);
    // density.py:63-64, spp = uni + adaptive * (e / sum); `adaptive` arrives
    // pre-divided by the sum (one rounding apart: like the libdevice exp,
    // ~1 ulp from numpy's spp -- the decisions below are exact given spp)
    const double spp = uni + adaptive * e;
    (void)ssum;
    const double fl = floor(spp);
    const double fr = spp - fl;
    const int idx = (int)(fl < (double)(S - 1) ? fl : (double)(S - 1));
    o.spp = (float)spp;
    if constexpr (VAR == SSB_VAR_STOCHASTIC) {
        const bool tk = k53 < fr * 0x1.0p53;  // u < frac (density.py:199)
        o.taken = o.drawn = tk;
        // the estimator value only feeds float32 outputs: float32 from here
        const float sden = (float)(spp > a.floor_ ? spp : a.floor_);
        const float rs = __frcp_rn(sden);  // == 1.0f / sden (both correctly rounded)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float acc = 0.0f;
            if (S2) {
                if (idx == 1) acc = bp[(0 * 3 + c) * hw];
            } else {
                for (int j = 0; j < idx; ++j) acc += bp[(j * 3 + c) * hw];
            }
            if (tk) acc += bp[(idx * 3 + c) * hw];
            const float nv = acc * rs;
            o.noisy[c] = nv > 0.0f ? nv : 0.0f;
            o.grad[c] = -nv * rs;
        }
    } else {
        const double u = k53 * 0x1.0p-53;
        double bs[3] = {0.0, 0.0, 0.0}, ho[3];
        for (int j = 0; j < idx; ++j)
            for (int c = 0; c < 3; ++c) bs[c] += (double)bp[(j * 3 + c) * hw];
        for (int c = 0; c < 3; ++c) ho[c] = (double)bp[(idx * 3 + c) * hw];
        const CoreOut co = core_pixel(VAR, spp, fr, u, bs, ho, a.lam, a.temp, a.floor_);
        constexpr int rule = VAR == SSB_VAR_RELAXED ? SSB_RULE_RELAXED
                                                    : (VAR == SSB_VAR_GUMBEL ? SSB_RULE_GUMBEL : SSB_RULE_STOCHASTIC);
        o.taken = rule == SSB_RULE_GUMBEL ? co.drawn : take_rule(rule, u, fr, a.temp);
        o.drawn = co.drawn;
        for (int c = 0; c < 3; ++c) {
            o.noisy[c] = (float)(co.noisy[c] > 0.0 ? co.noisy[c] : 0.0);
            o.grad[c] = (float)co.grad[c];
        }
    }
    return o;
}

// the frame's (max, sum) from its partial pairs, in a fixed order: the max
// of the partial maxima, then every partial sum rescaled by exp(m_b - max)
// and summed; stat[2b] = max, stat[2b+1] = sum.  (Measured: folding the pairs
// in every CTA of k_place instead costs more than this launch.)
__global__ void __launch_bounds__(kPlThreads) k_place_finish(const double* __restrict__ parts, int nparts,
                                                            double* __restrict__ stat) {
    __shared__ double t2[64];
    __shared__ double bm;
    load_exp_table(t2);
    const int b = blockIdx.x;
    const double* pb = parts + 2 * (long long)b * kPlParts;
    double m = -INFINITY;
    for (int k = threadIdx.x; k < nparts; k += kPlThreads) m = fmax(m, pb[2 * k]);
    const double mm = block_reduce(m, true);
    if (threadIdx.x == 0) bm = mm;
    __syncthreads();
    double s = 0.0;
    for (int k = threadIdx.x; k < nparts; k += kPlThreads) s += pb[2 * k + 1] * exp_neg(pb[2 * k] - bm, t2);
    const double ss = block_reduce(s, false);
    if (threadIdx.x == 0) {
        stat[2 * b] = bm;
        stat[2 * b + 1] = ss;
    }
}

template <bool VEC>
__device__ __forceinline__ void store_px(const PlaceArgs& a, int b, long long hw, long long p0, const PlacePx* px);

template <int VAR, bool S2, bool VEC>
__global__ void __launch_bounds__(kPlThreads, (VAR == SSB_VAR_STOCHASTIC || VAR == SSB_VAR_RELAXED) ? 4 : 1)
    k_place(PlaceArgs a) {
    __shared__ double t2[64];
    load_exp_table(t2);
    __syncthreads();
    const int b = blockIdx.y;
    const double m = a.stat[2 * b], ssum = a.stat[2 * b + 1];
    const long long hw = (long long)a.H * a.W;
    const double uni = 0.125 * a.budget, adaptive = (1.0 - 0.125) * a.budget * (double)hw / ssum;
    const int S = S2 ? 2 : a.S;
    const float* bankb = a.bank + (long long)b * S * 3 * hw;
    constexpr int NPX = VEC ? 4 : 1;
    const long long p0 = ((long long)blockIdx.x * kPlThreads + threadIdx.x) * NPX;
    // relaxed: the float64 fallback (the linear part of the ramp, ~frac / lam
    // of the pixels) would run divergently in almost every warp -- defer it,
    // then run the warp's deferred pixels together after the stores
    constexpr bool DEFER = VAR == SSB_VAR_RELAXED;
    const bool act = p0 < hw;
    if (!DEFER && !act) return;
    PlacePx px[NPX];
#pragma unroll
    for (int j = 0; j < NPX; ++j) px[j].pending = false;
    if (act) {
        const int y = (int)(p0 / a.W), x0 = (int)(p0 - (long long)y * a.W);
        float sc[NPX];
        if constexpr (VEC) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(a.scores + (long long)b * hw + p0));
            sc[0] = v.x;
            sc[1] = v.y;
            sc[2] = v.z;
            sc[3] = v.w;
        } else {
            sc[0] = a.scores[(long long)b * hw + p0];
        }
        // the column hashes of the frame (k_place_partials' table)
        uint64_t h1[NPX];
        const uint64_t* hxr = a.hx + (long long)b * a.W + x0;
        if constexpr (VEC) {
            const ulonglong2 u01 = __ldg(reinterpret_cast<const ulonglong2*>(hxr));
            const ulonglong2 u23 = __ldg(reinterpret_cast<const ulonglong2*>(hxr) + 1);
            h1[0] = u01.x;
            h1[1] = u01.y;
            h1[2] = u23.x;
            h1[3] = u23.y;
        } else {
            h1[0] = __ldg(hxr);
        }
#pragma unroll
        for (int j = 0; j < NPX; ++j)
            px[j] = place_px<VAR, S2, DEFER>(a, m, ssum, uni, adaptive, h1[j], y, sc[j], bankb + p0 + j, hw, t2);
        store_px<VEC>(a, b, hw, p0, px);
    }
    if constexpr (DEFER) {
        // compacted over the whole CTA (the float64 path then runs on ~2 of its
        // 8 warps instead of once in nearly every warp); each deferred pixel is
        // computed on its own, so the slot order does not affect any result
        __shared__ long long s_def[kPlThreads * NPX];
        __shared__ int s_cnt;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NPX; ++j)
            if (px[j].pending) s_def[atomicAdd(&s_cnt, 1)] = p0 + j;
        __syncthreads();
        const int total = s_cnt;
        for (int e = threadIdx.x; e < total; e += kPlThreads) {
            const long long q = s_def[e];
            const int yq = (int)(q / a.W), xq = (int)(q - (long long)yq * a.W);
            PlacePx r[1];
            r[0] = place_px<VAR, S2>(a, m, ssum, uni, adaptive, a.hx[(long long)b * a.W + xq], yq,
                                     a.scores[(long long)b * hw + q], bankb + q,
                                     hw, t2);
            store_px<false>(a, b, hw, q, r);
        }
    }
}

// the outputs of NPX = 4 (VEC) or 1 horizontally adjacent pixels from p0
template <bool VEC>
__device__ __forceinline__ void store_px(const PlaceArgs& a, int b, long long hw, long long p0, const PlacePx* px) {
    float* nz = a.noisy + (long long)b * 3 * hw + p0;
    float* gr = a.grad ? a.grad + (long long)b * 3 * hw + p0 : nullptr;
    if constexpr (VEC) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            __stcs(reinterpret_cast<float4*>(nz + c * hw),
                   make_float4(px[0].noisy[c], px[1].noisy[c], px[2].noisy[c], px[3].noisy[c]));
            if (gr)
                __stcs(reinterpret_cast<float4*>(gr + c * hw),
                       make_float4(px[0].grad[c], px[1].grad[c], px[2].grad[c], px[3].grad[c]));
        }
        if (a.spp)
            __stcs(reinterpret_cast<float4*>(a.spp + (long long)b * hw + p0),
                   make_float4(px[0].spp, px[1].spp, px[2].spp, px[3].spp));
        if (a.taken)
            *reinterpret_cast<uchar4*>(a.taken + (long long)b * hw + p0) =
                make_uchar4(px[0].taken, px[1].taken, px[2].taken, px[3].taken);
        if (a.drawn)
            *reinterpret_cast<uchar4*>(a.drawn + (long long)b * hw + p0) =
                make_uchar4(px[0].drawn, px[1].drawn, px[2].drawn, px[3].drawn);
    } else {
        for (int c = 0; c < 3; ++c) {
            nz[c * hw] = px[0].noisy[c];
            if (gr) gr[c * hw] = px[0].grad[c];
        }
        if (a.spp) a.spp[(long long)b * hw + p0] = px[0].spp;
        if (a.taken) a.taken[(long long)b * hw + p0] = px[0].taken;
        if (a.drawn) a.drawn[(long long)b * hw + p0] = px[0].drawn;
    }
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


// ---------------------------------------------------------------------------
// Small frames (BASELINE c0: one 256^2 frame): the whole inference path --
// placement (the partial pairs, their fold, place), the pooled pyramid and the
// forward levels coarse to fine -- in ONE cooperative kernel with grid-wide
// barriers between the stages, instead of eight dependent launches whose fixed
// cost dominates at this size.  Placement: the same partition into partial
// pairs, the same fold and the same place_px as ssb_place (identical noisy);
// the pyramid: k_pool2's arithmetic per level; the forward per pixel from
// global memory (L2-resident at these sizes) in k_pyr_fwd's form, native
// blend, float32 (pyramid.py:292-345).
constexpr int kInfMaxB = 8;
struct InferArgs {
    PlaceArgs pa;  // stochastic placement, pa.stat unused
    int nparts, L;
    double* parts;  // B x kPlParts x 2
    const float* demod;
    const float* logits[SSB_MAX_LEVELS];
    int hl[SSB_MAX_LEVELS], wl[SSB_MAX_LEVELS], nlog[SSB_MAX_LEVELS];
    float* x0;                      // (B,3,H,W) noisy / max(d, floor)
    float* lv[SSB_MAX_LEVELS];      // pooled levels, l >= 1
    float* lh[SSB_MAX_LEVELS];      // Lhat, l >= 1
    float* out;                     // (B,3,H,W)
};

// the k x k gather + upsample of one level pixel (k_pyr_fwd's arithmetic)
template <int K>
__device__ __forceinline__ void inf_fwd_px(const InferArgs& a, int l, int b, int y, int x) {
    constexpr int R = K / 2, NT = K * K;
    const int H = a.hl[l], W = a.wl[l];
    const bool up = l + 1 < a.L;
    const unsigned hw = (unsigned)H * (unsigned)W;
    const float* lg = a.logits[l] + (size_t)b * a.nlog[l] * hw + (unsigned)y * (unsigned)W + (unsigned)x;
    float e[NT + 4];
    float m = -INFINITY;
#pragma unroll
    for (int t = 0; t < NT + 4; ++t) {
        e[t] = (t < NT || up) ? __ldg(lg + (size_t)t * hw) : -INFINITY;
        m = fmaxf(m, e[t]);
    }
    const float mk = prep_max(m);
    float sum = 0.f;
#pragma unroll
    for (int t = 0; t < NT + 4; ++t) {
        e[t] = (t < NT || up) ? softmax_exp(e[t], mk) : 0.f;
        sum += e[t];
    }
    const float inv = frcp(sum);
    const float* src = l == 0 ? a.x0 + (size_t)b * 3 * hw : a.lv[l] + (size_t)b * 3 * hw;
    int ro[K], co[K];
#pragma unroll
    for (int d = 0; d < K; ++d) {
        ro[d] = clampi(y + d - R, 0, H - 1) * W;
        co[d] = clampi(x + d - R, 0, W - 1);
    }
    int cy0 = 0, cy1 = 0, cx0 = 0, cx1 = 0, Wc = 1;
    const float* lhc = nullptr;
    if (up) {
        const int Hc = a.hl[l + 1];
        Wc = a.wl[l + 1];
        cy0 = min(y >> 1, Hc - 1);
        cy1 = min((y + 1) >> 1, Hc - 1);
        cx0 = min(x >> 1, Wc - 1);
        cx1 = min((x + 1) >> 1, Wc - 1);
        lhc = a.lh[l + 1] + (size_t)b * 3 * Hc * Wc;
    }
    const unsigned o = (unsigned)y * (unsigned)W + (unsigned)x;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float* sc = src + (size_t)c * hw;
        float acc = 0.f;
#pragma unroll
        for (int dy = 0; dy < K; ++dy)
#pragma unroll
            for (int dx = 0; dx < K; ++dx) acc += e[dy * K + dx] * sc[ro[dy] + co[dx]];
        if (up) {
            const float* cp = lhc + (size_t)c * a.hl[l + 1] * Wc;
            acc += e[NT + 0] * cp[cy0 * Wc + cx0];
            acc += e[NT + 1] * cp[cy0 * Wc + cx1];
            acc += e[NT + 2] * cp[cy1 * Wc + cx0];
            acc += e[NT + 3] * cp[cy1 * Wc + cx1];
        }
        acc *= inv;
        if (l == 0) {
            acc *= demod_clamp(a.demod[((size_t)b * 3 + c) * hw + o]);
            a.out[((size_t)b * 3 + c) * hw + o] = acc;
        } else {
            a.lh[l][((size_t)b * 3 + c) * hw + o] = acc;
        }
    }
}

// one level-l pixel (Y, X) = k_pool2 of its 2x2 children at level l - 1
__device__ __forceinline__ void inf_pool_px(const InferArgs& a, int l, int b, int Y, int X) {
    const int H = a.hl[l - 1], W = a.wl[l - 1], Wc = a.wl[l];
    const float* in = (l == 1 ? a.x0 : a.lv[l - 1]) + (size_t)b * 3 * H * W;
    const int yb = 2 * Y, xb = 2 * X;
    const bool hy = yb + 1 < H, hx = xb + 1 < W;
    const float rcnt = (hy && hx) ? 0.25f : ((hy || hx) ? 0.5f : 1.f);
    const long long o00 = (long long)yb * W + xb;
    const long long o01 = hx ? o00 + 1 : o00, o10 = hy ? o00 + W : o00, o11 = hy ? o01 + W : o01;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float* p = in + (size_t)c * H * W;
        const float s01 = hx ? p[o01] : 0.f, s10 = hy ? p[o10] : 0.f, s11 = (hx && hy) ? p[o11] : 0.f;
        a.lv[l][((size_t)b * 3 + c) * a.hl[l] * Wc + (long long)Y * Wc + X] = ((p[o00] + s01) + (s10 + s11)) * rcnt;
    }
}

#ifdef SSB_INF_TIMING
static __device__ unsigned long long g_inf_t[16];
#define SSB_INF_T(k) \
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_inf_t[k]));
#else
#define SSB_INF_T(k)
#endif
template <int K>
__global__ void __launch_bounds__(kPlThreads, 2) k_infer_small(InferArgs a) {
    cg::grid_group grid = cg::this_grid();
    SSB_INF_T(0)
    __shared__ double t2[64];
    __shared__ double s_ms[kInfMaxB][2];
    __shared__ double bm;
    load_exp_table(t2);
    __syncthreads();
    const PlaceArgs& pa = a.pa;
    const int B = pa.B;
    const long long hw = (long long)pa.H * pa.W;
    const long long gtid = (long long)blockIdx.x * kPlThreads + threadIdx.x, gthreads = (long long)gridDim.x * kPlThreads;
    // 1. partial pairs: virtual block j of frame b = k_place_partials<VEC> block j
    for (int vb = blockIdx.x; vb < B * a.nparts; vb += gridDim.x) {
        const int b = vb / a.nparts, j = vb - b * a.nparts;
        const float4* p4 = reinterpret_cast<const float4*>(pa.scores + (long long)b * hw);
        const long long t0 = (long long)j * kPlThreads + threadIdx.x, step = (long long)a.nparts * kPlThreads;
        float mf = -INFINITY;
        for (long long g = t0; g < (hw >> 2); g += step) {
            const float4 v = __ldg(p4 + g);
            mf = fmaxf(fmaxf(mf, fmaxf(v.x, v.y)), fmaxf(v.z, v.w));
        }
        const double mb = block_reduce((double)mf, true);
        if (threadIdx.x == 0) bm = mb;
        __syncthreads();
        const double m = bm;
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        for (long long g = t0; g < (hw >> 2); g += step) {
            const float4 v = __ldg(p4 + g);
            s4[0] += exp_neg((double)v.x - m, t2);
            s4[1] += exp_neg((double)v.y - m, t2);
            s4[2] += exp_neg((double)v.z - m, t2);
            s4[3] += exp_neg((double)v.w - m, t2);
        }
        const double sb = block_reduce((s4[0] + s4[1]) + (s4[2] + s4[3]), false);
        if (threadIdx.x == 0) {
            a.parts[2 * ((long long)b * kPlParts + j)] = m;
            a.parts[2 * ((long long)b * kPlParts + j) + 1] = sb;
        }
    }
    grid.sync();
    SSB_INF_T(1)
    // 2. every CTA folds each frame's pairs (k_place_finish's order), then places
    for (int b = 0; b < B; ++b) {
        const double* pb = a.parts + 2 * (long long)b * kPlParts;
        double m = -INFINITY;
        for (int k = threadIdx.x; k < a.nparts; k += kPlThreads) m = fmax(m, pb[2 * k]);
        const double mm = block_reduce(m, true);
        if (threadIdx.x == 0) bm = mm;
        __syncthreads();
        double sl = 0.0;
        for (int k = threadIdx.x; k < a.nparts; k += kPlThreads) sl += pb[2 * k + 1] * exp_neg(pb[2 * k] - bm, t2);
        const double ss = block_reduce(sl, false);
        if (threadIdx.x == 0) {
            s_ms[b][0] = bm;
            s_ms[b][1] = ss;
        }
        __syncthreads();
    }
    const double uni = 0.125 * pa.budget;
    for (long long it = gtid; it < B * (hw >> 2); it += gthreads) {
        const int b = (int)(it / (hw >> 2));
        const long long p0 = (it - (long long)b * (hw >> 2)) * 4;
        const double m = s_ms[b][0], ssum = s_ms[b][1];
        const double adaptive = (1.0 - 0.125) * pa.budget * (double)hw / ssum;
        const uint64_t hf = mix64(mix64(pa.seed + kGold) ^ ((uint64_t)(pa.frame0 + b) * kGold + kGold));
        const float* bankb = pa.bank + (long long)b * 2 * 3 * hw;
        const int y = (int)(p0 / pa.W), x0 = (int)(p0 - (long long)y * pa.W);
        const float4 v = __ldg(reinterpret_cast<const float4*>(pa.scores + (long long)b * hw + p0));
        const float sc[4] = {v.x, v.y, v.z, v.w};
        PlacePx px[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            px[j] = place_px<SSB_VAR_STOCHASTIC, true>(pa, m, ssum, uni, adaptive,
                                                       mix64(hf ^ ((uint64_t)(x0 + j) * kGold + kGold)), y, sc[j],
                                                       bankb + p0 + j,
                                                       hw, t2);
        store_px<true>(pa, b, hw, p0, px);
        // the demodulated input of the pyramid (k_pool2's / the forward's x0)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float4 d = __ldg(reinterpret_cast<const float4*>(a.demod + ((long long)b * 3 + c) * hw + p0));
            *reinterpret_cast<float4*>(a.x0 + ((long long)b * 3 + c) * hw + p0) =
                make_float4(fdiv(px[0].noisy[c], demod_clamp(d.x)), fdiv(px[1].noisy[c], demod_clamp(d.y)),
                            fdiv(px[2].noisy[c], demod_clamp(d.z)), fdiv(px[3].noisy[c], demod_clamp(d.w)));
        }
    }
    grid.sync();
    SSB_INF_T(2)
    // 3. the pooled pyramid, one level per barrier (measured: a thread per
    // level-2 pixel pooling its four level-1 children first is slower -- its
    // dependent loads serialise)
    for (int l = 1; l < a.L; ++l) {
        const long long n = (long long)a.hl[l] * a.wl[l];
        for (long long it = gtid; it < B * n; it += gthreads) {
            const int b = (int)(it / n);
            const int q = (int)(it - (long long)b * n);
            inf_pool_px(a, l, b, q / a.wl[l], q % a.wl[l]);
        }
        grid.sync();
        SSB_INF_T(3)
    }
    // 4. the forward, coarse to fine
    for (int l = a.L - 1; l >= 0; --l) {
        const long long n = (long long)a.hl[l] * a.wl[l];
        for (long long it = gtid; it < B * n; it += gthreads) {
            const int b = (int)(it / n);
            const int q = (int)(it - (long long)b * n);
            inf_fwd_px<K>(a, l, b, q / a.wl[l], q % a.wl[l]);
        }
        if (l > 0) grid.sync();
        if (l > 0) {
            SSB_INF_T(4 + (a.L - 1 - l))
        }
    }
    SSB_INF_T(12)
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

int ssb_uniform_at(uint64_t seed, int64_t frame, int64_t x, int64_t y, uint64_t stream_id, double* u,
                   ssb_stream_t stream) {
    if (!u || x < 0 || y < 0) {
        set_error("ssb_uniform_at: null output or negative coordinate");
        return SSB_EINVAL;
    }
    SSB_LAUNCH((cudaStream_t)stream, k_uniform_at<<<1, 1, 0, (cudaStream_t)stream>>>(seed, frame, x, y, stream_id, u));
    return cuda_check("ssb_uniform_at");
}

int ssb_density_workspace_bytes(int B, int H, int W, size_t* bytes) {
    if (B < 1 || H < 1 || W < 1 || !bytes) {
        set_error("ssb_density_workspace_bytes: bad arguments");
        return SSB_EINVAL;
    }
    // (the fused placement uses 2 x kPlParts + 2 doubles per frame of it and
    // then B x W column hashes)
    *bytes = ((size_t)2 * B * (kRedBlocks > kPlParts ? kRedBlocks : kPlParts) + 2 * (size_t)B) * sizeof(double) +
             (size_t)B * W * sizeof(uint64_t);
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

int ssb_place(const ssb_place_desc* d, const ssb_place_cfg* cfg, const ssb_place_io* io, void* workspace,
              ssb_stream_t stream) {
    if (!d || !io || !io->scores || !io->bank || !io->noisy || !workspace || d->B < 1 || d->H < 1 || d->W < 1 ||
        d->capacity < 1) {
        set_error("ssb_place: bad arguments");
        return SSB_EINVAL;
    }
    if (d->variant < SSB_VAR_STOCHASTIC || d->variant > SSB_VAR_GUMBEL) {
        set_error("ssb_place: not a stochastic variant");
        return SSB_EINVAL;
    }
    if (d->variant != SSB_VAR_STOCHASTIC && !cfg) {
        set_error("ssb_place: the estimator config is required for this variant");
        return SSB_EINVAL;
    }
    if (!(d->budget > 0.0)) {
        set_error("budget must be positive");
        return SSB_EINVAL;
    }
    const long long n = (long long)d->H * d->W;
    if (n >= (1ll << 31)) {
        set_error("ssb_place: H*W must be < 2^31");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const bool vec = (d->W % 4) == 0;
    // partial pairs: ~4 float4 groups (16 scores) per thread, at most kPlParts
    // per frame (measured: 1 group per thread and 2048 pairs is no faster)
    const long long units = vec ? n / 4 : n;
    const long long np = place_nparts(units);
    double* parts = (double*)workspace;  // B x kPlParts x 2 doubles + B x 2 (inside the density workspace)
    dim3 pgrid((unsigned)np, d->B);
    double* stat = parts + (size_t)2 * d->B * kPlParts;
    uint64_t* hx = reinterpret_cast<uint64_t*>(stat + 2 * d->B);  // (B, W) column hashes
    if (vec)
        SSB_LAUNCH(s, k_place_partials<true><<<pgrid, kPlThreads, 0, s>>>(n, io->scores, parts, (int)np, d->W, d->seed,
                                                                          d->frame0, hx));
    else
        SSB_LAUNCH(s, k_place_partials<false><<<pgrid, kPlThreads, 0, s>>>(n, io->scores, parts, (int)np, d->W, d->seed,
                                                                           d->frame0, hx));
    SSB_LAUNCH(s, k_place_finish<<<d->B, kPlThreads, 0, s>>>(parts, (int)np, stat));

    PlaceArgs a{};
    a.B = d->B;
    a.H = d->H;
    a.W = d->W;
    a.S = d->capacity;
    a.variant = d->variant;
    a.nparts = (int)np;
    a.seed = d->seed;
    a.frame0 = d->frame0;
    a.budget = d->budget;
    a.lam = cfg ? cfg->lam : 10.0;
    a.gainf = (float)(2.0f * (float)a.lam / (2.0f * (float)a.lam - 1.0f));
    a.temp = cfg ? cfg->gumbel_temp : 1.0;
    a.floor_ = cfg ? cfg->density_floor : 1e-8;
    a.scores = io->scores;
    a.bank = io->bank;
    a.stat = stat;
    a.hx = hx;
    a.noisy = io->noisy;
    a.grad = io->grad;
    a.spp = io->spp;
    a.taken = io->taken;
    a.drawn = io->drawn;
    const long long per = vec ? 4 * kPlThreads : kPlThreads;
    dim3 grid((unsigned)((n + per - 1) / per), d->B);
    const bool s2 = d->capacity == 2;
    auto go = [&](auto var_t) {
        constexpr int V = decltype(var_t)::value;
        if (s2 && vec) SSB_LAUNCH(s, k_place<V, true, true><<<grid, kPlThreads, 0, s>>>(a));
        else if (s2) SSB_LAUNCH(s, k_place<V, true, false><<<grid, kPlThreads, 0, s>>>(a));
        else if (vec) SSB_LAUNCH(s, k_place<V, false, true><<<grid, kPlThreads, 0, s>>>(a));
        else SSB_LAUNCH(s, k_place<V, false, false><<<grid, kPlThreads, 0, s>>>(a));
    };
    switch (d->variant) {
        case SSB_VAR_STOCHASTIC: go(std::integral_constant<int, SSB_VAR_STOCHASTIC>{}); break;
        case SSB_VAR_RELAXED: go(std::integral_constant<int, SSB_VAR_RELAXED>{}); break;
        case SSB_VAR_STRAIGHT_THROUGH: go(std::integral_constant<int, SSB_VAR_STRAIGHT_THROUGH>{}); break;
        default: go(std::integral_constant<int, SSB_VAR_GUMBEL>{}); break;
    }
    return cuda_check("ssb_place");
}

int ssb_place_fused(const ssb_place_desc* d, const float* scores, const float* bank, float* noisy,
                    float* spp_out, uint8_t* taken_out, void* workspace, ssb_stream_t stream) {
    if (d && d->variant != SSB_VAR_STOCHASTIC) {
        set_error("ssb_place_fused: only the stochastic variant (use ssb_place for the others)");
        return SSB_EUNSUPPORTED;
    }
    ssb_place_io io{scores, bank, noisy, nullptr, spp_out, taken_out, nullptr};
    return ssb_place(d, nullptr, &io, workspace, stream);
}


static size_t inf_al(size_t n) { return (n + 255) & ~(size_t)255; }

#ifdef SSB_INF_TIMING
int ssb_debug_inf_times(unsigned long long* out16) {
    return cudaMemcpyFromSymbol(out16, g_inf_t, 16 * sizeof(unsigned long long)) == cudaSuccess ? 0 : -2;
}
#endif

int ssb_infer_small_workspace_bytes(int B, int H, int W, int levels, size_t* bytes) {
    if (!bytes || B < 1 || H < 1 || W < 1 || levels < 1 || levels > SSB_MAX_LEVELS) {
        set_error("ssb_infer_small_workspace_bytes: bad arguments");
        return SSB_EINVAL;
    }
    size_t t = inf_al((size_t)B * kPlParts * 2 * sizeof(double)) + inf_al((size_t)B * 3 * H * W * sizeof(float));
    int h = H, w = W;
    for (int l = 1; l < levels; ++l) {
        h = (h + 1) / 2;
        w = (w + 1) / 2;
        t += 2 * inf_al((size_t)B * 3 * h * w * sizeof(float));
    }
    *bytes = t;
    return SSB_OK;
}

int ssb_infer_small(const ssb_place_desc* pd, const float* scores, const float* bank, const float* demod,
                    int levels, int ksize, const float* const* logits, float* noisy, float* out, void* workspace,
                    ssb_stream_t stream) {
    if (!pd || !scores || !bank || !demod || !logits || !noisy || !out || !workspace || levels < 1 ||
        levels > SSB_MAX_LEVELS || pd->B < 1 || pd->H < 1 || pd->W < 1 || !(pd->budget > 0.0)) {
        set_error("ssb_infer_small: bad arguments");
        return SSB_EINVAL;
    }
    for (int l = 0; l < levels; ++l)
        if (!logits[l]) {
            set_error("ssb_infer_small: missing logits");
            return SSB_EINVAL;
        }
    const long long n = (long long)pd->H * pd->W;
    if (pd->variant != SSB_VAR_STOCHASTIC || pd->capacity != 2 || pd->W % 4 != 0 || pd->B > kInfMaxB ||
        (ksize != 3 && ksize != 5 && ksize != 7) || n * pd->B > (1ll << 20)) {
        set_error("ssb_infer_small: unsupported (stochastic, capacity 2, W % 4 == 0, <= 2^20 pixels, k 3/5/7)");
        return SSB_EUNSUPPORTED;
    }
    InferArgs a{};
    a.pa.B = pd->B;
    a.pa.H = pd->H;
    a.pa.W = pd->W;
    a.pa.S = 2;
    a.pa.variant = SSB_VAR_STOCHASTIC;
    a.pa.seed = pd->seed;
    a.pa.frame0 = pd->frame0;
    a.pa.budget = pd->budget;
    a.pa.lam = 10.0;
    a.pa.temp = 1.0;
    a.pa.floor_ = 1e-8;
    a.pa.scores = scores;
    a.pa.bank = bank;
    a.pa.noisy = noisy;
    const long long units = n / 4;
    a.nparts = place_nparts(units);
    a.L = levels;
    a.demod = demod;
    char* w = (char*)workspace;
    a.parts = (double*)w;
    w += inf_al((size_t)pd->B * kPlParts * 2 * sizeof(double));
    a.x0 = (float*)w;
    w += inf_al((size_t)pd->B * 3 * n * sizeof(float));
    a.hl[0] = pd->H;
    a.wl[0] = pd->W;
    for (int l = 0; l < levels; ++l) {
        if (l > 0) {
            a.hl[l] = (a.hl[l - 1] + 1) / 2;
            a.wl[l] = (a.wl[l - 1] + 1) / 2;
            const size_t sz = inf_al((size_t)pd->B * 3 * a.hl[l] * a.wl[l] * sizeof(float));
            a.lv[l] = (float*)w;
            w += sz;
            a.lh[l] = (float*)w;
            w += sz;
        }
        a.logits[l] = logits[l];
        a.nlog[l] = ksize * ksize + (l + 1 < levels ? 4 : 0);
    }
    a.out = out;
    cudaStream_t s = (cudaStream_t)stream;
    const void* kern = ksize == 3 ? (const void*)k_infer_small<3>
                                  : (ksize == 5 ? (const void*)k_infer_small<5> : (const void*)k_infer_small<7>);
    int dev = 0, nsm = 0;  // (per call: the current device's SM count)
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPlThreads, 0);
    if (per_sm < 1) {
        set_error("ssb_infer_small: no co-resident CTA");
        return SSB_ECUDA;
    }
    // one thread per level-0 pixel for the forward stage, at most what is
    // co-resident
    const long long want = (pd->B * n + kPlThreads - 1) / kPlThreads;
    const long long cap = (long long)nsm * per_sm;
    const unsigned grid = (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
    void* args[] = {&a};
    SSB_LAUNCH(s, cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kPlThreads), args, 0, s));
    return cuda_check("ssb_infer_small");
}
}  // extern "C"
