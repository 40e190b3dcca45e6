// Backward ordering without the coarse->fine sweep kernel (float32, C = 3,
// no temporal group): the level-0 backward runs LAST and writes the final
// g_noisy / g_demod directly.  Reference: reconstruct_backward sweeps
// (pyramid.py:383-421) -- level 0's upsample-transpose feeds the coarser
// levels (sweep 1), the pooled-input gradient of the coarser levels reaches
// level 0 through pool^T (sweep 2).  Reordered:
//   1. k_up_transpose: ghat^1 = U^T(w_up * gout) at level 0 from the 4
//      upsample logits and the forward's log-sum-exp (w = 2^(z log2e - lse)),
//      gout = upstream * max(d, 1e-3) -- no full softmax needed;
//   2. the level 1..L-1 backward kernels (unchanged);
//   3. k_pool_chain: T1 = gL1 + P^T(gL2 + P^T(...)) at level 1, in place;
//   4. the level-0 backward with the chain term T1(parent)/count added in
//      its flush (and no upsample transpose).
#pragma once

#include "pyr_kernels.cuh"

namespace ssb {

constexpr int UPT_X = 32, UPT_Y = 8;  // coarse pixels per CTA

struct UpTransposeArgs {
    int H, W, Hc, Wc, nlog;
    const void* logits;   // level-0 logits (B, nlog, H, W); upsample channels at NT..
    long long lg_b;
    const float* lse;     // (B, H, W) base-2 log-sum-exp from the forward
    const float* up;      // upstream (B, 3, H, W)
    const float* demod;   // (B, 3, H, W)
    float* ghat;          // ghat^1 (B, 3, Hc, Wc)
};

// two horizontally adjacent values of a plane (x even, W even: 8-B / 4-B aligned)
// (default caching: the neighbouring coarse pixels' threads re-read edge
// rows / columns -- an evict-first load would send those back to DRAM)
__device__ __forceinline__ float2 ld_pair_lg(const float* p) { return __ldg(reinterpret_cast<const float2*>(p)); }
__device__ __forceinline__ float2 ld_pair_lg(const __nv_bfloat16* p) {
    const unsigned w = __ldg(reinterpret_cast<const unsigned*>(p));
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// One thread per coarse pixel (Y, X), no shared memory: tap (i, j) of fine
// pixel (y, x) lands on (min((y+i)/2, Hc-1), min((x+j)/2, Wc-1))
// (pyramid.py:216-241), so (Y, X) gathers its own 2x2 block (rows 2Y, 2Y+1
// with tap i = 0; row 2Y with i = 1; row 2Y+1 with i = 1 only on the last
// coarse row), row 2Y-1 with i = 1, and likewise for columns.  Every
// (pixel, tap) exponential is evaluated by exactly one thread.
template <int NT, bool TIED, typename TL>
__global__ void __launch_bounds__(256) k_up_transpose(const UpTransposeArgs a) {
    const int X = blockIdx.x * blockDim.x + threadIdx.x;
    const int Y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (X >= a.Wc || Y >= a.Hc) return;
    const unsigned hw = (unsigned)a.H * (unsigned)a.W;
    const TL* lg = (const TL*)a.logits + (size_t)b * a.lg_b;
    const float* lse = a.lse + (size_t)b * hw;
    const float* up = a.up + (size_t)b * 3 * hw;
    const float* dm = a.demod + (size_t)b * 3 * hw;
    const bool lastY = Y == a.Hc - 1, lastX = X == a.Wc - 1;
    const int x0 = 2 * X;  // even; x0 + 1 < W since W is even on this path
    float acc[3] = {0.f, 0.f, 0.f};
    auto gout = [&](unsigned p, int c) { return up[c * hw + p] * demod_clamp(dm[c * hw + p]); };
    auto wt = [&](float z, float l2) { return ex2_ftz(fmaf(z, kLog2e, -l2)); };
    // own rows y = 2Y (taps i = 0, 1) and y = 2Y + 1 (i = 0; i = 1 on the last row)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int y = 2 * Y + r;
        if (y >= a.H) break;
        const bool i1 = r == 0 || lastY;
        const unsigned p = (unsigned)y * (unsigned)a.W + (unsigned)x0;
        const float2 l2 = __ldg(reinterpret_cast<const float2*>(lse + p));
        float2 z[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) z[t] = ld_pair_lg(lg + (size_t)(TIED ? NT : NT + t) * hw + p);
        // pixel x0: taps j = 0, 1 both land on X; pixel x0 + 1: j = 0 (and j = 1 on the last column)
        float ws0 = wt(z[0].x, l2.x) + wt(z[1].x, l2.x);
        float ws1 = wt(z[0].y, l2.y) + (lastX ? wt(z[1].y, l2.y) : 0.f);
        if (i1) {
            ws0 += wt(z[2].x, l2.x) + wt(z[3].x, l2.x);
            ws1 += wt(z[2].y, l2.y) + (lastX ? wt(z[3].y, l2.y) : 0.f);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float2 u = __ldg(reinterpret_cast<const float2*>(up + c * hw + p));
            const float2 d = __ldg(reinterpret_cast<const float2*>(dm + c * hw + p));
            acc[c] = fmaf(ws0, u.x * demod_clamp(d.x), acc[c]);
            acc[c] = fmaf(ws1, u.y * demod_clamp(d.y), acc[c]);
        }
        // left neighbour column x0 - 1: tap j = 1 lands on X
        if (x0 > 0) {
            const unsigned q = p - 1;
            const float lq = lse[q];
            float w = wt(ld_logit<float>(lg + (size_t)(TIED ? NT : NT + 1) * hw + q), lq);
            if (i1) w += wt(ld_logit<float>(lg + (size_t)(TIED ? NT : NT + 3) * hw + q), lq);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = fmaf(w, gout(q, c), acc[c]);
        }
    }
    // upper neighbour row y = 2Y - 1: tap i = 1 lands on Y
    if (Y > 0) {
        const int y = 2 * Y - 1;
        const unsigned p = (unsigned)y * (unsigned)a.W + (unsigned)x0;
        const float2 l2 = *reinterpret_cast<const float2*>(lse + p);
        const float2 z2 = ld_pair_lg(lg + (size_t)(TIED ? NT : NT + 2) * hw + p);
        const float2 z3 = ld_pair_lg(lg + (size_t)(TIED ? NT : NT + 3) * hw + p);
        const float ws0 = wt(z2.x, l2.x) + wt(z3.x, l2.x);
        const float ws1 = wt(z2.y, l2.y) + (lastX ? wt(z3.y, l2.y) : 0.f);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            acc[c] = fmaf(ws0, gout(p, c), acc[c]);
            acc[c] = fmaf(ws1, gout(p + 1, c), acc[c]);
        }
        if (x0 > 0) {  // corner (2Y - 1, 2X - 1): tap (1, 1)
            const unsigned q = p - 1;
            const float w = wt(ld_logit<float>(lg + (size_t)(TIED ? NT : NT + 3) * hw + q), lse[q]);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = fmaf(w, gout(q, c), acc[c]);
        }
    }
    const size_t hwc = (size_t)a.Hc * a.Wc, o = (size_t)Y * a.Wc + X;
#pragma unroll
    for (int c = 0; c < 3; ++c) a.ghat[((size_t)b * 3 + c) * hwc + o] = acc[c];
}

struct ChainArgs {
    int levels;
    int dims_h[SSB_MAX_LEVELS], dims_w[SSB_MAX_LEVELS];
    float* gl[SSB_MAX_LEVELS];  // gL_l for l >= 1 (B, 3, H_l, W_l); gl[1] becomes T1 in place
};

// T1(P) = gL1(P) + sum over ancestors A at level l >= 2 of gL_l(A) / (children
// counts along the chain) -- the coarse part of sweep 2 at level 1
static __global__ void k_pool_chain(const ChainArgs a) {
    // four level-1 pixels per thread along x: one float4 of gL1 per channel,
    // the coarser ancestors of the quad loaded once (their per-pixel children
    // counts differ only at the image edge)
    const int x4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    const int W1 = a.dims_w[1], H1 = a.dims_h[1];
    if (x4 >= W1 || y >= H1) return;
    const int top = a.levels - 1;
    const size_t hw1 = (size_t)H1 * W1;
    const bool vec = (W1 & 3) == 0;  // whole quad inside the row, 16-B aligned
    float pb[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) pb[k][c] = 0.f;
    if (top >= 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int x = min(x4 + k, W1 - 1);
            const size_t hwt = (size_t)a.dims_h[top] * a.dims_w[top];
            const size_t ot = (size_t)(y >> (top - 1)) * a.dims_w[top] + (x >> (top - 1));
#pragma unroll
            for (int c = 0; c < 3; ++c) pb[k][c] = __ldg(&a.gl[top][((size_t)b * 3 + c) * hwt + ot]);
        }
        for (int l = top - 1; l >= 1; --l) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int x = min(x4 + k, W1 - 1);
                const int Yp = y >> l, Xp = x >> l;  // the level-(l+1) ancestor, its children at level l
                const bool hy = 2 * Yp + 1 < a.dims_h[l], hx = 2 * Xp + 1 < a.dims_w[l];
                const float rcnt = (hy && hx) ? 0.25f : ((hy || hx) ? 0.5f : 1.f);
#pragma unroll
                for (int c = 0; c < 3; ++c) pb[k][c] *= rcnt;
                if (l == 1) continue;
                const size_t hwl = (size_t)a.dims_h[l] * a.dims_w[l];
                const size_t ol = (size_t)(y >> (l - 1)) * a.dims_w[l] + (x >> (l - 1));
#pragma unroll
                for (int c = 0; c < 3; ++c) pb[k][c] += __ldg(&a.gl[l][((size_t)b * 3 + c) * hwl + ol]);
            }
        }
    }
    const size_t o1 = (size_t)y * W1 + x4;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float* p = &a.gl[1][((size_t)b * 3 + c) * hw1 + o1];
        if (vec) {
            float4 v = *reinterpret_cast<const float4*>(p);
            v.x += pb[0][c];
            v.y += pb[1][c];
            v.z += pb[2][c];
            v.w += pb[3][c];
            *reinterpret_cast<float4*>(p) = v;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (x4 + k < W1) p[k] = p[k] + pb[k][c];
        }
    }
}

}  // namespace ssb
