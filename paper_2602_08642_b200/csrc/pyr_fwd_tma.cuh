// Level forward, TMA-pipelined row walker (fp32 images, fp32 or bf16 logits;
// the temporal group on the one-pixel-per-thread path; other configurations
// use k_pyr_fwd).
//
// CTA = column strip of TXF = 64 own columns x one segment of rows, walked in
// steps of S = 4 rows (256 threads, one own pixel each).  Per step one thread
// issues, one step ahead, TMA boxes for: the step's logits (TXF x S x C_l),
// the image rows R ahead of it (x0 = noisy / max(d, 1e-3) at level 0, or the
// pooled level, landing in a block ring that also keeps the R rows above) and
// the coarse Lhat rows of the upsample taps.  Then: softmax from smem into
// registers, in-place demodulation of the new image rows, one barrier, k x k
// gather + 4 upsample taps, remodulation, store.  One __syncthreads per step.
#pragma once

#include "pyr_kernels.cuh"
#include "tma.cuh"

namespace ssb {

struct FwdTmaMaps {
    CUtensorMap lg;   // logits (W, H, NLOG, B), box (TXF, S, NLOG)
    CUtensorMap lin;  // noisy (level 0) or L^l, box (RX, S, 3)
    CUtensorMap dem;  // demod (level 0), box (RX, S, 3)
    CUtensorMap lhc;  // coarse Lhat^{l+1}, box (CB, S/2 + 1, 3)
    CUtensorMap prv;  // PREV: the warped history, box (RX, S, 3)
};

// PREV (level 0 with history): the temporal group's K*K logits follow the
// upsample logits; the history rides in the image ring as a third plane
// group, divided by max(d, floor) like the noisy image (pyramid.py:302-309,332-334)
template <int K, typename TL, bool L0, bool UP, bool TIED, bool PREV = false>
struct FwdTmaShape {
    static constexpr int R = K / 2, NT = K * K, NUP = UP ? 4 : 0, NW0 = NT + NUP, NW = NW0 + (PREV ? NT : 0);
    static constexpr int NLOG0 = NT + (UP ? (TIED ? 1 : 4) : 0), NLOG = NLOG0 + (PREV ? NT : 0);
    static constexpr int S = 4, TXF = 64, RA = 4, RX = TXF + 2 * RA;
    static constexpr int NPRO = (2 * R + S - 1) / S, NBL = NPRO + 2;
    static constexpr int NI = L0 ? (PREV ? 3 : 2) : 1;  // image planes per block: x0 [, demod [, history]]
    static_assert(!PREV || L0, "the temporal group is level 0's");
    static constexpr int CB = 36, CROWS = S / 2 + 1;
    static constexpr int al32(int n) { return (n + 31) & ~31; }
    static constexpr int LGE = (int)sizeof(TL);          // logit element size (4 or 2)
    static constexpr int LGF = al32((NLOG * S * TXF * LGE + 3) / 4);  // floats per logits buffer
    static constexpr int DEMOFF = al32(3 * S * RX);
    static constexpr int BLKF = NI * DEMOFF;
    static constexpr int LHF = UP ? al32(3 * CROWS * CB) : 0;
    static constexpr uint32_t TX_IMG = 3 * S * RX * 4;
    static constexpr uint32_t TX_STEP = NLOG * S * TXF * LGE + NI * TX_IMG + (UP ? 3 * CROWS * CB * 4 : 0);
    static constexpr uint32_t TX_PRO = NPRO * NI * TX_IMG;
    static constexpr size_t FLOATS = (size_t)LGF + NBL * BLKF + 2 * LHF;
    static constexpr size_t SMEM = FLOATS * 4 + 32;
    static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB = MINB_SMEM > 4 ? 4 : (MINB_SMEM < 1 ? 1 : MINB_SMEM);
    // PAIR (bf16 logits, k = 7: instruction bound): 128 threads, each two
    // horizontally adjacent pixels -- 32-bit logit loads carry both pixels,
    // FFMA2 / FADD2 over the pair, one 8-B shared load per two window values
    static constexpr bool PAIR = LGE == 2 && K == 7 && !PREV;
    static constexpr int NTH = PAIR ? 128 : 256;
};

template <int K, typename TL, bool L0, bool UP, bool TIED, bool PREV = false>
__global__ void __launch_bounds__((FwdTmaShape<K, TL, L0, UP, TIED, PREV>::NTH),
                                  (FwdTmaShape<K, TL, L0, UP, TIED, PREV>::MINB))
    k_pyr_fwd_tma(const FwdLevel a, const __grid_constant__ FwdTmaMaps mp) {
    using SH = FwdTmaShape<K, TL, L0, UP, TIED, PREV>;
    constexpr int R = SH::R, NT = SH::NT, NW = SH::NW, NLOG = SH::NLOG, S = SH::S;
    constexpr int TXF = SH::TXF, RA = SH::RA, RX = SH::RX, NPRO = SH::NPRO, NBL = SH::NBL;
    constexpr int NI = SH::NI, CB = SH::CB, CROWS = SH::CROWS, LGF = SH::LGF, BLKF = SH::BLKF;
    constexpr int DEMOFF = SH::DEMOFF, PL = S * RX, LPL = S * TXF;
    constexpr bool PAIR = SH::PAIR;
    constexpr int NTH = SH::NTH;

    extern __shared__ __align__(128) unsigned char smem_ftma[];
    const TL* s_lg = reinterpret_cast<const TL*>(smem_ftma);  // [NLOG][S][TXF]
    float* s_lin = reinterpret_cast<float*>(smem_ftma) + LGF;                          // [NBL][NI][3][S][RX]
    float* s_lhc = s_lin + NBL * BLKF;                   // [2][3][CROWS][CB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_ftma + SH::FLOATS * 4);

    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int H = a.H, W = a.W, c0 = a.c0, nc = a.nc;
    const int x0 = blockIdx.x * TXF, xs0 = x0 - RA;
    const int cxs = (x0 >> 1) & ~3;
    const int y0 = blockIdx.y * a.seg_h, y1 = min(y0 + a.seg_h, H);
    const int nsteps = (y1 - y0 + S - 1) / S;
    // own pixel (PAIR: pixels xi, xi + 1) of this thread in a step
    const int s_t = PAIR ? tid >> 5 : tid >> 6, xi = PAIR ? 2 * (tid & 31) : tid & 63;

    auto lin_block = [&](int j) { return s_lin + ((j + 64 * NBL) % NBL) * BLKF; };
    int sl_i = 0;  // slot of the current step's image block
    auto lin_row_step = [&](int qs, int r, int which) {
        const int rel = r - qs - R + NPRO * S;  // >= 0, S == 4
        int slt = sl_i - NPRO + (rel >> 2);
        slt += slt < 0 ? NBL : 0;
        slt -= slt >= NBL ? NBL : 0;
        return s_lin + slt * BLKF + which * DEMOFF + (rel & 3) * RX;
    };
    auto issue_step = [&](int j) {
        uint64_t* bar = &bars[0];
        const int qs = y0 + j * S;
        mbar_expect_tx(bar, SH::TX_STEP);
        tma_load_4d((void*)s_lg, &mp.lg, x0, qs, 0, b, bar);
        tma_load_4d(lin_block(j), &mp.lin, xs0, qs + R, c0, b, bar);
        if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xs0, qs + R, c0, b, bar);
        if constexpr (PREV) tma_load_4d(lin_block(j) + 2 * DEMOFF, &mp.prv, xs0, qs + R, c0, b, bar);
        if constexpr (UP) tma_load_4d(s_lhc + (j & 1) * SH::LHF, &mp.lhc, cxs, qs >> 1, c0, b, bar);
    };
    const bool col_border = xs0 < 0 || xs0 + RX > W;
    // clamp-to-edge patch of image rows [r0, r1) of the ring (after conversion)
    auto patch_rows = [&](int qs, int r0, int r1) {
        if (col_border) {
            for (int i = tid; i < (r1 - r0) * NI * 3 * RX; i += NTH) {
                const int ri = i % RX, rest = i / RX;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int src = clampi(xs0 + ri, 0, W - 1) - xs0;
                float* row = lin_row_step(qs, r, pc / 3) + (pc % 3) * PL;
                if (src != ri) row[ri] = row[src];
            }
            __syncthreads();
        }
        if (r0 < 0 || r1 > H) {
            for (int i = tid; i < (r1 - r0) * NI * 3 * RX; i += NTH) {
                const int ri = i % RX, rest = i / RX;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int src = clampi(r, 0, H - 1);
                if (src != r)
                    lin_row_step(qs, r, pc / 3)[(pc % 3) * PL + ri] = lin_row_step(qs, src, pc / 3)[(pc % 3) * PL + ri];
            }
            __syncthreads();
        }
    };
    auto convert_rows = [&](float* blk) {  // x0 = noisy / max(d, floor) [, history / max(d, floor)], in place
        if constexpr (L0) {
            for (int i = tid; i < S * RX; i += NTH) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float r = frcp(demod_clamp(blk[DEMOFF + c * PL + i]));
                    blk[c * PL + i] *= r;
                    if constexpr (PREV) blk[2 * DEMOFF + c * PL + i] *= r;
                }
            }
        }
    };

    // ---- prologue: image rows [y0 - NPRO*S + R, y0 + R) and step 0
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bars[1], SH::TX_PRO);
        for (int j = -NPRO; j < 0; ++j) {
            tma_load_4d(lin_block(j), &mp.lin, xs0, y0 + R + j * S, c0, b, &bars[1]);
            if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xs0, y0 + R + j * S, c0, b, &bars[1]);
            if constexpr (PREV) tma_load_4d(lin_block(j) + 2 * DEMOFF, &mp.prv, xs0, y0 + R + j * S, c0, b, &bars[1]);
        }
        issue_step(0);
    }
    mbar_wait(&bars[1], 0);
    for (int j = -NPRO; j < 0; ++j) convert_rows(lin_block(j));
    __syncthreads();
    sl_i = 0;
    patch_rows(y0, y0 + R - NPRO * S, y0 + R);

    float* const ofb = (float*)a.out + (long long)b * a.in_b;
    const unsigned hw32 = (unsigned)H * (unsigned)W;

    for (int i = 0; i < nsteps; ++i, sl_i = (sl_i + 1 == NBL) ? 0 : sl_i + 1) {
        const int qs = y0 + i * S;
        mbar_wait(&bars[0], i & 1);
        if constexpr (PAIR) {
            // softmax of the thread's two pixels (one 32-bit load per channel)
            float2 e2[NW];
            float2 mk2;
            {
                float2 z2[NLOG];
#pragma unroll
                for (int t = 0; t < NLOG; ++t) {
                    const unsigned wv = *reinterpret_cast<const unsigned*>(s_lg + t * LPL + s_t * TXF + xi);
                    z2[t] = make_float2(__uint_as_float(wv << 16), __uint_as_float(wv & 0xffff0000u));
                }
                float ma[2][2] = {{z2[0].x, z2[0].y}, {z2[NLOG - 1].x, z2[NLOG - 1].y}};  // 2 chains per pixel
#pragma unroll
                for (int t = 1; t < NLOG - 1; ++t) {
                    ma[t & 1][0] = fmaxf(ma[t & 1][0], z2[t].x);
                    ma[t & 1][1] = fmaxf(ma[t & 1][1], z2[t].y);
                }
                const float m0 = fmaxf(ma[0][0], ma[1][0]), m1 = fmaxf(ma[0][1], ma[1][1]);
                mk2 = make_float2(m0 * kLog2e, m1 * kLog2e);
                const float2 nm = make_float2(-mk2.x, -mk2.y);
                auto ex = [&](float2 z) {
                    const float2 q = ffma2(z, bcast2(kLog2e), nm);
                    return make_float2(ex2_ftz(q.x), ex2_ftz(q.y));
                };
#pragma unroll
                for (int t = 0; t < NT; ++t) e2[t] = ex(z2[t]);
                if constexpr (UP) {
                    if constexpr (TIED) {
                        const float2 eb = ex(z2[NT]);
#pragma unroll
                        for (int t = NT; t < NW; ++t) e2[t] = eb;
                    } else {
#pragma unroll
                        for (int t = NT; t < NW; ++t) e2[t] = ex(z2[t]);
                    }
                }
            }
            convert_rows(lin_block(i));
            __syncthreads();  // logits consumed, new image rows converted
            if (tid == 0 && i + 1 < nsteps) {
                fence_proxy_async();
                issue_step(i + 1);
            }
            if (col_border || qs + R + S > H) patch_rows(qs, qs + R, qs + R + S);

            const int qy = qs + s_t, gx = x0 + xi;
            if (qy < y1 && gx < W) {
                float2 sa[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int t = 0; t < NW; ++t) sa[t & 1] = fadd2(sa[t & 1], e2[t]);
                const float2 sum2 = fadd2(sa[0], sa[1]);
                const float inv0 = frcp(sum2.x), inv1 = frcp(sum2.y);
                const bool two = gx + 1 < W;
                if (a.lse) {  // base-2 log-sum-exp: the backward's weights 2^(z log2 e - lse)
                    float* lp = (float*)a.lse + (size_t)b * hw32 + (unsigned)qy * (unsigned)W + (unsigned)gx;
                    lp[0] = mk2.x + __log2f(sum2.x);
                    if (two) lp[1] = mk2.y + __log2f(sum2.y);
                }
                float2 acc[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                // window of the pair: smem columns xi + RA - R .. xi + RA + R + 1,
                // read as 8-B pairs from the even column below (PAR = 1 here)
                constexpr int PAR = (RA - R) & 1, NV = (2 * R + 2 + PAR + 1) / 2;
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    const float* lb = lin_row_step(qs, qy + dy, 0) + xi + RA - R - PAR;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float v[2 * NV];
#pragma unroll
                        for (int k2 = 0; k2 < NV; ++k2) {
                            const float2 t2 = *reinterpret_cast<const float2*>(lb + c * PL + 2 * k2);
                            v[2 * k2] = t2.x;
                            v[2 * k2 + 1] = t2.y;
                        }
#pragma unroll
                        for (int dx = -R; dx <= R; ++dx) {
                            const int j = dx + R + PAR;  // pixel 0's window value; pixel 1 takes j + 1
                            const float2 wv = e2[(dy + R) * K + dx + R];
                            if ((j & 1) == 0) {
                                acc[c] = ffma2(wv, make_float2(v[j], v[j + 1]), acc[c]);
                            } else {
                                acc[c].x = fmaf(wv.x, v[j], acc[c].x);
                                acc[c].y = fmaf(wv.y, v[j + 1], acc[c].y);
                            }
                        }
                    }
                }
                if constexpr (UP) {
                    const float* lh = s_lhc + (i & 1) * SH::LHF;
                    const int cyb = qs >> 1;
#pragma unroll
                    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int cy = min((qy + ii) >> 1, a.Hc - 1) - cyb;
                            const int cx0 = min((gx + jj) >> 1, a.Wc - 1) - cxs;
                            const int cx1 = min((gx + 1 + jj) >> 1, a.Wc - 1) - cxs;
                            const float2 wv = e2[NT + 2 * ii + jj];
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                acc[c].x = fmaf(wv.x, lh[(c * CROWS + cy) * CB + cx0], acc[c].x);
                                acc[c].y = fmaf(wv.y, lh[(c * CROWS + cy) * CB + cx1], acc[c].y);
                            }
                        }
                }
                const unsigned po = (unsigned)qy * (unsigned)W + (unsigned)gx;
                const float* dr = L0 ? lin_row_step(qs, qy, 1) + xi + RA : nullptr;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (c >= nc) break;
                    float v0 = acc[c].x * inv0, v1 = acc[c].y * inv1;
                    if constexpr (L0) {
                        v0 *= demod_clamp(dr[c * PL]);
                        v1 *= demod_clamp(dr[c * PL + 1]);
                    }
                    float* op = ofb + po + c * hw32;
                    if (two && ((po & 1) == 0)) {
                        *reinterpret_cast<float2*>(op) = make_float2(v0, v1);
                    } else {
                        op[0] = v0;
                        if (two) op[1] = v1;
                    }
                }
            }
        } else {
        // softmax of this thread's own pixel, from smem into registers
        float e[NW];
        float mk;
        {
            float z[NLOG];
#pragma unroll
            for (int t = 0; t < NLOG; ++t) z[t] = to_f32(s_lg[t * LPL + s_t * TXF + xi]);
            mk = max4(z) * kLog2e;
#pragma unroll
            for (int t = 0; t < NT; ++t) e[t] = ex2_ftz(fmaf(z[t], kLog2e, -mk));
            if constexpr (UP) {
                if constexpr (TIED) {
                    const float eb = ex2_ftz(fmaf(z[NT], kLog2e, -mk));
#pragma unroll
                    for (int t = NT; t < SH::NW0; ++t) e[t] = eb;
                } else {
#pragma unroll
                    for (int t = NT; t < SH::NW0; ++t) e[t] = ex2_ftz(fmaf(z[t], kLog2e, -mk));
                }
            }
            if constexpr (PREV) {
#pragma unroll
                for (int t = 0; t < NT; ++t) e[SH::NW0 + t] = ex2_ftz(fmaf(z[SH::NLOG0 + t], kLog2e, -mk));
            }
        }
        convert_rows(lin_block(i));
        __syncthreads();  // logits consumed, new image rows converted
        if (tid == 0 && i + 1 < nsteps) {
            fence_proxy_async();
            issue_step(i + 1);
        }
        if (col_border || qs + R + S > H) patch_rows(qs, qs + R, qs + R + S);

        const int qy = qs + s_t, gx = x0 + xi;
        if (qy < y1 && gx < W) {
            const float sum = sum4(e);
            const float inv = frcp(sum);
            // base-2 log-sum-exp: the backward's weights 2^(z log2 e - lse)
            if (a.lse) ((float*)a.lse)[(size_t)b * hw32 + (unsigned)qy * (unsigned)W + (unsigned)gx] = mk + __log2f(sum);
            float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int dy = -R; dy <= R; ++dy) {
                const float* lr = lin_row_step(qs, qy + dy, 0) + xi + RA;
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                    const float wv = e[(dy + R) * K + dx + R];
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[c] = fmaf(wv, lr[c * PL + dx], acc[c]);
                }
            }
            if constexpr (UP) {
                const float* lh = s_lhc + (i & 1) * SH::LHF;
                const int cyb = qs >> 1;
#pragma unroll
                for (int ii = 0; ii < 2; ++ii)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int cy = min((qy + ii) >> 1, a.Hc - 1) - cyb;
                        const int cx = min((gx + jj) >> 1, a.Wc - 1) - cxs;
                        const float wv = e[NT + 2 * ii + jj];
#pragma unroll
                        for (int c = 0; c < 3; ++c) acc[c] = fmaf(wv, lh[(c * CROWS + cy) * CB + cx], acc[c]);
                    }
            }
            if constexpr (PREV) {
                // temporal taps over the (converted) history plane group
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    const float* pr = lin_row_step(qs, qy + dy, 2) + xi + RA;
#pragma unroll
                    for (int dx = -R; dx <= R; ++dx) {
                        const float wv = e[SH::NW0 + (dy + R) * K + dx + R];
#pragma unroll
                        for (int c = 0; c < 3; ++c) acc[c] = fmaf(wv, pr[c * PL + dx], acc[c]);
                    }
                }
            }
            const unsigned po = (unsigned)qy * (unsigned)W + (unsigned)gx;
            const float* dr = L0 ? lin_row_step(qs, qy, 1) + xi + RA : nullptr;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c >= nc) break;
                float v = acc[c] * inv;
                if constexpr (L0) v *= demod_clamp(dr[c * PL]);
                ofb[po + c * hw32] = v;
            }
        }
        }
    }
}

}  // namespace ssb
