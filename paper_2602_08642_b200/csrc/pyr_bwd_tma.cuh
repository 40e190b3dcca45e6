// Level backward, TMA-pipelined strip walker (fp32 images, fp32 or bf16
// logits, no temporal group; other configurations use k_pyr_bwd in
// pyr_kernels.cuh).
//
// Same column-strip / S-row-step structure and the same arithmetic as
// k_pyr_bwd, with the data movement rebuilt for sm_100a:
//  * every global input of a step arrives by cp.async.bulk.tensor (TMA) into
//    shared memory, issued by one thread one step ahead (double-buffered
//    logits, block rings for the image rows), completion on mbarriers --
//    no per-thread address math, no load latency on the critical path,
//    out-of-image texels arrive as zeros (clamp-to-edge is patched in smem);
//  * the softmax is not normalised per weight: s_g holds G * (1/sum) and the
//    softmax backward is rewritten in terms of the exponentials;
//  * the gather-transpose (B2) and upsample-transpose (B3) run one thread per
//    (column, channel) over the S rows with register accumulators, so one
//    accumulator ring suffices.
// ~104 KB shared memory at k = 5 -> 2 CTAs (16 warps) per SM.
#pragma once

#include "pyr_kernels.cuh"
#include "tma.cuh"

namespace ssb {

struct TmaMaps {
    CUtensorMap lg;   // logits (W, H, NLOG, B), box (RX, S, NLOG)
    CUtensorMap lin;  // noisy (level 0) or L^l, box (RX, S, 3)
    CUtensorMap dem;  // demod (level 0), box (RX, S, 3)
    CUtensorMap up;   // upstream (level 0) or ghat^l, box (RX, S, 3)
    CUtensorMap out;  // forward output (level 0), box (RX, S + R, 3)
    CUtensorMap lhc;  // coarse Lhat^{l+1}, box (CB, S/2 + 1, 3)
};

template <int K, typename TL, bool L0, bool UP, bool TIED>
struct TmaShape {
    static constexpr int R = K / 2, NT = K * K, NUP = UP ? 4 : 0, NW = NT + NUP;
    static constexpr int NLOG = NT + (UP ? (TIED ? 1 : 4) : 0);
    // TMA boxes must start 16-B aligned in x: smem column 0 is global x0 - RA
    // with RA = 16 B of logits (4 fp32 / 8 bf16), rows are RX = TXB + 2 RA
    // wide, TXB a multiple of RA.
    static constexpr int LGE = (int)sizeof(TL);  // logit element size
    static constexpr bool SEP = LGE != 4;        // bf16: staging box + separate fp32 exponentials
    static constexpr int RA = 16 / LGE, S = 4;
    static constexpr int TXB = ((64 - 2 * R) / RA) * RA, RX = TXB + 2 * RA, RW = TXB + 2 * R;
    static constexpr int TXC = TXB / 2;
    static constexpr int NPRO = (2 * R + S - 1) / S;  // image-ring blocks above step 0
    static constexpr int NBL = NPRO + 2;               // image-ring blocks (incl. prefetch)
    static constexpr int NBU = 3;                      // upstream-ring blocks
    static constexpr int NI = L0 ? 2 : 1;              // image planes per block (x0 [, demod])
    static constexpr int FFQ = R >= S ? S * ((R - S + 1 + S - 1) / S) : 0;
    static constexpr int AR = S + 2 * R + FFQ;         // accumulator ring rows
    static constexpr int CR = 4, CB = 36, CROWS = S / 2 + 1;  // coarse box: aligned start, TXC + 1 + 2 cols
    // every TMA destination starts 128-B aligned (sizes rounded up to 32 floats)
    static constexpr int al32(int n) { return (n + 31) & ~31; }
    static constexpr int LGF = al32(NLOG * S * RX);    // floats per exponentials buffer
    // logits staging (storage type): fp32 = the two exponential buffers
    // themselves (in place); bf16 = one staging box + one fp32 buffer
    static constexpr int LGS = SEP ? al32((NLOG * S * RX * LGE + 3) / 4) : 0;
    static constexpr int LGBUF = SEP ? LGF + LGS : 2 * LGF;
    static constexpr int DEMOFF = al32(3 * S * RX);    // demod plane offset inside a ring block
    static constexpr int BLKF = NI * DEMOFF;           // floats per image-ring block
    static constexpr int UPF = al32(3 * S * RX);
    static constexpr int OUTF = L0 ? al32(3 * (S + R) * RX) : 0;
    static constexpr int LHF = UP ? al32(3 * CROWS * CB) : 0;
    // transaction bytes (exact box sizes, not the padded buffer sizes)
    static constexpr uint32_t TX_IMG = 3 * S * RX * 4;
    static constexpr uint32_t TX_STEP = NLOG * S * RX * LGE + (NI + 1) * TX_IMG + (UP ? 3 * CROWS * CB * 4 : 0);
    static constexpr uint32_t TX_OUT = 3 * (S + R) * RX * 4;
    static constexpr uint32_t TX_PRO = NPRO * NI * TX_IMG;
    static constexpr size_t FLOATS = (size_t)LGBUF + NBL * BLKF + NBU * UPF + OUTF + 2 * LHF +
                                     3 * S * RX + S * RX + AR * 3 * TXB + (UP ? CR * 3 * TXC : 0);
    static constexpr size_t SMEM = FLOATS * 4 + 64;
};

template <int K, typename TL, bool L0, bool UP, bool TIED>
__global__ void __launch_bounds__(256, 2)
    k_pyr_bwd_tma(const BwdLevel a, const __grid_constant__ TmaMaps mp) {
    using SH = TmaShape<K, TL, L0, UP, TIED>;
    constexpr bool SEP = SH::SEP;
    constexpr int R = SH::R, NT = SH::NT, NW = SH::NW, NLOG = SH::NLOG, S = SH::S, RX = SH::RX;
    constexpr int RA = SH::RA, RW = SH::RW;
    constexpr int TXB = SH::TXB, TXC = SH::TXC, NPRO = SH::NPRO, NBL = SH::NBL, NBU = SH::NBU;
    constexpr int NI = SH::NI, AR = SH::AR, CR = SH::CR, CB = SH::CB, CROWS = SH::CROWS;
    constexpr int LGF = SH::LGF, BLKF = SH::BLKF, UPF = SH::UPF, DEMOFF = SH::DEMOFF;
    constexpr int PL = S * RX;  // floats per image plane in a block
    constexpr int RUP = (R + 1) & ~1;

    extern __shared__ __align__(128) unsigned char smem_tma[];
    float* s_lg = reinterpret_cast<float*>(smem_tma);  // [2][NLOG][S][RX] | [NLOG][S][RX] + staging
    float* s_lin = s_lg + SH::LGBUF;                   // [NBL][NI][3][S][RX]
    float* s_up = s_lin + NBL * BLKF;                  // [NBU][3][S][RX]
    float* s_out = s_up + NBU * UPF;                   // [3][S+R][RX]
    float* s_lhc = s_out + SH::OUTF;                   // [2][3][CROWS][CB]
    float* s_g = s_lhc + 2 * SH::LHF;                  // [3][S][RX]  G * (1/sum)
    float* s_inv = s_g + 3 * PL;                       // [S][RX]
    float* s_acc = s_inv + PL;                         // [AR][3][TXB]
    float* s_cac = s_acc + AR * 3 * TXB;               // [CR][3][TXC]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + SH::FLOATS * 4);

    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int nc = a.nc, H = a.H, W = a.W, c0 = a.c0;
    const int x0 = blockIdx.x * TXB, xs0 = x0 - RA;   // xs0: global x of smem column 0
    const int cxs = (x0 >> 1) & ~3, cxo = (x0 >> 1) - cxs;  // coarse box start (aligned), offset
    const int y0 = blockIdx.y * a.seg_h, y1 = min(y0 + a.seg_h, H);
    const int qstart = max(y0 - RUP, 0);
    const int qend = min(y1 + R, H);
    const int nsteps = (qend - qstart + S - 1) / S;
    const unsigned hw32 = (unsigned)H * (unsigned)W;
    auto slot = [](int P) { return (P + 8 * AR) % AR; };
    auto lin_block = [&](int j) { return s_lin + ((j + 64 * NBL) % NBL) * BLKF; };
    int sl_i = 0;  // ring slot of the current step's image block (i mod NBL), kept incrementally
    // image-ring row r for rows of the current step's window [qs - NPRO*S + R, qs + 2S + R)
    auto lin_row_step = [&](int qs, int r, int which) {
        const int rel = r - qs - R + NPRO * S;      // >= 0
        int slt = sl_i - NPRO + (rel >> 2);         // S == 4
        slt += slt < 0 ? NBL : 0;
        slt -= slt >= NBL ? NBL : 0;
        return s_lin + slt * BLKF + which * DEMOFF + (rel & 3) * RX;
    };
    auto up_block = [&](int j) { return s_up + ((j + 64 * NBU) % NBU) * UPF; };
    // image-ring row r (absolute) -> pointer to plane `which` (0: x0/L, 1: demod), channel 0
    auto lin_row = [&](int r, int which) {
        const int rel = r - qstart - R + NPRO * S;
        return lin_block(rel / S - NPRO) + which * DEMOFF + (rel % S) * RX;
    };
    auto up_row = [&](int r) {  // q row r -> upstream ring, channel 0
        const int rel = r - qstart + S;
        return up_block(rel / S - 1) + (rel % S) * RX;
    };

    // ---- TMA issue (thread 0)
    auto issue_step = [&](int j) {
        uint64_t* bar = &bars[j & 1];
        const int qs = qstart + j * S;
        mbar_expect_tx(bar, SH::TX_STEP);
        tma_load_4d(SEP ? s_lg + LGF : s_lg + (j & 1) * LGF, &mp.lg, xs0, qs, 0, b, bar);
        tma_load_4d(lin_block(j), &mp.lin, xs0, qs + R, c0, b, bar);
        if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xs0, qs + R, c0, b, bar);
        tma_load_4d(up_block(j), &mp.up, xs0, qs, c0, b, bar);
        if constexpr (UP) tma_load_4d(s_lhc + (j & 1) * SH::LHF, &mp.lhc, cxs, qs >> 1, c0, b, bar);
    };
    auto issue_out = [&](int j) {
        if constexpr (L0) {
            mbar_expect_tx(&bars[2], SH::TX_OUT);
            tma_load_4d(s_out, &mp.out, xs0, qstart + j * S - R, c0, b, &bars[2]);
        }
    };

    // ---- clamp-to-edge patch of image-ring rows [r0, r1) (after conversion)
    const bool col_border = xs0 < 0 || xs0 + RX > W;
    auto patch_rows = [&](int r0, int r1) {
        if (col_border) {
            for (int i = tid; i < (r1 - r0) * NI * 3 * RX; i += 256) {
                const int ri = i % RX, rest = i / RX;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int src = clampi(xs0 + ri, 0, W - 1) - xs0;
                float* row = lin_row(r, pc / 3) + (pc % 3) * PL;
                if (src != ri) row[ri] = row[src];
            }
            __syncthreads();
        }
        if (r0 < 0 || r1 > H) {
            for (int i = tid; i < (r1 - r0) * NI * 3 * RX; i += 256) {
                const int ri = i % RX, rest = i / RX;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int src = clampi(r, 0, H - 1);
                if (src != r) lin_row(r, pc / 3)[(pc % 3) * PL + ri] = lin_row(src, pc / 3)[(pc % 3) * PL + ri];
            }
            __syncthreads();
        }
    };
    // x0 = noisy / max(d, floor) in place (level 0), for ring rows of block j
    auto convert_block = [&](int j, int s, int ri) {
        if constexpr (L0) {
            float* blk = lin_block(j);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float d = blk[DEMOFF + c * PL + s * RX + ri];
                blk[c * PL + s * RX + ri] *= rcp_dem(demod_clamp(d));
            }
        }
    };

    // ---- prologue
    for (int i = tid; i < AR * 3 * TXB; i += 256) s_acc[i] = 0.f;
    if constexpr (UP)
        for (int i = tid; i < CR * 3 * TXC; i += 256) s_cac[i] = 0.f;
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bars[3], SH::TX_PRO);
        for (int j = -NPRO; j < 0; ++j) {
            tma_load_4d(lin_block(j), &mp.lin, xs0, qstart + R + j * S, c0, b, &bars[3]);
            if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xs0, qstart + R + j * S, c0, b, &bars[3]);
        }
        if (nsteps > 0) issue_step(0);
        issue_out(0);
    }
    mbar_wait(&bars[3], 0);
    for (int i = tid; i < NPRO * S * RX; i += 256) {
        const int jj = i / (S * RX), rem = i % (S * RX);
        convert_block(jj - NPRO, rem / RX, rem % RX);
    }
    __syncthreads();
    patch_rows(qstart + R - NPRO * S, qstart + R);

    int next_flush = max(qstart - R, 0);
    int cnext = qstart >> 1;
    const int s_a = tid >> 6, rw_a = tid & 63;  // phase A: S rows x 64 threads, RW <= 64 used
    const int ri_a = RA - R + rw_a;               // smem column of this thread's region pixel
    const bool act_a = rw_a < RW;

    for (int i = 0; i < nsteps; ++i, sl_i = (sl_i + 1 == NBL) ? 0 : sl_i + 1) {
        const int qs = qstart + i * S;
        float* lgb = SEP ? s_lg : s_lg + (i & 1) * LGF;  // exponentials of this step
        const TL* lgs = reinterpret_cast<const TL*>(SEP ? s_lg + LGF : lgb);  // staged logits
        mbar_wait(&bars[i & 1], (i >> 1) & 1);

        // ------------------------------------------------ A: softmax, G', x0
        if (act_a) {
            float e[NLOG];
#pragma unroll
            for (int t = 0; t < NLOG; ++t) e[t] = to_f32(lgs[t * PL + s_a * RX + ri_a]);
            float m = e[0];
#pragma unroll
            for (int t = 1; t < NLOG; ++t) m = fmaxf(m, e[t]);
            const float mk = m * kLog2e;
            float sum = 0.f;
#pragma unroll
            for (int t = 0; t < NLOG; ++t) {
                e[t] = ex2_ftz(fmaf(e[t], kLog2e, -mk));
                sum += (TIED && t == NT) ? 4.f * e[t] : e[t];
            }
#pragma unroll
            for (int t = 0; t < NLOG; ++t) lgb[t * PL + s_a * RX + ri_a] = e[t];
            const float inv = __fdividef(1.f, sum);
            s_inv[s_a * RX + ri_a] = inv;
            convert_block(i, s_a, ri_a);  // (block i = slot sl_i)
            const float* ub = up_block(i) + s_a * RX + ri_a;
            float dq[3] = {1.f, 1.f, 1.f};
            if constexpr (L0) {
                const float* dr = lin_row_step(qs, qs + s_a, 1) + ri_a;
#pragma unroll
                for (int c = 0; c < 3; ++c) dq[c] = demod_clamp(dr[c * PL]);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) s_g[c * PL + s_a * RX + ri_a] = ub[c * PL] * dq[c] * inv;
        }
        __syncthreads();
        // every thread has finished the previous step's flush and this step's
        // phase A: the buffers of step i+1 (and this step's out box) are free
        if (tid == 0) {
            if (i + 1 < nsteps) {
                fence_proxy_async();
                issue_step(i + 1);
            }
            if (i > 0) issue_out(i);
        }
        if (col_border || qs + R + S > H) patch_rows(qs + R, qs + R + S);

        // ------------------------------------------------ B1: logit gradients
        if (a.want_params && tid < S * TXB) {
            const int s = tid / TXB, xi = tid - s * TXB;
            const int qy = qs + s, gx = x0 + xi, ri = xi + RA;
            if (qy >= y0 && qy < y1 && gx < W) {
                float gq[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) gq[c] = s_g[c * PL + s * RX + ri];
                const float inv = s_inv[s * RX + ri];
                float gw[NW];
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
                    const float* lr = lin_row_step(qs, qy + dy, 0) + ri;
#pragma unroll
                    for (int dx = -R; dx <= R; ++dx) {
                        float acc = 0.f;
#pragma unroll
                        for (int c = 0; c < 3; ++c) acc = fmaf(gq[c], lr[c * PL + dx], acc);
                        gw[(dy + R) * K + dx + R] = acc;
                    }
                }
                if constexpr (UP) {
                    const float* lh = s_lhc + (i & 1) * SH::LHF;
                    const int cyb = qs >> 1, cxb = cxs;
#pragma unroll
                    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int cy = min((qy + ii) >> 1, a.Hc - 1) - cyb;
                            const int cx = min((gx + jj) >> 1, a.Wc - 1) - cxb;
                            float acc = 0.f;
#pragma unroll
                            for (int c = 0; c < 3; ++c) acc = fmaf(gq[c], lh[(c * CROWS + cy) * CB + cx], acc);
                            gw[NT + 2 * ii + jj] = acc;
                        }
                }
                const float* ep = lgb + s * RX + ri;
                float dot = 0.f;
#pragma unroll
                for (int t = 0; t < NW; ++t) {
                    const int slot_t = (TIED && t >= NT) ? NT : t;
                    dot = fmaf(ep[slot_t * PL], gw[t], dot);
                }
                const float inner = dot * inv;
                TL* const gfb = (TL*)a.glogits + (long long)b * a.lg_b;  // uniform per CTA
                const unsigned po = (unsigned)qy * (unsigned)W + (unsigned)gx;
                const bool acc_mode = a.accum != 0;
                float gz[NLOG];
#pragma unroll
                for (int t = 0; t < NT; ++t) gz[t] = ep[t * PL] * (gw[t] - inner);
                if constexpr (UP) {
                    if constexpr (TIED) {
                        gz[NT] = ep[NT * PL] * (((gw[NT] + gw[NT + 1]) + (gw[NT + 2] + gw[NT + 3])) - 4.f * inner);
                    } else {
#pragma unroll
                        for (int t = NT; t < NW; ++t) gz[t] = ep[t * PL] * (gw[t] - inner);
                    }
                }
#pragma unroll
                for (int t = 0; t < NLOG; ++t) st_gz(gfb + (po + t * hw32), gz[t], acc_mode);
            }
        }

        // ------------------------------------------------ B2: gather transpose
        if (tid >= 256 - 3 * TXB) {
            const int u2 = tid - (256 - 3 * TXB);
            const int c = u2 / TXB, xi = u2 - c * TXB;
            const int gx = x0 + xi, ri = xi + RA;
            if (gx < W) {
                float acc[S + 2 * R];
#pragma unroll
                for (int k2 = 0; k2 < S + 2 * R; ++k2) acc[k2] = 0.f;
#pragma unroll
                for (int s = 0; s < S; ++s) {
#pragma unroll
                    for (int dx = -R; dx <= R; ++dx) {
                        const int rj = ri - dx;
                        const float g = s_g[c * PL + s * RX + rj];
#pragma unroll
                        for (int d = 0; d < K; ++d)
                            acc[s + d] = fmaf(lgb[(d * K + dx + R) * PL + s * RX + rj], g, acc[s + d]);
                    }
                }
                if (gx == 0 || gx == W - 1) {
                    // clamp fold along x: logical columns beyond the border land on it
                    for (int side = 0; side < 2; ++side) {
                        if ((side == 0 && gx != 0) || (side == 1 && gx != W - 1)) continue;
                        for (int e = 1; e <= R; ++e) {
                            const int Pc = side == 0 ? -e : W - 1 + e;
                            for (int dx = -R; dx <= R; ++dx) {
                                const int qx = Pc - dx;
                                if (qx < 0 || qx >= W) continue;
                                const int rj = qx - xs0;
#pragma unroll
                                for (int s = 0; s < S; ++s) {
                                    const float g = s_g[c * PL + s * RX + rj];
#pragma unroll
                                    for (int d = 0; d < K; ++d)
                                        acc[s + d] = fmaf(lgb[(d * K + dx + R) * PL + s * RX + rj], g, acc[s + d]);
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int k2 = 0; k2 < S + 2 * R; ++k2) s_acc[(slot(qs - R + k2) * 3 + c) * TXB + xi] += acc[k2];
            }
        }
        // ------------------------------------------------ B3: upsample transpose
        if constexpr (UP) {
            // B3 items on the threads not running B2 first, then wrap onto the top threads
            const int nb3 = 256 - 3 * TXB;
            const int u = tid < nb3 ? tid : (tid >= 256 - (3 * TXC - nb3) ? nb3 + tid - (256 - (3 * TXC - nb3)) : -1);
            if (u >= 0 && u < 3 * TXC) {
                const int c = u / TXC, cxi = u - c * TXC;
                const int X = (x0 >> 1) + cxi;
                if (X < a.Wc) {
                    float cv[CROWS];
#pragma unroll
                    for (int k2 = 0; k2 < CROWS; ++k2) cv[k2] = 0.f;
                    const int cyb = qs >> 1;  // qs is even
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const int qy = qs + s;
                        if (qy >= H) break;
                        // parents: row s/2 (tap i = 0) and (s+1)/2 (tap i = 1), the latter
                        // clamped onto the last coarse row when it falls off the image
                        const bool clamp1 = ((qy + 1) >> 1) > a.Hc - 1;
#pragma unroll
                        for (int k3 = -1; k3 <= 1; ++k3) {
                            const int xx = 2 * X + k3;
                            if (xx < 0 || xx >= W) continue;
                            const int rj = xx - xs0;
                            const float g = s_g[c * PL + s * RX + rj];
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj) {
                                if (min((xx + jj) >> 1, a.Wc - 1) != X) continue;
                                const float w0 = lgb[(TIED ? NT : NT + jj) * PL + s * RX + rj];
                                const float w1 = lgb[(TIED ? NT : NT + 2 + jj) * PL + s * RX + rj];
                                cv[s >> 1] = fmaf(w0, g, cv[s >> 1]);
                                if (clamp1) cv[(s + 1) >> 1 == 0 ? 0 : ((s + 1) >> 1) - 1] = fmaf(w1, g, cv[(s + 1) >> 1 == 0 ? 0 : ((s + 1) >> 1) - 1]);
                                else cv[(s + 1) >> 1] = fmaf(w1, g, cv[(s + 1) >> 1]);
                            }
                        }
                    }
#pragma unroll
                    for (int k2 = 0; k2 < CROWS; ++k2)
                        s_cac[(((cyb + k2) & (CR - 1)) * 3 + c) * TXC + cxi] += cv[k2];
                }
            }
        }
        __syncthreads();

        // ------------------------------------------------ flush finished rows
        const bool bottom = qs + S >= H;
        const int pend = max(bottom ? H : qs + S - R, next_flush);
        if constexpr (L0) mbar_wait(&bars[2], i & 1);
        for (int k2 = tid; k2 < (pend - next_flush) * TXB; k2 += 256) {
            const int rr = k2 / TXB, xi = k2 - rr * TXB;
            const int P = next_flush + rr, gx = x0 + xi;
            float v[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float* p = &s_acc[(slot(P) * 3 + c) * TXB + xi];
                v[c] = *p;
                *p = 0.f;
            }
            if (P == 0)
                for (int e = 1; e <= R; ++e)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float* p = &s_acc[(slot(-e) * 3 + c) * TXB + xi];
                        v[c] += *p;
                        *p = 0.f;
                    }
            if (P == H - 1)
                for (int e = 1; e <= R; ++e)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float* p = &s_acc[(slot(H - 1 + e) * 3 + c) * TXB + xi];
                        v[c] += *p;
                        *p = 0.f;
                    }
            if (P < y0 || P >= y1 || gx >= W) continue;
            const long long off = (long long)P * W + gx;
            float* glo = (float*)a.gl_out + (long long)b * a.in_b;
            if constexpr (L0) {
                float* gdo = a.gdc_out ? (float*)a.gdc_out + (long long)b * a.in_b : nullptr;
                const int ri = xi + RA;
                const float* xr = lin_row_step(qs, P, 0) + ri;
                const float* dr = lin_row_step(qs, P, 1) + ri;
                const float* ur = up_row(P) + ri;
                const float* orow = s_out + (P - (qs - R)) * RX + ri;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (c >= nc) break;
                    const long long o = c * a.in_c + off;
                    if (a.demod) {
                        const float rd = rcp_dem(demod_clamp(dr[c * PL]));
                        glo[o] = v[c] * rd;
                        if (gdo) gdo[o] = ur[c * PL] * (orow[c * (S + R) * RX] * rd) - v[c] * xr[c * PL] * rd;
                    } else {
                        glo[o] = v[c];
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c < nc) glo[c * a.in_c + off] = v[c];
            }
        }
        next_flush = pend;

        if constexpr (UP) {
            const int cend = bottom ? a.Hc : (qs + S) >> 1;
            const int own0 = y0 >> 1, own1 = (y1 + 1) >> 1;
            for (int k2 = tid; k2 < (cend - cnext) * TXC; k2 += 256) {
                const int rr = k2 / TXC, cxi = k2 - rr * TXC;
                const int Y = cnext + rr, X = (x0 >> 1) + cxi;
                float v[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float* p = &s_cac[((Y & (CR - 1)) * 3 + c) * TXC + cxi];
                    v[c] = *p;
                    *p = 0.f;
                }
                if (Y < own0 || Y >= own1 || X >= a.Wc) continue;
                float* gc = (float*)a.ghat_c + (long long)b * a.c_b + (long long)Y * a.Wc + X;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c < nc) gc[c * a.c_c] = v[c];
            }
            cnext = cend;
        }
        // no barrier here: the next phase A touches none of the buffers this
        // flush reads; the next prefetch is issued after the next phase-A barrier
    }
}

}  // namespace ssb
