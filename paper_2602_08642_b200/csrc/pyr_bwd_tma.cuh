// Level backward, TMA-pipelined strip walker (fp32 images, fp32 or bf16
// logits, no temporal group; other configurations use k_pyr_bwd in
// pyr_kernels.cuh).  Reference: reconstruct_backward (pyramid.py:362-455).
//
// CTA = column strip of TXB own columns (+R halo columns each side) x one
// segment of rows, walked in steps of S = 4 rows.  Data movement: every
// global input of a step (logits, image rows R ahead, upstream, forward
// output, coarse Lhat rows) arrives by cp.async.bulk.tensor into shared
// memory, issued by one thread one step ahead, completion on mbarriers;
// out-of-image texels arrive as zeros (clamp-to-edge is patched in smem).
//
// Per step, with w = e * inv the softmax of the pixel's logits:
//  A  (all warps) exponentials e, G = gout * inv, and the softmax backward's
//     inner product from the level output the tape already holds:
//        sum_t w_t gw_t = sum_c gout_c * y_c(q)   (y = the level output),
//     inner' = inv * sum_c gin_c out_c (level 0: gin = upstream, out = the
//     remodulated output; level l: gin = ghat^l, out = Lhat^l).  So every
//     tap's logit gradient is final as soon as its gw is known:
//        g_logit_t = e_t * (sum_c G_c x_c(q + o_t) - inner').
//  Then the warps split by role (one loop each, CTA barriers in step):
//  B1 (warps 0-3) logit gradients, one thread per horizontal pixel QUAD
//     (float4 shared loads, FFMA2 over tap pairs, 16-B streaming stores),
//     and the upsample transpose (B3) separably per (coarse column, channel).
//  B2 (warps 4-7) gather-transpose, one thread per (column, group of tap
//     columns) with a register window of the S + 2R output rows the step
//     touches; finished rows are reduced across the groups with warp
//     shuffles and written directly (level 0: partial g_noisy and g_demod) --
//     no accumulator ring in shared memory, no atomics, deterministic.
#pragma once

#include <type_traits>

#include "pyr_kernels.cuh"
#include "tma.cuh"

namespace ssb {

struct TmaMaps {
    CUtensorMap lg;   // logits (W, H, NLOG, B), box (RX, S, NLOG)
    CUtensorMap lin;  // noisy (level 0) or L^l, box (RXI, S, 3)
    CUtensorMap dem;  // demod (level 0), box (RXI, S, 3)
    CUtensorMap up;   // upstream (level 0) or ghat^l, box (RXI, S, 3)
    CUtensorMap out;  // forward output (level 0) or Lhat^l, box (RXI, S, 3)
    CUtensorMap lhc;  // coarse Lhat^{l+1}, box (CB, S/2 + 1, 3)
    CUtensorMap t1;   // CH (level 0 last): T1 = level-1 input gradient incl. the pool chain, box (CB, CT, 3)
    CUtensorMap lse;  // the forward's base-2 log-sum-exp, box (RXI, S, 1)
    CUtensorMap gd;   // temporal pass: g_demod as level 0 wrote it, box (RXI, S, 3) at the flush rows
};

// CH: level 0 runs after the coarser levels (pyr_chain.cuh): no upsample
// transpose (ghat^1 comes from k_up_transpose) and the flush adds the pool
// chain T1(parent) / count, writing the final g_noisy / g_demod
// NST = TMA ring depth: step j's boxes land in slot j % NST and are issued
// NST - 1 steps ahead (at the top of step j - NST + 1, right after the end
// barrier of step j - NST, whose slot it reuses).  TXO != 0 overrides the
// strip's own-column count (a multiple of RA).
// MODE bits: kBwdLsw forces the log-sum-exp weights (LSW) at any k; kBwdTp =
// the temporal-group pass of level 0 with history (image = the warped
// history, logits = the temporal channels, flush = g_prev and the history
// term of g_demod)
constexpr int kBwdLsw = 1, kBwdTp = 2;
template <int K, typename TL, bool L0, bool UP, bool TIED, bool CH = false, int SS = 4, int NST = 2, int TXO = 0,
          int MODE = 0>
struct TmaShape {
    static constexpr int R = K / 2, NT = K * K, NUP = UP ? 4 : 0, NW = NT + NUP;
    static constexpr int NLOG = NT + (UP ? (TIED ? 1 : 4) : 0);
    // TMA boxes must start 16-B aligned in x: smem column 0 is global x0 - RA
    // with RA = 16 B of logits (4 fp32 / 8 bf16), rows are RX = TXB + 2 RA
    // wide, TXB a multiple of RA.  k = 7 uses narrower strips (shared memory).
    static constexpr int LGE = (int)sizeof(TL);  // logit element size
    // SS = rows per step: 4 (256 threads, 2 CTAs per SM) or 8 (512 threads, one
    // CTA per SM: twice the TMA box rows per request)
    static constexpr int RA = 16 / LGE, S = SS;
    static constexpr int NTH = 64 * SS, HN = NTH / 2;
    static constexpr int TXW = ((64 - 2 * R) / RA) * RA;
    static constexpr int TXB = TXO ? TXO : (K >= 7 ? 32 : TXW), RX = TXB + 2 * RA, RW = TXB + 2 * R;
    static constexpr int TXC = TXB / 2, NQUAD = TXB / 4;
    // fp32 image boxes need only 16 B = 4 columns of alignment halo: image
    // rows are RXI = TXB + 8 wide from global x0 - 4, so image column =
    // logit column - DI (bf16: DI = 4, fp32: 0)
    static constexpr int RAI = 4, DI = RA - RAI, RXI = TXB + 2 * RAI;
    static constexpr int NPRO = (2 * R + S - 1) / S;  // image-ring blocks above step 0
    static constexpr int NBL = NPRO + NST;             // image-ring blocks (incl. prefetch)
    // upstream ring (level 0: the flush needs u * out, R rows behind); other
    // levels and the forward output / Lhat^l: one block (read in phase A only)
    static constexpr int NBU0 = L0 ? (R + S - 1) / S + NST : NST;  // gradient-input ring (NST at l >= 1 with early issue)
    static constexpr int NI = L0 ? 2 : 1;              // image planes per block (x0 [, demod])
    // B1: S * NQUAD pixel quads on warps 0-3; tap rows split in B1SPL warp-uniform parts
    static constexpr int NB1 = S * NQUAD;
    // quads of a row occupy QS = 8 or 16 consecutive lanes (one idle slot at
    // 15 quads): a 16-B shared access's 8-lane phase never straddles two rows,
    // whose 272-B pitch would put two lanes of the phase on the same banks
    static constexpr int QS = NQUAD <= 8 ? 8 : 16;
    static constexpr int NB1S = S * QS;
    static constexpr int B1SPL = NB1S <= HN / 4 ? 4 : (NB1S <= HN / 2 ? 2 : 1);
    static constexpr int B1ITEMS = HN / B1SPL;
    static constexpr int DYS = (K + B1SPL - 1) / B1SPL;  // tap rows per part
    // B2: TXB columns x B2SPL tap-column groups on warps 4-7 (adjacent lanes)
    static constexpr int B2SPL = TXB * 4 <= HN ? 4 : (TXB * 2 <= HN ? 2 : 1);
    // B2W: each tap-column group (part) on its own warp(s) -- 32 consecutive
    // columns per warp, so the parts' shared loads (exponentials of different
    // tap planes) cannot collide on banks -- and the parts' window partials
    // summed through shared memory at the flush (each part owns rows r with
    // r % B2SPL == part) instead of lane shuffles
#ifndef SSB_B2W
#define SSB_B2W 1
#endif
    // (measured, same-box A/B: k7 bf16 level 0 -13%, k5 level 1 -4%; k5 level
    // 0, whose two parts split the 5 tap columns 3:2, +3..7% -- kept on shuffles)
    static constexpr bool B2W = SSB_B2W && SS == 4 && (B2SPL == 4 || (B2SPL == 2 && !L0));
    static constexpr int WPP = B2W ? 4 / B2SPL : 1;  // warps per part (the 4 B2 warps)
    static constexpr int B2C = 32 * WPP;              // column slots per part
    static constexpr int AW = S + 2 * R, NPW = (AW + 1) / 2;  // output-row window (float2 pairs)
    // coarse box: 16-B aligned start (x0/2 rounded down to 4), TXC + 1 + 3 cols
    static constexpr int CR = 4, CB = ((TXB / 2 + 4 + 3) / 4) * 4, CROWS = S / 2 + 1;
    // every TMA destination starts 128-B aligned (sizes rounded up to 32 floats)
    static constexpr int al32(int n) { return (n + 31) & ~31; }
    // phase A: pixel (row s, region column rw) on thread s * PV + rw -- PV =
    // the image row pitch when S of them fit the CTA, so every
    // warp's shared accesses are one contiguous run (no bank conflicts where
    // a warp straddles two rows); else dense (PV = RW)
    static constexpr int PV = S * RXI <= NTH ? RXI : RW;
    // LSW (k = 7): the weights are evaluated where they are used, as
    // w_t = 2^(z_t log2 e - lse) from the logits (one TMA box per ring stage,
    // storage type, pitch RX) and the forward's base-2 log-sum-exp (one more
    // plane per step) -- phase A is G / inner only, no exponentials buffer.
    // k <= 5 keeps the softmax pass: phase A runs on all 8 warps there and
    // its in-place exponentials are read once by B1 and once by B2.
    // (Measured, same-box A/B: k7 bf16 level 0 -9%; k5 fp32 level 0 +19%.)
    static constexpr bool LSW = K >= 7 || (MODE & kBwdLsw) != 0;
    static constexpr bool TP = (MODE & kBwdTp) != 0;
    static constexpr bool SEP = !LSW && LGE != 4;  // bf16 softmax pass: separate fp32 exponentials
    // exponentials (softmax pass): fp32 logits = in place in the staging box
    // (pitch RX); bf16 = a separate fp32 buffer with a tighter pitch RXE over
    // the columns phase A fills, shifted by ESH (keeps 16-B alignment of quads)
    static constexpr int ESH = SEP ? RA - 4 : 0;
    static constexpr int RXE = SEP ? ((TXB + R + 4 + 3) / 4) * 4 : RX;
    static constexpr int EPL = S * RXE;                // floats per exponential plane
    static_assert(LSW || (ESH == DI && RXE == RXI), "exponential and image columns coincide");
    static constexpr int LGF = al32(NLOG * EPL);       // floats per exponentials buffer
    // logits staging box in the storage type: LSW and bf16 (fp32 softmax pass:
    // the exponential buffers themselves, in place)
    static constexpr int LGS1 = (LSW || SEP) ? al32((NLOG * S * RX * LGE + 3) / 4) : 0;
    static constexpr int LSF = LSW ? al32(S * RXI) : 0;  // log-sum-exp block (LSW)
    static constexpr int GDF = TP ? al32(3 * S * RXI) : 0;  // temporal pass: g_demod rows R behind
    static constexpr int DEMOFF = al32(3 * S * RXI);   // demod plane offset inside a ring block
    static constexpr int BLKF = NI * DEMOFF;           // floats per image-ring block
    static constexpr int UPF = al32(3 * S * RXI);      // floats per upstream / output block
    static constexpr int LHF = UP ? al32(3 * CROWS * CB) : 0;
    // coarse rows of the flushed fine rows (bottom step: the AW window rows from
    // qs - R; qs is even, so the first coarse row is aligned when R is even)
    static constexpr int CT = (R & 1) ? (S + 2 * R + 1) / 2 + 1 : (S + 2 * R) / 2;
    static constexpr int T1F = CH ? al32(3 * CT * CB) : 0;
    static constexpr bool B3ON = UP && !CH;
    // EARLY: the next step's TMA is issued at the top of the step (right after
    // the previous step's end barrier) instead of after phase A -- every
    // buffer it overwrites belongs to step i-1; needs a second output block,
    // and a second staging box for bf16 logits with the softmax pass
    // (measured no gain at k = 7 before LSW -- issued after phase A there)
    static constexpr bool EARLY = LSW || !SEP || NST > 2;
    static constexpr int NOB = EARLY ? NST : 1;
    static constexpr int LGS = EARLY ? NST * LGS1 : LGS1;  // staging floats (all boxes)
    static constexpr int LGBUF = LSW ? LGS : (SEP ? LGF + LGS : NST * LGF);
    // transaction bytes (exact box sizes, not the padded buffer sizes)
    static constexpr uint32_t TX_IMG = 3 * S * RXI * 4;
    static constexpr uint32_t TX_STEP = NLOG * S * RX * LGE + (NI + 2) * TX_IMG + (UP ? 3 * CROWS * CB * 4 : 0) +
                                        (CH ? 3 * CT * CB * 4 : 0) + (LSW ? S * RXI * 4 : 0) + (TP ? 3 * S * RXI * 4 : 0);
    static constexpr uint32_t TX_PRO = NPRO * NI * TX_IMG;
    static constexpr int NBU = L0 ? NBU0 : (EARLY ? 2 : 1);
    static constexpr int REDF = B2W ? al32(4 * (B2SPL - 1) * 3 * B2C) : 0;  // B2W partial rows
    // AHEAD: phase A of step i+1 runs at the end of step i (each warp after its
    // B work, before the end-of-step barrier, which then also publishes
    // G / inner of step i+1): one CTA barrier per step instead of two, and
    // phase A overlaps the B work of slower warps.  G / inner double-buffered;
    // needs the early-issued ring (every buffer phase A of step i+1 writes is
    // one step i does not read).  (Measured, same-box A/B: level 0 k5 -1.4%,
    // k7 -4.6%; k7 level 1 -6%; k5 levels >= 1, whose B1 warps also carry the
    // upsample transpose, +4.5% -- kept in order there.)
    // (and only where the second G / inner buffer keeps 2 CTAs per SM)
    static constexpr size_t FLOATS0 = (size_t)LGBUF + NBL * BLKF + (NBU + NOB) * UPF + NST * LHF + NST * T1F +
                                      NST * LSF + NST * GDF + (B3ON ? CR * 3 * TXC : 0) + REDF;
    static constexpr bool AHEAD = EARLY && (L0 || LSW) &&
                                  (SS != 4 || 2 * ((FLOATS0 + 8 * S * RXI) * 4 + 64 + 1024) <= 233472);
    static constexpr int NGB = AHEAD ? 2 : 1;

    static constexpr size_t FLOATS = FLOATS0 + NGB * 4 * S * RXI;
    static constexpr size_t SMEM = FLOATS * 4 + 64;
    // 2 CTAs per SM (16 warps) whenever two fit the 228 KB of shared memory
    static constexpr int MINB = (SS == 4 && 2 * (SMEM + 1024) <= 233472) ? 2 : 1;
    static_assert(NB1S <= B1ITEMS && NQUAD <= QS, "B1 pixel quads exceed warps 0-3");
    // the upsample-tap gradients follow the last part's tap rows (t = NT)
    static_assert(!UP || (B1SPL - 1) * DYS < K, "last B1 part must own the last tap row");
    static_assert(TXB * B2SPL <= HN && 3 * TXC <= HN && TXB % 4 == 0, "B2/B3 items exceed their warps");
    static_assert(S * PV <= NTH && RW <= 64, "phase A items exceed the CTA");
    static_assert((S == 4 || S == 8) && (32 % B2SPL) == 0 && NST >= 2 && NST <= 4 && TXB % RA == 0, "step geometry");
    static_assert(!(UP && !CH) || S == 4, "the B3 coarse-row ring (CR = 4) assumes 4-row steps");
    static_assert(SMEM + 1024 <= 233472 / MINB, "CTAs per SM");
};

// paired gradient store (two horizontally adjacent pixels, 8-B / 4-B aligned)
template <bool ACC>
__device__ __forceinline__ void st_gz2(float* p, float a, float b) {
    float2* q = reinterpret_cast<float2*>(p);
    if constexpr (ACC) {
        float2 o = *q;
        o.x += a;
        o.y += b;
        *q = o;
    } else {
        __stcs(q, make_float2(a, b));
    }
}
template <bool ACC>
__device__ __forceinline__ void st_gz2(__nv_bfloat16* p, float a, float b) {
    __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(p);
    if constexpr (ACC) {
        const float2 o = __bfloat1622float2(*q);
        a += o.x;
        b += o.y;
    }
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    __stcs(reinterpret_cast<unsigned*>(q), *reinterpret_cast<const unsigned*>(&v));
}

// quad gradient store (four horizontally adjacent pixels, 16-B / 8-B aligned)
template <bool ACC>
__device__ __forceinline__ void st_gz4(float* p, float a, float b, float c, float d) {
    float4* q = reinterpret_cast<float4*>(p);
    if constexpr (ACC) {
        float4 o = *q;
        o.x += a;
        o.y += b;
        o.z += c;
        o.w += d;
        *q = o;
    } else {
        __stcs(q, make_float4(a, b, c, d));
    }
}
template <bool ACC>
__device__ __forceinline__ void st_gz4(__nv_bfloat16* p, float a, float b, float c, float d) {
    uint2* q = reinterpret_cast<uint2*>(p);
    if constexpr (ACC) {
        const uint2 o = *q;
        const float2 o0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.x));
        const float2 o1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&o.y));
        a += o0.x;
        b += o0.y;
        c += o1.x;
        d += o1.y;
    }
    const __nv_bfloat162 v0 = __floats2bfloat162_rn(a, b), v1 = __floats2bfloat162_rn(c, d);
    __stcs(q, make_uint2(*reinterpret_cast<const unsigned*>(&v0), *reinterpret_cast<const unsigned*>(&v1)));
}

__device__ __forceinline__ float rcp_fast(float x) {  // MUFU.RCP (x >= 1e-3 here)
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <int NTH = 256>
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 0, %0;" ::"n"(NTH) : "memory"); }

#ifdef SSB_ROLE_TIMING
// experiment build only: per role (warps 0-3 / 4-7) cycles spent waiting for
// the step's TMA, in phase A (incl. its barrier), in the role's B work, and at
// the end-of-step barrier (tools/role_timing.py)
// (internal linkage: one copy per translation unit -- read through the
// per-k entry points in pyr_k{3,5,7}.cu)
static __device__ unsigned long long g_role_cycles[8];
static inline int role_cycles_read(unsigned long long* out8) {
    if (cudaMemcpyFromSymbol(out8, g_role_cycles, 8 * sizeof(unsigned long long)) != cudaSuccess) return -2;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_role_cycles, z, sizeof(z));
    return 0;
}
#define SSB_RT(...) __VA_ARGS__
#else
#define SSB_RT(...)
#endif

template <int K, typename TL, bool L0, bool UP, bool TIED, bool CH = false, int SS = 4, int NST = 2, int TXO = 0,
          int MODE = 0>
__global__ void __launch_bounds__((TmaShape<K, TL, L0, UP, TIED, CH, SS, NST, TXO, MODE>::NTH),
                                  (TmaShape<K, TL, L0, UP, TIED, CH, SS, NST, TXO, MODE>::MINB))
    k_pyr_bwd_tma(const BwdLevel a, const __grid_constant__ TmaMaps mp) {
    using SH = TmaShape<K, TL, L0, UP, TIED, CH, SS, NST, TXO, MODE>;
    constexpr int NTH = SH::NTH, HN = SH::HN;
    constexpr bool B3ON = SH::B3ON;
    constexpr int CT = SH::CT, T1F = SH::T1F;
    constexpr int R = SH::R, NT = SH::NT, NLOG = SH::NLOG, S = SH::S, RX = SH::RX, RXI = SH::RXI, DI = SH::DI;
    constexpr int RA = SH::RA, RW = SH::RW, NQUAD = SH::NQUAD;
    constexpr int TXB = SH::TXB, TXC = SH::TXC, NPRO = SH::NPRO, NBL = SH::NBL, NBU = SH::NBU;
    constexpr int NI = SH::NI, CR = SH::CR, CB = SH::CB, CROWS = SH::CROWS;
    constexpr int BLKF = SH::BLKF, UPF = SH::UPF, DEMOFF = SH::DEMOFF, LGS1 = SH::LGS1, LSF = SH::LSF;
    constexpr bool LSW = SH::LSW, SEP = SH::SEP;
    constexpr int LGF = SH::LGF, EPL = SH::EPL, RXE = SH::RXE, ESH = SH::ESH;
    constexpr int B1SPL = SH::B1SPL, B2SPL = SH::B2SPL, AW = SH::AW, NPW = SH::NPW;
    constexpr int PL = S * RXI;  // floats per image plane in a block
    constexpr int PLG = S * RX;  // logits per plane in the staging box
    constexpr int RUP = (R + 1) & ~1;

    extern __shared__ __align__(128) unsigned char smem_tma[];
    // LSW: [NST] logits boxes [NLOG][S][RX] (storage type); softmax pass:
    // [NST][NLOG][S][RX] in place (fp32) | [NLOG][S][RXE] + staging box(es)
    float* s_lg = reinterpret_cast<float*>(smem_tma);
    float* s_lin = s_lg + SH::LGBUF;                   // [NBL][NI][3][S][RXI]
    float* s_up = s_lin + NBL * BLKF;                  // [NBU][3][S][RXI] (level 0: u * out after A)
    float* s_ob = s_up + NBU * UPF;                    // [NOB][3][S][RXI] forward output / Lhat^l
    float* s_lhc = s_ob + SH::NOB * UPF;               // [NST][3][CROWS][CB]
    float* s_t1 = s_lhc + NST * SH::LHF;               // [NST][3][CT][CB]   (CH)
    float* s_lse = s_t1 + NST * T1F;                   // [NST][S][RXI] log-sum-exp (LSW)
    // [NGB][4][S][RXI] per step: G = gout (softmax pass: / sum), then
    // inner = sum_c gin_c out_c (/ sum)
    float* s_gd = s_lse + NST * LSF;                   // [NST][3][S][RXI] g_demod rows (TP)
    float* s_gi = s_gd + NST * SH::GDF;
    float* s_cac = s_gi + SH::NGB * 4 * PL;            // [CR][3][TXC] coarse ghat accumulators
    float* s_red = s_cac + (B3ON ? CR * 3 * TXC : 0);  // [4 (B2SPL-1)][3][B2C] B2W partial rows
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_tma + SH::FLOATS * 4);

    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int nc = a.nc, H = a.H, W = a.W, c0 = a.c0;
    const int x0 = blockIdx.x * TXB, xs0 = x0 - RA;   // xs0: global x of logit column 0
    const int xsi0 = xs0 + DI;                         // global x of image column 0
    const int cxs = (x0 >> 1) & ~3;                   // coarse box start (16-B aligned)
    const int y0 = blockIdx.y * a.seg_h, y1 = min(y0 + a.seg_h, H);
    const int qstart = max(y0 - RUP, 0);
    const int qend = min(y1 + R, H);
    const int nsteps = (qend - qstart + S - 1) / S;
    const unsigned hw32 = (unsigned)H * (unsigned)W;
    auto lin_block = [&](int j) { return s_lin + ((j + 64 * NBL) % NBL) * BLKF; };
    int sl_i = 0;  // ring slot of the current step's image block (i mod NBL), kept incrementally
    // image-ring row r for rows of the current step's window [qs - NPRO*S + R, qs + 2S + R)
    auto lin_row_step = [&](int qs, int r, int which) {
        const int rel = r - qs - R + NPRO * S;      // >= 0
        int slt = sl_i - NPRO + rel / S;
        slt += slt < 0 ? NBL : 0;
        slt -= slt >= NBL ? NBL : 0;
        return s_lin + slt * BLKF + which * DEMOFF + (rel % S) * RXI;
    };
    auto ring_block = [&](float* base, int j) { return base + ((j + 64 * NBU) % NBU) * UPF; };
    // image-ring row r (absolute) -> pointer to plane `which` (0: x0/L, 1: demod), channel 0
    auto lin_row = [&](int r, int which) {
        const int rel = r - qstart - R + NPRO * S;
        return lin_block(rel / S - NPRO) + which * DEMOFF + (rel % S) * RXI;
    };
    auto ring_row = [&](float* base, int r) {  // q row r -> upstream ring, channel 0
        const int rel = r - qstart + S;
        return ring_block(base, rel / S - 1) + (rel % S) * RXI;
    };

    // ---- TMA issue (thread 0)
    auto issue_step = [&](int j) {
        const int js = j % NST;
        uint64_t* bar = &bars[js];
        const int qs = qstart + j * S;
        mbar_expect_tx(bar, SH::TX_STEP - ((SH::TP && !a.gdc_out) ? 3 * S * RXI * 4 : 0));
        if constexpr (LSW) {
            tma_load_4d(s_lg + js * LGS1, &mp.lg, xs0, qs, a.lg_c0, b, bar);
            tma_load_4d(s_lse + js * LSF, &mp.lse, xsi0, qs, 0, b, bar);
            if constexpr (SH::TP)
                if (a.gdc_out) tma_load_4d(s_gd + js * SH::GDF, &mp.gd, xsi0, qs - R, c0, b, bar);
        } else {
            tma_load_4d(SEP ? s_lg + LGF + (SH::EARLY ? js * LGS1 : 0) : s_lg + js * LGF, &mp.lg, xs0, qs, 0, b, bar);
        }
        tma_load_4d(lin_block(j), &mp.lin, xsi0, qs + R, c0, b, bar);
        if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xsi0, qs + R, c0, b, bar);
        tma_load_4d(ring_block(s_up, j), &mp.up, xsi0, qs, c0, b, bar);
        tma_load_4d(s_ob + (SH::EARLY ? js * UPF : 0), &mp.out, xsi0, qs, c0, b, bar);
        if constexpr (UP) tma_load_4d(s_lhc + js * SH::LHF, &mp.lhc, cxs, qs >> 1, c0, b, bar);
        if constexpr (CH) tma_load_4d(s_t1 + js * T1F, &mp.t1, cxs, (qs - R) >> 1, c0, b, bar);
    };
    constexpr int PBAR = 7;  // prologue barrier (step barriers: 0 .. NST-1)

    // ---- clamp-to-edge patch of image-ring rows [r0, r1) (after conversion);
    // called by all threads with uniform arguments
    const bool col_border = xsi0 < 0 || xsi0 + RXI > W;
    auto patch_rows = [&](int r0, int r1) {
        if (col_border) {
            // only the columns outside the image: [0, lo) and [hi, RXI)
            const int lo = max(0, -xsi0), hi = min(RXI, W - xsi0), nb = lo + (RXI - hi);
            for (int i = tid; i < (r1 - r0) * NI * 3 * nb; i += NTH) {
                const int k = i % nb, rest = i / nb;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int ri = k < lo ? k : hi + (k - lo), src = k < lo ? lo : hi - 1;
                float* row = lin_row(r, pc / 3) + (pc % 3) * PL;
                row[ri] = row[src];
            }
            cta_sync<NTH>();
        }
        if (r0 < 0 || r1 > H) {
            for (int i = tid; i < (r1 - r0) * NI * 3 * RXI; i += NTH) {
                const int ri = i % RXI, rest = i / RXI;
                const int pc = rest % (NI * 3), r = r0 + rest / (NI * 3);
                const int src = clampi(r, 0, H - 1);
                if (src != r) lin_row(r, pc / 3)[(pc % 3) * PL + ri] = lin_row(src, pc / 3)[(pc % 3) * PL + ri];
            }
            cta_sync<NTH>();
        }
    };
    // x0 = noisy / max(d, floor) in place (level 0), for ring rows of block j
    // (ri: image column)
    auto convert_block = [&](int j, int s, int ri) {
        if constexpr (L0) {
            float* blk = lin_block(j);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float d = blk[DEMOFF + c * PL + s * RXI + ri];
                blk[c * PL + s * RXI + ri] *= rcp_fast(fmaxf(d, (float)kDemodFloor));
            }
        }
    };

    // ---- prologue
    if constexpr (B3ON)
        for (int i = tid; i < CR * 3 * TXC; i += NTH) s_cac[i] = 0.f;
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&bars[PBAR], SH::TX_PRO);
        for (int j = -NPRO; j < 0; ++j) {
            tma_load_4d(lin_block(j), &mp.lin, xsi0, qstart + R + j * S, c0, b, &bars[PBAR]);
            if constexpr (L0) tma_load_4d(lin_block(j) + DEMOFF, &mp.dem, xsi0, qstart + R + j * S, c0, b, &bars[PBAR]);
        }
        // the first steps: NST - 1 ahead when issuing early, else one
        for (int j = 0; j < (SH::EARLY ? NST - 1 : 1) && j < nsteps; ++j) issue_step(j);
    }
    mbar_wait(&bars[PBAR], 0);
    for (int i = tid; i < NPRO * S * RXI; i += NTH) {
        const int jj = i / (S * RXI), rem = i % (S * RXI);
        convert_block(jj - NPRO, rem / RXI, rem % RXI);
    }
    __syncthreads();
    patch_rows(qstart + R - NPRO * S, qstart + R);

    // phase A: pixel item p = tid = (row p / PV, region column p % PV) of the
    // S x RW region (pitch PV).  (Measured: handing the B1 warps, which finish
    // their B work first, a second phase-A pixel for 64 of their threads:
    // k5 level 0 +4.5%.)

    SSB_RT(long long rt_tw = 0; unsigned long long rt_acc[4] = {0, 0, 0, 0};)
    // ------------------------------------------------ A: [softmax,] G, inner
    // of step j (rows qs_j ..) into G / inner buffer gb.  LSW: no softmax --
    // B1 / B2 / B3 evaluate the normalised weights where they use them; else
    // the exponentials e land in lgb_j and G, inner carry 1 / sum.
    auto lgb_of = [&](int j) -> float* { return LSW ? nullptr : (SEP ? s_lg : s_lg + (j % NST) * LGF); };
    auto lgs_of = [&](int j) -> const TL* {
        return reinterpret_cast<const TL*>(
            LSW ? s_lg + (j % NST) * LGS1 : (SEP ? s_lg + LGF + (SH::EARLY ? (j % NST) * LGS1 : 0) : lgb_of(j)));
    };
    auto gbuf = [&](int j) { return s_gi + (SH::AHEAD ? (j & 1) * 4 * PL : 0); };
    auto phase_a_px = [&](int j, int qs_j, float* lgb_j, const TL* lgs_j, float* gb, int p) {
        const int s_a = p / SH::PV, rw_a = p - s_a * SH::PV;
        const int ri_a = RA - R + rw_a;  // logit column of the region pixel
        const int ii_a = ri_a - DI;      // its image / exponential column
        if (rw_a < RW) {
            float inv = 1.f;
            if constexpr (!LSW) {
                float e[NLOG];
#pragma unroll
                for (int t = 0; t < NLOG; ++t) e[t] = to_f32(lgs_j[t * PLG + s_a * RX + ri_a]);
                const float m = max4(e);
                const float2 mk2 = bcast2(-m * kLog2e);
                float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // 4 chains
#pragma unroll
                for (int t = 0; t + 1 < NLOG; t += 2) {
                    const float2 z2 = ffma2(make_float2(e[t], e[t + 1]), bcast2(kLog2e), mk2);
                    e[t] = ex2_ftz(z2.x);
                    e[t + 1] = ex2_ftz(z2.y);
                    sum2[(t >> 1) & 1] = fadd2(sum2[(t >> 1) & 1],
                                               make_float2((TIED && t == NT) ? 4.f * e[t] : e[t],
                                                           (TIED && t + 1 == NT) ? 4.f * e[t + 1] : e[t + 1]));
                }
                float sum = (sum2[0].x + sum2[1].x) + (sum2[0].y + sum2[1].y);
                if constexpr (NLOG & 1) {
                    e[NLOG - 1] = ex2_ftz(fmaf(e[NLOG - 1], kLog2e, mk2.x));
                    sum += (TIED && NLOG - 1 == NT) ? 4.f * e[NLOG - 1] : e[NLOG - 1];
                }
#pragma unroll
                for (int t = 0; t < NLOG; ++t) lgb_j[t * EPL + s_a * RXE + ii_a] = e[t];
                inv = rcp_fast(sum);
            }
            convert_block(j, s_a, ii_a);
            float* ub = ring_block(s_up, j) + s_a * RXI + ii_a;
            const float* ob = s_ob + (SH::EARLY ? (j % NST) * UPF : 0) + s_a * RXI + ii_a;
            float dq[3] = {1.f, 1.f, 1.f};
            if constexpr (L0) {
                const float* dr = lin_row(qs_j + s_a, 1) + ii_a;
#pragma unroll
                for (int c = 0; c < 3; ++c) dq[c] = fmaxf(dr[c * PL], (float)kDemodFloor);
            }
            float inner = 0.f;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float u = ub[c * PL], uo = u * ob[c * PL];
                inner += uo;
                gb[c * PL + s_a * RXI + ii_a] = LSW ? u * dq[c] : u * dq[c] * inv;
                if constexpr (L0) ub[c * PL] = uo;  // the flush's demod gradient needs u * out
            }
            gb[3 * PL + s_a * RXI + ii_a] = LSW ? inner : inner * inv;
        }
    };
    auto phase_a_body = [&](int j, int qs_j, float* lgb_j, const TL* lgs_j, float* gb) {
        if (tid < S * SH::PV) phase_a_px(j, qs_j, lgb_j, lgs_j, gb, tid);
    };
    // every thread passed step i-1's end barrier: the buffers of step i+NST-1
    // (those of step i-1) are free -- prefetch NST-1 steps ahead
    auto issue_ahead = [&](int i) {
        if (tid == 0 && i + NST - 1 < nsteps) {
            fence_proxy_async();
            issue_step(i + NST - 1);
        }
    };

    const bool want = a.want_params != 0;
    const bool acc_mode = a.accum != 0;

    // B1 / B3 role (warps 0-3)
    int cnext = qstart >> 1;
    const int part = B1SPL == 1 ? 0 : (tid % HN) / SH::B1ITEMS;
    const int item = (tid % HN) - part * SH::B1ITEMS;
    const int s = item / SH::QS, xi = 4 * (item % SH::QS), ri = xi + RA;
    const bool act_b1 = item < SH::NB1S && (item % SH::QS) < NQUAD;
    // B2 role (warps 4-7)
    const int b2 = tid % HN;
    const int col = SH::B2W ? ((b2 >> 5) % SH::WPP) * 32 + (b2 & 31) : b2 / B2SPL;
    const int part2 = SH::B2W ? (b2 >> 5) / SH::WPP : b2 - col * B2SPL;
    const int gx2 = x0 + col, ri2 = col + RA;
    const bool act2 = tid >= HN && col < TXB && gx2 < W;
    // the lanes of a column split the tap columns dx (window rows stay compile-time)
    constexpr int DXN = (K + B2SPL - 1) / B2SPL;
    const int dx0 = -R + part2 * DXN, ndx = min(DXN, R + 1 - dx0);
    float* const glo = (float*)a.gl_out + (long long)b * a.in_b;
    float* const gdo = (L0 && a.gdc_out) ? (float*)a.gdc_out + (long long)b * a.in_b : nullptr;
    // output rows qs - R + k, k in [0, AW), packed in pairs (2p, 2p+1) so
    // taps d, d+1 landing on one pair go as one FFMA2
    float2 win[NPW][3];
#pragma unroll
    for (int p = 0; p < NPW; ++p)
#pragma unroll
        for (int c = 0; c < 3; ++c) win[p][c] = make_float2(0.f, 0.f);
    auto wget = [&](int k, int c) { return (k & 1) ? win[k >> 1][c].y : win[k >> 1][c].x; };
    auto wadd = [&](int k, int c, float v) {
        if (k & 1) win[k >> 1][c].y += v;
        else win[k >> 1][c].x += v;
    };

    if constexpr (SH::AHEAD) {
        // phase A of step 0 (later steps: at the end of the step before)
        if (nsteps > 0) {
            mbar_wait(&bars[0], 0);
            phase_a_body(0, qstart, lgb_of(0), lgs_of(0), gbuf(0));
        }
        cta_sync<NTH>();
        if (nsteps > 0 && (col_border || qstart + R + S > H)) patch_rows(qstart + R, qstart + R + S);
    }
    int su_i = 0;  // upstream-ring slot of step i (i mod NBU), kept incrementally
    for (int i = 0; i < nsteps; ++i, sl_i = (sl_i + 1 == NBL) ? 0 : sl_i + 1, su_i = (su_i + 1 == NBU) ? 0 : su_i + 1) {
        const int qs = qstart + i * S;
        // LSW: the logits of this step and their log-sum-exp; softmax pass: the
        // exponentials of this step (lgb) and the logits' staging box
        float* lgb = lgb_of(i);
        const TL* lgs = lgs_of(i);
        const float* lsb = s_lse + (i % NST) * LSF;
        const float* s_g = gbuf(i);         // G of this step
        const float* s_inn = s_g + 3 * PL;  // inner of this step
        SSB_RT(long long rt_t0 = clock64(); long long rt_t1 = rt_t0;)
        if constexpr (SH::EARLY) issue_ahead(i);
        if constexpr (!SH::AHEAD) {
            mbar_wait(&bars[i % NST], (i / NST) & 1);
            SSB_RT(rt_tw = clock64();)
            phase_a_body(i, qs, lgb, lgs, gbuf(i));
            cta_sync<NTH>();
            if constexpr (!SH::EARLY) {
                // every thread has finished the previous step and this step's
                // phase A: the buffers of step i+1 are free
                if (tid == 0 && i + 1 < nsteps) {
                    fence_proxy_async();
                    issue_step(i + 1);
                }
            }
            if (col_border || qs + R + S > H) patch_rows(qs + R, qs + R + S);
            SSB_RT(rt_t1 = clock64(); rt_acc[0] += rt_tw - rt_t0; rt_acc[1] += rt_t1 - rt_tw;)
        }
        if (tid < HN) {
            // -------------------------------------------- B1: logit gradients
            const int qy = qs + s, gx = x0 + xi;
            // W is a multiple of 4 on this path: the quad (gx .. gx + 3) is in
            // the image and 16-B aligned in every gradient plane
            if (want && act_b1 && qy >= y0 && qy < y1 && gx < W) {
                float g[4][3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float4 gg = *reinterpret_cast<const float4*>(s_g + c * PL + s * RXI + ri - DI);
                    g[0][c] = gg.x;
                    g[1][c] = gg.y;
                    g[2][c] = gg.z;
                    g[3][c] = gg.w;
                }
                const float4 inn4 = *reinterpret_cast<const float4*>(s_inn + s * RXI + ri - DI);
                const float inn[4] = {inn4.x, inn4.y, inn4.z, inn4.w};
                // weights of the quad's taps: LSW w_t = 2^(z_t log2 e - lse); else
                // the exponentials of phase A (G, inner carry the 1 / sum)
                const TL* lq = lgs + s * RX + ri;
                float2 nl01 = make_float2(0.f, 0.f), nl23 = nl01;
                if constexpr (LSW) {
                    const float4 ls4 = lds128(lsb + s * RXI + ri - DI);
                    nl01 = make_float2(-ls4.x, -ls4.y);
                    nl23 = make_float2(-ls4.z, -ls4.w);
                }
                const float* ep = LSW ? nullptr : lgb + s * RXE + ri - ESH;
                auto wquad = [&](int t) {
                    if constexpr (LSW) {
                        const float4 z = ld_quad(lq + t * PLG);
                        const float2 p01 = ffma2(make_float2(z.x, z.y), bcast2(kLog2e), nl01);
                        const float2 p23 = ffma2(make_float2(z.z, z.w), bcast2(kLog2e), nl23);
                        return make_float4(ex2_ftz(p01.x), ex2_ftz(p01.y), ex2_ftz(p23.x), ex2_ftz(p23.y));
                    } else {
                        return *reinterpret_cast<const float4*>(
                            static_cast<const float*>(__builtin_assume_aligned(ep, 16)) + t * EPL);
                    }
                };
                auto body = [&](auto acc_t) {
                    constexpr bool ACC = decltype(acc_t)::value;
                    constexpr int OFF = 4 - R;  // window value m = x(ri - 4 + m); pixel p, tap d -> m = p + d + OFF
                    const int t_first = part * SH::DYS * K;
                    TL* gp = (TL*)a.glogits + (long long)b * a.lg_b + ((unsigned)qy * (unsigned)W + (unsigned)gx) +
                             (size_t)t_first * hw32;
                    auto tap_row = [&](int dy) {
                        const float* xr =
                            static_cast<const float*>(__builtin_assume_aligned(lin_row_step(qs, qy + dy, 0) + ri - DI - 4, 16));
                        // accumulators start at -inner': g_logit_t = e_t * (gw_t - inner')
                        float gw[4][K];
#pragma unroll
                        for (int p = 0; p < 4; ++p)
#pragma unroll
                            for (int d = 0; d < K; ++d) gw[p][d] = -inn[p];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            float2 vv[6];
#pragma unroll
                            for (int k2 = 0; k2 < 3; ++k2) {
                                const float4 t4 = lds128(xr + c * PL + 4 * k2);
                                vv[2 * k2] = make_float2(t4.x, t4.y);
                                vv[2 * k2 + 1] = make_float2(t4.z, t4.w);
                            }
                            auto V = [&](int m) { return (m & 1) ? vv[m >> 1].y : vv[m >> 1].x; };
                            // taps whose window value starts an aligned pair go two at a time
#pragma unroll
                            for (int p = 0; p < 4; ++p)
#pragma unroll
                                for (int d = 0; d < K; ++d) {
                                    const int m = p + d + OFF;
                                    if ((m & 1) == 0 && d + 1 < K) {
                                        const float2 r = ffma2(bcast2(g[p][c]), vv[m >> 1], make_float2(gw[p][d], gw[p][d + 1]));
                                        gw[p][d] = r.x;
                                        gw[p][d + 1] = r.y;
                                    } else if (!(d >= 1 && ((m - 1) & 1) == 0)) {
                                        gw[p][d] = fmaf(g[p][c], V(m), gw[p][d]);
                                    }
                                }
                        }
#pragma unroll
                        for (int d = 0; d < K; ++d) {
                            const int t = (dy + R) * K + d;
                            const float4 e4 = wquad(t);
                            st_gz4<ACC>(gp, e4.x * gw[0][d], e4.y * gw[1][d], e4.z * gw[2][d], e4.w * gw[3][d]);
                            gp += hw32;
                        }
                    };
                    {
                        const int dy_lo = -R + part * SH::DYS, dy_hi = min(dy_lo + SH::DYS, R + 1);
#pragma unroll 1
                        for (int dy = dy_lo; dy < dy_hi; ++dy) tap_row(dy);
                    }
                    if constexpr (UP) {
                        if (part == B1SPL - 1) {
                            // parents: pixel p takes column (gx + p + jj) / 2 (clamped): the
                            // quad reads coarse columns gx/2, gx/2 + 1, gx/2 + 2 (clamped)
                            const float* lh = s_lhc + (i % NST) * SH::LHF;
                            const int cyb = qs >> 1;
                            int Xc[3];
#pragma unroll
                            for (int k2 = 0; k2 < 3; ++k2) Xc[k2] = min((gx >> 1) + k2, a.Wc - 1) - cxs;
                            float gu[4][4];  // [pixel][tap 2ii + jj]
#pragma unroll
                            for (int ii = 0; ii < 2; ++ii) {
                                const int cy = min((qy + ii) >> 1, a.Hc - 1) - cyb;
                                float dotc[4][3];  // [pixel][parent column offset 0..2]
#pragma unroll
                                for (int p = 0; p < 4; ++p)
#pragma unroll
                                    for (int k2 = 0; k2 < 3; ++k2) dotc[p][k2] = -inn[p];
#pragma unroll
                                for (int c = 0; c < 3; ++c) {
                                    float lv[3];
#pragma unroll
                                    for (int k2 = 0; k2 < 3; ++k2) lv[k2] = lh[(c * CROWS + cy) * CB + Xc[k2]];
#pragma unroll
                                    for (int p = 0; p < 4; ++p)
#pragma unroll
                                        for (int jj = 0; jj < 2; ++jj) {
                                            const int k2 = (p + jj) >> 1;  // parent offset of (pixel p, tap jj)
                                            if (jj == 1 && ((p + 1) >> 1) == (p >> 1)) continue;  // same parent as jj = 0
                                            dotc[p][k2] = fmaf(g[p][c], lv[k2], dotc[p][k2]);
                                        }
                                }
#pragma unroll
                                for (int p = 0; p < 4; ++p)
#pragma unroll
                                    for (int jj = 0; jj < 2; ++jj) gu[p][2 * ii + jj] = dotc[p][(p + jj) >> 1];
                            }
                            if constexpr (TIED) {
                                const float4 e4 = wquad(NT);
                                float z[4];
#pragma unroll
                                for (int p = 0; p < 4; ++p) z[p] = (gu[p][0] + gu[p][1]) + (gu[p][2] + gu[p][3]);
                                st_gz4<ACC>(gp, e4.x * z[0], e4.y * z[1], e4.z * z[2], e4.w * z[3]);
                            } else {
#pragma unroll
                                for (int t4 = 0; t4 < 4; ++t4) {
                                    const float4 e4 = wquad(NT + t4);
                                    st_gz4<ACC>(gp, e4.x * gu[0][t4], e4.y * gu[1][t4], e4.z * gu[2][t4], e4.w * gu[3][t4]);
                                    gp += hw32;
                                }
                            }
                        }
                    }
                };
                if (acc_mode) body(std::true_type{});
                else body(std::false_type{});
            }

            // -------------------------------------------- B3: upsample transpose
            // item (coarse column X, channel c).  Coarse X receives fine columns
            // 2X-1 (tap j=1), 2X (j=0,1), 2X+1 (j=0; and j=1 at the last coarse
            // column, W even); coarse row (y+i)/2 per fine row y and tap row i,
            // clamped onto Hc-1 at the image bottom (fixed up below)
            if constexpr (B3ON) {
                if (tid < 3 * TXC) {
                    const int c = tid / TXC, cxi = tid - c * TXC;
                    const int X = (x0 >> 1) + cxi;
                    if (X < a.Wc) {
                        const int rj = 2 * cxi + RA;  // smem column of fine x = 2X
                        const bool lastX = X == a.Wc - 1;
                        float cv[CROWS + 1];
#pragma unroll
                        for (int k2 = 0; k2 <= CROWS; ++k2) cv[k2] = 0.f;
                        const int cyb = qs >> 1;  // qs is even
#pragma unroll
                        for (int ss = 0; ss < S; ++ss) {
                            const float* gr = s_g + c * PL + ss * RXI + rj - DI;
                            const float gm = gr[-1], g0 = gr[0], gq = gr[1];
#pragma unroll
                            for (int ii = 0; ii < 2; ++ii) {
                                float am, a0, aq;
                                if constexpr (LSW) {
                                    // log-sum-exp of fine columns 2X-1, 2X, 2X+1
                                    const float* lr = lsb + ss * RXI + rj - DI;
                                    const float nlm = -lr[-1], nl0 = -lr[0], nlq = -lr[1];
                                    const TL* z0 = lgs + (TIED ? NT : NT + 2 * ii) * PLG + ss * RX + rj;
                                    const TL* z1 = lgs + (TIED ? NT : NT + 2 * ii + 1) * PLG + ss * RX + rj;
                                    auto wt = [](TL z, float nl) { return ex2_ftz(fmaf(to_f32(z), kLog2e, nl)); };
                                    const float w0q = wt(z0[1], nlq);
                                    am = wt(z1[-1], nlm);
                                    a0 = wt(z0[0], nl0) + wt(z1[0], nl0);
                                    aq = lastX ? w0q + wt(z1[1], nlq) : w0q;
                                } else {
                                    const float* w0 = lgb + (TIED ? NT : NT + 2 * ii) * EPL + ss * RXE + rj - ESH;
                                    const float* w1 = lgb + (TIED ? NT : NT + 2 * ii + 1) * EPL + ss * RXE + rj - ESH;
                                    am = w1[-1];
                                    a0 = w0[0] + w1[0];
                                    aq = lastX ? w0[1] + w1[1] : w0[1];
                                }
                                const int yl = (ss + ii) >> 1;  // compile-time after unrolling
                                cv[yl] = fmaf(am, gm, fmaf(a0, g0, fmaf(aq, gq, cv[yl])));
                            }
                        }
                        // fine rows past the image contribute nothing (G = 0 there); the
                        // tap i = 1 of the last fine row of an even-height image points at
                        // coarse row Hc: clamp it onto Hc - 1
                        const int yc = a.Hc - cyb;  // local index of coarse row Hc
#pragma unroll
                        for (int k2 = 1; k2 <= CROWS; ++k2)
                            if (k2 == yc) {
                                cv[k2 - 1] += cv[k2];
                                cv[k2] = 0.f;
                            }
#pragma unroll
                        for (int k2 = 0; k2 < CROWS; ++k2) s_cac[(((cyb + k2) & (CR - 1)) * 3 + c) * TXC + cxi] += cv[k2];
                    }
                }
            }

        } else {
            // -------------------------------------------- B2: gather-transpose (warps 4-7)
            // taps of tap column dx for every source row of the step: window row
            // k = s + d (compile-time), smem column rj = ri - dx (runtime)
            auto gather_dx = [&](int rj, int dx) {
#pragma unroll
                for (int ss = 0; ss < S; ++ss) {
                    float g[3], w[K];
#pragma unroll
                    for (int c = 0; c < 3; ++c) g[c] = s_g[c * PL + ss * RXI + rj - DI];
                    if constexpr (LSW) {
                        const float nl = -lsb[ss * RXI + rj - DI];
#pragma unroll
                        for (int d = 0; d < K; ++d)
                            w[d] = ex2_ftz(fmaf(to_f32(lgs[(d * K + dx + R) * PLG + ss * RX + rj]), kLog2e, nl));
                    } else {
#pragma unroll
                        for (int d = 0; d < K; ++d) w[d] = lgb[(d * K + dx + R) * EPL + ss * RXE + rj - ESH];
                    }
#pragma unroll
                    for (int d = 0; d < K; ++d) {
                        const int k = ss + d;
                        if ((k & 1) == 0 && d + 1 < K) {
#pragma unroll
                            for (int c = 0; c < 3; ++c)
                                win[k >> 1][c] = ffma2(make_float2(w[d], w[d + 1]), bcast2(g[c]), win[k >> 1][c]);
                        } else if (!(d >= 1 && ((k - 1) & 1) == 0)) {
#pragma unroll
                            for (int c = 0; c < 3; ++c) wadd(k, c, w[d] * g[c]);
                        }
                    }
                }
            };
            if (act2) {
                // this lane's tap columns: [dx0, dx0 + ndx)
#pragma unroll
                for (int j = 0; j < DXN; ++j)
                    if (j < ndx) gather_dx(ri2 - (dx0 + j), dx0 + j);
                if (part2 == 0 && (gx2 == 0 || gx2 == W - 1)) {
                    // clamp fold along x: taps of in-image sources that land beyond
                    // the border column are gathered onto it (border columns only)
#pragma unroll 1
                    for (int e = 1; e <= R; ++e) {
                        const int Pc = gx2 == 0 ? -e : W - 1 + e;
#pragma unroll 1
                        for (int dx = -R; dx <= R; ++dx) {
                            const int qx = Pc - dx;
                            if (qx >= 0 && qx < W) gather_dx(qx - xs0, dx);
                        }
                    }
                }
            }

            // ---- finished output rows: image-border row folds, reduce over the
            // row groups (adjacent lanes), write
            const bool bottom = qs + S >= H;
            if (qs == 0) {
                // rows above the image fold onto row 0 (window row R)
#pragma unroll
                for (int k = 0; k < R; ++k)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        wadd(R, c, wget(k, c));
                        if (k & 1) win[k >> 1][c].y = 0.f;
                        else win[k >> 1][c].x = 0.f;
                    }
            }
            const int klast = H - 1 - (qs - R);  // window row of the image's last row
            if (bottom) {
                // rows below the image fold onto row H-1
#pragma unroll
                for (int k = 1; k < AW; ++k)
#pragma unroll
                    for (int kl = 0; kl < k; ++kl)
                        if (kl == klast)
#pragma unroll
                            for (int c = 0; c < 3; ++c) wadd(kl, c, wget(k, c));
            }
            // block of S window rows starting at compile-time kb: reduce-scatter
            // across the B2SPL lanes of the column, each lane writes S/B2SPL rows
            // window row J (compile-time) = image row qs - R + J: its image-ring
            // block / row and upstream-ring block / row are compile-time offsets
            // from this step's slots (no per-row division / modulo)
            auto lin_base_j = [&](auto j_t) -> const float* {
                constexpr int J = decltype(j_t)::value;
                constexpr int REL = J - 2 * R + NPRO * S;
                static_assert(REL >= 0, "window row above the image ring");
                int slt = sl_i + (REL / S - NPRO);
                slt += slt < 0 ? NBL : 0;
                slt -= slt >= NBL ? NBL : 0;
                return s_lin + slt * BLKF + (REL % S) * RXI + ri2 - DI;
            };
            auto up_base_j = [&](auto j_t) -> const float* {
                constexpr int J = decltype(j_t)::value;
                constexpr int RELU = J - R + S;
                static_assert(RELU >= 0, "window row above the upstream ring");
                int slt = su_i + (RELU / S - 1);
                slt += slt < 0 ? NBU : 0;
                slt -= slt >= NBU ? NBU : 0;
                return s_up + slt * UPF + (RELU % S) * RXI + ri2 - DI;
            };
            auto flush_block = [&](auto kb_t) {
                constexpr int KB = decltype(kb_t)::value;
                constexpr int PB = KB / 2;  // first pair (KB even)
                float2 keep[3];             // rows of this lane (pair or one component)
                int krow;                   // first window row this lane writes
                int nrow;                   // rows this lane writes (1 or 2 or 4)
                int rstep = 1;              // window-row stride between them
                float vout[4][3];
                if constexpr (SH::B2W) {
                    // partials of the rows other parts own -> shared memory; the
                    // owner (r % B2SPL == part) adds them to its own
                    if constexpr (KB > 0) asm volatile("bar.sync 1, %0;" ::"n"(HN) : "memory");  // (bottom blocks)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int own = r % B2SPL;
                        if (own != part2) {
                            const int sl = r * (B2SPL - 1) + (part2 < own ? part2 : part2 - 1);
#pragma unroll
                            for (int c = 0; c < 3; ++c) s_red[(sl * 3 + c) * SH::B2C + col] = wget(KB + r, c);
                        }
                    }
                    asm volatile("bar.sync 1, %0;" ::"n"(HN) : "memory");
                    constexpr int NOWN = 4 / B2SPL;
#pragma unroll
                    for (int m = 0; m < NOWN; ++m) {
                        const int r = part2 + B2SPL * m;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            // own partial of row r (compile-time window rows, selected)
                            float v;
                            if constexpr (B2SPL == 2) v = part2 ? wget(KB + 1 + 2 * m, c) : wget(KB + 2 * m, c);
                            else v = part2 == 0 ? wget(KB, c) : (part2 == 1 ? wget(KB + 1, c) : (part2 == 2 ? wget(KB + 2, c) : wget(KB + 3, c)));
#pragma unroll
                            for (int w = 0; w < B2SPL; ++w)
                                if (w != part2) v += s_red[((r * (B2SPL - 1) + (w < part2 ? w : w - 1)) * 3 + c) * SH::B2C + col];
                            vout[m][c] = v;
                        }
                    }
                    krow = KB + part2;
                    nrow = NOWN;
                    rstep = B2SPL;
                } else if constexpr (B2SPL == 1) {
#pragma unroll
                    for (int r = 0; r < 4; ++r)
#pragma unroll
                        for (int c = 0; c < 3; ++c) vout[r][c] = wget(KB + r, c);
                    krow = KB;
                    nrow = 4;
                } else if constexpr (B2SPL == 2) {
                    // the two lanes of a column split the block's rows even / odd
                    // (rows 0, 2 | 1, 3): the rows a lane pair then reads in the
                    // ring are 1 row (272 B = 16 banks) apart, not 2 (same banks)
                    const bool odd = (part2 & 1) != 0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float2 lo = PB < NPW ? win[PB][c] : make_float2(0.f, 0.f);
                        const float2 hi = PB + 1 < NPW ? win[PB + 1][c] : make_float2(0.f, 0.f);
                        const float2 send = odd ? make_float2(lo.x, hi.x) : make_float2(lo.y, hi.y);
                        float2 recv;
                        recv.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
                        recv.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
                        keep[c] = fadd2(odd ? make_float2(lo.y, hi.y) : make_float2(lo.x, hi.x), recv);
                        vout[0][c] = keep[c].x;
                        vout[1][c] = keep[c].y;
                    }
                    krow = KB + (odd ? 1 : 0);
                    nrow = 2;
                    rstep = 2;
                } else {
                    // round 1: halves (pairs PB, PB+1) between lanes part ^ (B2SPL/2)
                    const int hm = B2SPL / 2;
                    const bool upper = (part2 & hm) != 0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float2 lo = PB < NPW ? win[PB][c] : make_float2(0.f, 0.f);
                        const float2 hi = PB + 1 < NPW ? win[PB + 1][c] : make_float2(0.f, 0.f);
                        const float2 send = upper ? lo : hi;
                        float2 recv;
                        recv.x = __shfl_xor_sync(0xffffffffu, send.x, hm);
                        recv.y = __shfl_xor_sync(0xffffffffu, send.y, hm);
                        keep[c] = fadd2(upper ? hi : lo, recv);
                    }
                    {
                        // round 2: components between lanes part ^ 1
                        const bool odd = (part2 & 1) != 0;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const float send = odd ? keep[c].x : keep[c].y;
                            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                            vout[0][c] = (odd ? keep[c].y : keep[c].x) + recv;
                        }
                        krow = KB + (upper ? 2 : 0) + (odd ? 1 : 0);
                        nrow = 1;
                    }
                }
                if (!act2) return;
                // the block's 4 window rows KB .. KB+3: ring pointers (compile-time
                // offsets), selected per written row below
                const float* lb4[4] = {lin_base_j(std::integral_constant<int, KB>{}),
                                       lin_base_j(std::integral_constant<int, KB + 1>{}),
                                       lin_base_j(std::integral_constant<int, KB + 2>{}),
                                       lin_base_j(std::integral_constant<int, KB + 3>{})};
                const float* ub4[4] = {up_base_j(std::integral_constant<int, KB>{}),
                                       up_base_j(std::integral_constant<int, KB + 1>{}),
                                       up_base_j(std::integral_constant<int, KB + 2>{}),
                                       up_base_j(std::integral_constant<int, KB + 3>{})};
                auto sel4 = [](const float* const* a, int k) {
                    return k == 0 ? a[0] : (k == 1 ? a[1] : (k == 2 ? a[2] : a[3]));
                };
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r >= nrow) break;
                    const int P = qs - R + krow + r * rstep;
                    if (P < y0 || P >= y1 || P > H - 1) continue;
                    const unsigned off = (unsigned)P * (unsigned)W + (unsigned)gx2;
                    if constexpr (L0 && CH) {
                        // final outputs: the pool chain of the coarser levels,
                        // T1(parent) / (children of the parent), joins the
                        // level-0 input gradient; g_d masked by d > floor
                        // (pyramid.py:415-421, 436-447)
                        // (B2SPL = 4: one row per lane -- the generic row lookup is
                        // cheaper than selecting among the block's four)
                        const int kk = krow - KB + r * rstep;  // 0..3
                        const float* xr = B2SPL <= 2 ? sel4(lb4, kk) : lin_row_step(qs, P, 0) + ri2 - DI;
                        const float* dr = xr + DEMOFF;
                        const float* uor = B2SPL <= 2 ? sel4(ub4, kk) : ring_row(s_up, P) + ri2 - DI;  // u * out
                        const int Yp = P >> 1, Xp = gx2 >> 1;
                        const bool hy = 2 * Yp + 1 < H, hx = 2 * Xp + 1 < W;
                        const float rcnt = (hy && hx) ? 0.25f : ((hy || hx) ? 0.5f : 1.f);
                        // T1 row of parent Yp: window row J -> (J + (R & 1)) >> 1
                        const float* t1 = s_t1 + (i % NST) * T1F + ((KB + kk + (R & 1)) >> 1) * CB + (Xp - cxs);
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            if (c >= nc) break;
                            const unsigned o = c * hw32 + off;
                            const float d = dr[c * PL];
                            const float rd = rcp_fast(fmaxf(d, (float)kDemodFloor));
                            const float v = fmaf(t1[c * CT * CB], rcnt, vout[r][c]);
                            __stcs(glo + o, v * rd);
                            if (gdo) __stcs(gdo + o, d > (float)kDemodFloor ? (uor[c * PL] - v * xr[c * PL]) * rd : 0.f);
                        }
                    } else if constexpr (L0 && SH::TP) {
                        // temporal pass: g_prev = g(prev_in) / d; the history
                        // term of g_demod, -g(prev_in) prev_in / d, joins the
                        // (masked) value the level-0 kernel wrote (pyramid.py:436-447)
                        const int kk = krow - KB + r * rstep;
                        const float* xr = B2SPL <= 2 ? sel4(lb4, kk) : lin_row_step(qs, P, 0) + ri2 - DI;
                        const float* dr = xr + DEMOFF;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            if (c >= nc) break;
                            const unsigned o = c * hw32 + off;
                            const float d = dr[c * PL];
                            const float rd = rcp_fast(fmaxf(d, (float)kDemodFloor));
                            const float v = vout[r][c];
                            __stcs(glo + o, v * rd);
                            if (gdo && d > (float)kDemodFloor) {
                                // the step's box holds rows qs - R .. qs - R + S - 1 (KB = 0);
                                // the bottom step's further rows are read directly
                                const float g0 = KB == 0 ? s_gd[(i % NST) * SH::GDF + (c * S + kk) * RXI + ri2 - DI]
                                                         : gdo[o];
                                __stcs(gdo + o, g0 - v * xr[c * PL] * rd);
                            }
                        }
                    } else if constexpr (L0) {
                        const int kk = krow - KB + r * rstep;
                        const float* xr = B2SPL <= 2 ? sel4(lb4, kk) : lin_row_step(qs, P, 0) + ri2 - DI;
                        const float* dr = xr + DEMOFF;
                        const float* uor = B2SPL <= 2 ? sel4(ub4, kk) : ring_row(s_up, P) + ri2 - DI;  // u * out
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            if (c >= nc) break;
                            const unsigned o = c * hw32 + off;
                            if (a.demod) {
                                const float rd = rcp_fast(fmaxf(dr[c * PL], (float)kDemodFloor));
                                const float v = vout[r][c];
                                __stcs(glo + o, v * rd);
                                if (gdo) __stcs(gdo + o, (uor[c * PL] - v * xr[c * PL]) * rd);
                            } else {
                                __stcs(glo + o, vout[r][c]);
                            }
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            if (c < nc) glo[c * hw32 + off] = vout[r][c];
                    }
                }
            };
            // the step's S finished rows, four per block
            flush_block(std::integral_constant<int, 0>{});
            if constexpr (S > 4) flush_block(std::integral_constant<int, 4>{});
            if (bottom) {
                // the image's last rows: the whole window is final
                if constexpr (AW > S) flush_block(std::integral_constant<int, (AW > S ? S : 0)>{});
                if constexpr (AW > S + 4) flush_block(std::integral_constant<int, (AW > S + 4 ? S + 4 : 0)>{});
            }
            // slide the window by S rows
#pragma unroll
            for (int p = 0; p < NPW; ++p)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    win[p][c] = p + S / 2 < NPW ? win[p + S / 2][c] : make_float2(0.f, 0.f);
        }
        SSB_RT(const long long rt_t2 = clock64(); long long rt_t2b = rt_t2;)
        if constexpr (SH::AHEAD) {
            // phase A of the next step, as soon as this warp's B work is done
            if (i + 1 < nsteps) {
                mbar_wait(&bars[(i + 1) % NST], ((i + 1) / NST) & 1);
                SSB_RT(rt_tw = clock64(); rt_acc[0] += rt_tw - rt_t2;)
                phase_a_body(i + 1, qs + S, lgb_of(i + 1), lgs_of(i + 1), gbuf(i + 1));
                SSB_RT(rt_t2b = clock64(); rt_acc[1] += rt_t2b - rt_tw;)
            }
        }
        cta_sync<NTH>();  // end of step (AHEAD: G / inner of step i+1 published)
        SSB_RT(const long long rt_t3 = clock64(); rt_acc[2] += rt_t2 - rt_t1; rt_acc[3] += rt_t3 - rt_t2b;)
        if (B3ON && tid < HN) {
            // coarse ghat rows finished by this step (all B3 items are in)
            const bool bottom = qs + S >= H;
            const int cend = bottom ? a.Hc : (qs + S) >> 1;
            const int own0 = y0 >> 1, own1 = (y1 + 1) >> 1;
            for (int k2 = tid; k2 < (cend - cnext) * TXC; k2 += HN) {
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
        if constexpr (SH::AHEAD) {
            // the image rows that arrived with step i+1 (converted by its phase A)
            if (i + 1 < nsteps && (col_border || qs + S + R + S > H)) patch_rows(qs + S + R, qs + S + R + S);
        }
    }
#ifdef SSB_ROLE_TIMING
#ifndef SSB_ROLE_TIMING_L0
#define SSB_ROLE_TIMING_L0 -1  // -1: every level; 1: level 0 only; 0: levels >= 1 only
#endif
    if ((tid & 31) == 0 && (SSB_ROLE_TIMING_L0 < 0 || (SSB_ROLE_TIMING_L0 == 1) == L0))
        for (int k = 0; k < 4; ++k) atomicAdd(&g_role_cycles[(tid < HN ? 0 : 4) + k], rt_acc[k]);
#endif
}

}  // namespace ssb
