// Gather-pyramid filter kernels (forward, backward, pooling, final sweep).
//
// Reference semantics: pkg/src/sparse_sampler/pyramid.py (Appendix A of
// arXiv 2602.08642).  Design notes (DESIGN.md section "Kernels"):
//  * images planar (B, C, H, W); level-l logits planar (B, C_l, H_l, W_l);
//  * forward: one kernel per level, 2-D tile, per-pixel softmax in registers,
//    k x k gather from a clamp-padded shared-memory tile, upsample taps read
//    from the (L2-resident) coarse partial reconstruction;
//  * backward: one kernel per level that walks a column strip top->bottom in
//    steps of S rows.  Each step computes the softmax of S new rows (strip +
//    r halo columns) once, then (B1) the logit gradients of the strip's own
//    pixels, (B2) the gather-transpose into a ring of per-row accumulators
//    (clamp "fold" applied at the image border, pyramid.py:206-213) and
//    (B3) the upsample-transpose into a ring of coarse-row accumulators.
//    Finished rows are flushed to HBM.  No atomics: every accumulator cell is
//    owned by exactly one thread per phase.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ssb {

constexpr int kMaxCh = 3;  // channels per launch; larger C is split by the host

struct FwdLevel {
    int nc, H, W, Hc, Wc;
    int c0, ctot, batch, nlog, seg_h;  // channel group start, total channels, batch, logit channels
    const void* logits;
    long long lg_b;  // batch stride of logits (elements)
    const void* lin;  // L^l (l > 0) or noisy (l == 0)
    long long in_b, in_c;
    const void* demod;  // l == 0 only (same strides as lin); may be null
    const void* prev;   // l == 0 temporal history (same strides); may be null
    const void* lhat_c;  // coarse Lhat^{l+1}
    long long c_b, c_c;
    void* out;  // Lhat^l (l > 0) or out (l == 0); same strides as lin
    void* lse;  // l == 0, float32: per-pixel base-2 log-sum-exp of the logits (B, H, W); may be null
};

struct BwdLevel {
    int nc, H, W, Hc, Wc;
    int c0, ctot, batch, nlog;  // channel group start, total channels, batch, logit channels
    int seg_h;
    int want_params;
    int accum;
    const void* logits;
    long long lg_b;
    void* glogits;
    const void* lin;  // L^l or noisy
    long long in_b, in_c;
    const void* demod;
    const void* prev;
    const void* gin;   // ghat^l (l > 0) or upstream (l == 0)
    const void* outp;  // l == 0: forward output (for the demod gradient); may be null
    void* gl_out;      // l > 0: g of L^l via this level's gather; l == 0: partial g_noisy
    void* gdc_out;     // l == 0: partial gradient w.r.t. d; may be null
    void* gprev_out;   // l == 0 with history: g_prev (final)
    const void* lhat_c;
    long long c_b, c_c;
    void* ghat_c;  // coarse ghat^{l+1}
    const void* t1;  // level 0 after the coarse levels (CH): T1 = level-1 input gradient incl. the pool chain
    const float* lse;  // the forward's base-2 log-sum-exp of this level (TMA kernels), (B, H, W)
    int lg_c0;         // first logit channel the (TMA) kernel reads (temporal pass: K*K + 4)
};

// Load one pixel's logits in weight order (denoise, 4 upsample -- the tied
// blend logit broadcast --, temporal); `hw` is the per-frame channel stride
// (32-bit: one uniform multiply + one IMAD.WIDE per load).
template <typename T, int NT, int NUP, int NLUP, int NTM, typename TL>
__device__ __forceinline__ void load_softmax_logits(const TL* __restrict__ lp, unsigned hw, T* e) {
#pragma unroll
    for (int t = 0; t < NT; ++t) e[t] = ld_logit<T>(lp + t * hw);
    if constexpr (NUP > 0) {
        if constexpr (NLUP == 1) {
            const T v = ld_logit<T>(lp + NT * hw);
#pragma unroll
            for (int i = 0; i < 4; ++i) e[NT + i] = v;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) e[NT + i] = ld_logit<T>(lp + (NT + i) * hw);
        }
    }
#pragma unroll
    for (int t = 0; t < NTM; ++t) e[NT + NUP + t] = ld_logit<T>(lp + (NT + NLUP + t) * hw);
}

template <typename T, int NT, int NUP, int NLUP, int NTM, typename TL>
__device__ __forceinline__ void load_softmax_logits_off(const TL* __restrict__ fb, unsigned po,
                                                        unsigned hw, T* e) {
#pragma unroll
    for (int t = 0; t < NT; ++t) e[t] = ld_logit<T>(fb + (po + t * hw));
    if constexpr (NUP > 0) {
        if constexpr (NLUP == 1) {
            const T v = ld_logit<T>(fb + (po + NT * hw));
#pragma unroll
            for (int i = 0; i < 4; ++i) e[NT + i] = v;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) e[NT + i] = ld_logit<T>(fb + (po + (NT + i) * hw));
        }
    }
#pragma unroll
    for (int t = 0; t < NTM; ++t) e[NT + NUP + t] = ld_logit<T>(fb + (po + (NT + NLUP + t) * hw));
}

// ===========================================================================
// Forward level kernel
// ===========================================================================
constexpr int FWD_TX = 32, FWD_TY = 8;

template <int K, typename TL, typename T, bool L0, bool UP, bool TIED, bool PREV>
__global__ void __launch_bounds__(FWD_TX* FWD_TY)
    k_pyr_fwd(const FwdLevel a) {
    constexpr int R = K / 2, NT = K * K;
    constexpr int NUP = UP ? 4 : 0;
    constexpr int NLUP = UP ? (TIED ? 1 : 4) : 0;
    constexpr int NTM = PREV ? NT : 0;
    constexpr int NW = NT + NUP + NTM;
    constexpr int RXF = FWD_TX + 2 * R, RYF = FWD_TY + 2 * R;
    __shared__ T s_in[kMaxCh][RYF][RXF];
    __shared__ T s_pv[PREV ? kMaxCh : 1][PREV ? RYF : 1][PREV ? RXF : 1];

    const int b = blockIdx.z;
    const int x0 = blockIdx.x * FWD_TX, y0 = blockIdx.y * FWD_TY;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * FWD_TX + tx;
    const int nc = a.nc, H = a.H, W = a.W;

    const int x = x0 + tx, y = y0 + ty;
    const bool valid = (x < W) && (y < H);
    T e[NW];
    T sum = (T)0;
    if (valid) {  // logit loads first: they overlap the image staging below
        const unsigned hw = (unsigned)H * (unsigned)W;
        const TL* lfb = (const TL*)a.logits + b * a.lg_b;  // uniform per CTA
        load_softmax_logits_off<T, NT, NUP, NLUP, NTM>(lfb, (unsigned)y * (unsigned)W + (unsigned)x, hw, e);
    }
    const T* lin = (const T*)a.lin + b * a.in_b;
    const T* dem = (L0 && a.demod) ? (const T*)a.demod + b * a.in_b : nullptr;
    const T* prv = PREV ? (const T*)a.prev + b * a.in_b : nullptr;
    for (int i = tid; i < RYF * RXF; i += FWD_TX * FWD_TY) {
        const int ry = i / RXF, rx = i - ry * RXF;
        const int gy = clampi(y0 - R + ry, 0, H - 1), gx = clampi(x0 - R + rx, 0, W - 1);
        const long long off = (long long)gy * W + gx;
#pragma unroll
        for (int c = 0; c < kMaxCh; ++c) {
            if (c < nc) {
                T v = lin[c * a.in_c + off];
                T rd = (T)1;
                if (dem) {
                    rd = frcp(demod_clamp(dem[c * a.in_c + off]));
                    v = v * rd;
                }
                s_in[c][ry][rx] = v;
                if constexpr (PREV) {
                    T p = prv[c * a.in_c + off];
                    if (dem) p = p * rd;
                    s_pv[c][ry][rx] = p;
                }
            }
        }
    }

    T mk = (T)0;
    if (valid) {
        T m = e[0];
#pragma unroll
        for (int t = 1; t < NW; ++t) m = tmax(m, e[t]);
        mk = prep_max(m);
#pragma unroll
        for (int t = 0; t < NW; ++t) {
            e[t] = softmax_exp(e[t], mk);
            sum += e[t];
        }
    }
    __syncthreads();
    if (!valid) return;

    const T inv = frcp(sum);
    const long long off = (long long)y * W + x;
    if constexpr (std::is_same<T, float>::value) {
        // w_t = 2^(z_t log2 e - lse2): the TMA backward's weights
        if (a.lse) ((float*)a.lse)[(long long)b * H * W + off] = mk + __log2f(sum);
    }
    T* outp = (T*)a.out + b * a.in_b;
    const T* lhc = UP ? (const T*)a.lhat_c + b * a.c_b : nullptr;
    int cy0 = 0, cy1 = 0, cx0 = 0, cx1 = 0;
    if constexpr (UP) {
        cy0 = min(y >> 1, a.Hc - 1);
        cy1 = min((y + 1) >> 1, a.Hc - 1);
        cx0 = min(x >> 1, a.Wc - 1);
        cx1 = min((x + 1) >> 1, a.Wc - 1);
    }
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        if (c >= nc) break;
        T acc = (T)0;
#pragma unroll
        for (int dy = -R; dy <= R; ++dy)
#pragma unroll
            for (int dx = -R; dx <= R; ++dx)
                acc += e[(dy + R) * K + dx + R] * s_in[c][ty + R + dy][tx + R + dx];
        if constexpr (UP) {
            const T* cp = lhc + c * a.c_c;
            acc += e[NT + 0] * cp[cy0 * a.Wc + cx0];
            acc += e[NT + 1] * cp[cy0 * a.Wc + cx1];
            acc += e[NT + 2] * cp[cy1 * a.Wc + cx0];
            acc += e[NT + 3] * cp[cy1 * a.Wc + cx1];
        }
        if constexpr (PREV) {
#pragma unroll
            for (int dy = -R; dy <= R; ++dy)
#pragma unroll
                for (int dx = -R; dx <= R; ++dx)
                    acc += e[NT + NUP + (dy + R) * K + dx + R] * s_pv[c][ty + R + dy][tx + R + dx];
        }
        acc *= inv;
        if (L0 && dem) acc *= demod_clamp(dem[c * a.in_c + off]);
        outp[c * a.in_c + off] = acc;
    }
}

// ===========================================================================
// Backward level kernel (column-strip walker)
//
// CTA = one column strip of TXB own columns (+r halo columns = 64 region
// columns) and one segment of rows; it walks the segment in steps of S rows.
// Per step (q rows [qs, qs+S)):
//   A  every thread owns one region pixel: joint softmax of its logits ->
//      s_w, upstream gradient G -> s_g, next image-ring row -> s_lin;
//   B1 own pixels: weight gradients gw_t = sum_c G_c * L_c(q + o_t) (image
//      ring, compile-time tap offsets), upsample-tap gradients from the
//      coarse Lhat, softmax backward, logit gradients -> HBM;
//   B2 own columns, all S rows: horizontal transposed gather
//      h[dy] = sum_dx w_{dy,dx}(q_y, x-dx) G(q_y, x-dx), added into a
//      per-(row-in-step) accumulator ring at row q_y + dy (each thread owns
//      its ring column, so no races; the vertical clamp fold is applied at
//      flush, the horizontal one in the border columns);
//   B3 upsample transpose into per-row coarse accumulator rings;
//   flush rows whose contributions are complete (sum over the S rings).
// All arithmetic runs on 3 channels (missing channels are zero-filled), so
// the inner loops carry no channel guards.
// ===========================================================================
constexpr int BWD_THREADS = 256;
constexpr int BWD_RX = 64;  // region columns per strip (own columns + 2r halo)
constexpr int BWD_LR = 16;  // image ring rows (>= 2S + 2r)
constexpr int BWD_CR = 4;   // coarse accumulator ring rows (>= S/2 + 1)

template <int K, bool UP, bool PREV, typename T>
struct BwdShape {
    static constexpr int R = K / 2, NT = K * K;
    static constexpr int NUP = UP ? 4 : 0;
    static constexpr int NTM = PREV ? NT : 0;
    static constexpr int NW = NT + NUP + NTM;
    static constexpr int TXB = BWD_RX - 2 * R;
    static constexpr int TXC = TXB / 2;
    // accumulator rows live at once: S + 2r, plus -- while row 0 is not yet
    // flushed (until the first step with qs + S - r > 0) -- the r fold rows
    // above the image: r + (qs* + S + r) with qs* that first step's start row
    static constexpr int first_flush_qs(int S) { return R >= S ? S * ((R - S + 1 + S - 1) / S) : 0; }
    static constexpr int ar(int S) { return S + 2 * R + first_flush_qs(S); }
    static constexpr size_t bytes_for(int S) {
        return sizeof(T) * ((size_t)NW * S * BWD_RX + (size_t)kMaxCh * S * BWD_RX +
                            (size_t)kMaxCh * BWD_LR * BWD_RX * (PREV ? 2 : 1) +
                            (size_t)S * ar(S) * kMaxCh * TXB * (PREV ? 2 : 1) +
                            (size_t)S * BWD_CR * kMaxCh * TXC);
    }
    static constexpr int S = bytes_for(4) <= 200 * 1024 ? 4 : 2;
    static constexpr int AR = ar(S);
    static constexpr size_t SMEM = bytes_for(S);
    static constexpr int MINB_SMEM = (int)((227 * 1024) / (SMEM + 1024));
    static constexpr int MINB = MINB_SMEM > 3 ? 3 : (MINB_SMEM < 1 ? 1 : MINB_SMEM);
    static constexpr bool REG_GW = NW <= 56;
};

__device__ __forceinline__ float rcp_dem(float d) { return __fdividef(1.0f, d); }
__device__ __forceinline__ double rcp_dem(double d) { return 1.0 / d; }

template <int K, typename TL, typename T, bool L0, bool UP, bool TIED, bool PREV>
__global__ void __launch_bounds__(BWD_THREADS, (BwdShape<K, UP, PREV, T>::MINB))
    k_pyr_bwd(const BwdLevel a) {
    using SH = BwdShape<K, UP, PREV, T>;
    constexpr int R = SH::R, NT = SH::NT, NUP = SH::NUP, NW = SH::NW;
    constexpr int TXB = SH::TXB, TXC = SH::TXC, S = SH::S, AR = SH::AR;
    constexpr int RX = BWD_RX, CH = kMaxCh, CR = BWD_CR;
    constexpr int NLUP = UP ? (TIED ? 1 : 4) : 0;
    constexpr int RUP = (R + 1) & ~1;  // top halo rows, rounded up to even
    constexpr int LRM = BWD_LR - 1;
    constexpr int LSTR = BWD_LR * RX;  // channel stride of the image rings

    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* s_w = reinterpret_cast<T*>(smem_raw);               // [NW][S][RX]
    T* s_g = s_w + NW * S * RX;                            // [CH][S][RX]
    T* s_lin = s_g + CH * S * RX;                          // [CH][LR][RX]
    T* s_prv = s_lin + CH * LSTR;                          // [CH][LR][RX] (PREV)
    T* s_acc = s_prv + (PREV ? CH * LSTR : 0);             // [S][AR][CH][TXB]
    T* s_pac = s_acc + S * AR * CH * TXB;                  // [S][AR][CH][TXB] (PREV)
    T* s_cac = s_pac + (PREV ? S * AR * CH * TXB : 0);     // [S][CR][CH][TXC]
#define SW(t, s, ri) s_w[((t) * S + (s)) * RX + (ri)]
#define SG(c, s, ri) s_g[((c) * S + (s)) * RX + (ri)]
#define SLIN(c, r, ri) s_lin[(c) * LSTR + ((r) & LRM) * RX + (ri)]
#define SPRV(c, r, ri) s_prv[(c) * LSTR + ((r) & LRM) * RX + (ri)]
#define SACC(s, sl, c, xi) s_acc[(((s) * AR + (sl)) * CH + (c)) * TXB + (xi)]
#define SPAC(s, sl, c, xi) s_pac[(((s) * AR + (sl)) * CH + (c)) * TXB + (xi)]
#define SCAC(s, sl, c, xi) s_cac[(((s) * CR + (sl)) * CH + (c)) * TXC + (xi)]

    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int nc = a.nc, H = a.H, W = a.W;
    const int x0 = blockIdx.x * TXB, xr0 = x0 - R;
    const int y0 = blockIdx.y * a.seg_h, y1 = min(y0 + a.seg_h, H);
    const int qstart = max(y0 - RUP, 0);
    const int qend = min(y1 + R, H);
    const unsigned hw32 = (unsigned)H * (unsigned)W;
    auto slot = [](int P) { return (P + 8 * AR) % AR; };

    const TL* __restrict__ lg = (const TL*)a.logits + b * a.lg_b;
    TL* glg = a.want_params ? (TL*)a.glogits + b * a.lg_b : nullptr;
    const T* __restrict__ lin = (const T*)a.lin + b * a.in_b;
    const T* __restrict__ gin = (const T*)a.gin + b * a.in_b;
    const T* __restrict__ dem = (L0 && a.demod) ? (const T*)a.demod + b * a.in_b : nullptr;
    const T* __restrict__ prv = PREV ? (const T*)a.prev + b * a.in_b : nullptr;
    const T* __restrict__ lhc = UP ? (const T*)a.lhat_c + b * a.c_b : nullptr;

    // ---- prologue
    for (int i = tid; i < S * AR * CH * TXB; i += BWD_THREADS) {
        s_acc[i] = (T)0;
        if constexpr (PREV) s_pac[i] = (T)0;
    }
    for (int i = tid; i < S * CR * CH * TXC; i += BWD_THREADS) s_cac[i] = (T)0;

    auto load_image_row = [&](int r, int ri) {
        const int gy = clampi(r, 0, H - 1), gx = clampi(xr0 + ri, 0, W - 1);
        const long long off = (long long)gy * W + gx;
        T v[CH], p[CH], rd[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            v[c] = c < nc ? lin[c * a.in_c + off] : (T)0;
            rd[c] = (dem && c < nc) ? rcp_dem(demod_clamp(dem[c * a.in_c + off])) : (T)1;
            if constexpr (PREV) p[c] = c < nc ? prv[c * a.in_c + off] : (T)0;
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            SLIN(c, r, ri) = v[c] * rd[c];
            if constexpr (PREV) SPRV(c, r, ri) = p[c] * rd[c];
        }
    };
    for (int i = tid; i < 2 * R * RX; i += BWD_THREADS) {
        const int rr = i / RX, ri = i - rr * RX;
        load_image_row(qstart - R + rr, ri);
    }
    int next_flush = max(qstart - R, 0);
    int cnext = qstart >> 1;
    __syncthreads();

    for (int qs = qstart; qs < qend; qs += S) {
        // ------------------------------------------------ A: new rows
        if (tid < S * RX) {
            const int s = tid / RX, ri = tid - s * RX;
            const int qy = qs + s, qx = xr0 + ri;
            if ((qy < H) && (qx >= 0) && (qx < W)) {
                const long long off = (long long)qy * W + qx;
                const TL* lp = lg + off;
                if constexpr (SH::REG_GW) {
                    T e[NW];
                    load_softmax_logits<T, NT, NUP, NLUP, SH::NTM>(lp, hw32, e);
                    T m = e[0];
#pragma unroll
                    for (int t = 1; t < NW; ++t) m = tmax(m, e[t]);
                    const T mk = prep_max(m);
                    T sum = (T)0;
#pragma unroll
                    for (int t = 0; t < NW; ++t) {
                        e[t] = softmax_exp(e[t], mk);
                        sum += e[t];
                    }
                    const T inv = frcp(sum);
#pragma unroll
                    for (int t = 0; t < NW; ++t) SW(t, s, ri) = e[t] * inv;
                } else {
                    T m = (T)-INFINITY;
                    for (int t = 0; t < NW; ++t) {
                        int ch;
                        if (t < NT) ch = t;
                        else if (t < NT + NUP) ch = TIED ? NT : t;
                        else ch = t - NUP + NLUP;
                        const T v = ld_logit<T>(lp + ch * hw32);
                        SW(t, s, ri) = v;
                        m = tmax(m, v);
                    }
                    const T mk = prep_max(m);
                    T sum = (T)0;
                    for (int t = 0; t < NW; ++t) {
                        const T ev = softmax_exp(SW(t, s, ri), mk);
                        SW(t, s, ri) = ev;
                        sum += ev;
                    }
                    const T inv = frcp(sum);
                    for (int t = 0; t < NW; ++t) SW(t, s, ri) *= inv;
                }
                T g[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    g[c] = c < nc ? gin[c * a.in_c + off] : (T)0;
                    if (dem && c < nc) g[c] *= demod_clamp(dem[c * a.in_c + off]);
                }
#pragma unroll
                for (int c = 0; c < CH; ++c) SG(c, s, ri) = g[c];
            } else {
#pragma unroll 4
                for (int t = 0; t < NW; ++t) SW(t, s, ri) = (T)0;
#pragma unroll
                for (int c = 0; c < CH; ++c) SG(c, s, ri) = (T)0;
            }
            load_image_row(qs + R + s, ri);
        }
        __syncthreads();

        if (tid < S * TXB) {
            const int s = tid / TXB, xi = tid - s * TXB;
            const int qy = qs + s, gx = x0 + xi;
            const int ri = xi + R;
            // -------------------------------------------- B1: logit gradients
            if (glg && qy >= y0 && qy < y1 && gx < W) {
                T gv[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c) gv[c] = SG(c, s, ri);
                const T* lrow[K];
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) lrow[dy + R] = &SLIN(0, qy + dy, ri);
                auto gw_of = [&](int t) -> T {
                    T acc = (T)0;
                    if (t < NT) {
                        const int dy = t / K, dx = t % K - R;
#pragma unroll
                        for (int c = 0; c < CH; ++c) acc += gv[c] * lrow[dy][c * LSTR + dx];
                    } else if (t < NT + NUP) {
                        const int i = (t - NT) >> 1, j = (t - NT) & 1;
                        const int cy = min((qy + i) >> 1, a.Hc - 1), cx = min((gx + j) >> 1, a.Wc - 1);
                        const T* cp = lhc + (long long)cy * a.Wc + cx;
#pragma unroll
                        for (int c = 0; c < CH; ++c)
                            if (c < nc) acc += gv[c] * cp[c * a.c_c];
                    } else {
                        const int tt = t - NT - NUP;
                        const int dy = tt / K - R, dx = tt % K - R;
#pragma unroll
                        for (int c = 0; c < CH; ++c) acc += gv[c] * SPRV(c, qy + dy, ri + dx);
                    }
                    return acc;
                };
                TL* gp = glg + (long long)qy * W + gx;
                const bool acc_mode = a.accum != 0;
                if constexpr (SH::REG_GW) {
                    T gw[NW];
#pragma unroll
                    for (int t = 0; t < NW; ++t) gw[t] = gw_of(t);
                    T inner = (T)0;
#pragma unroll
                    for (int t = 0; t < NW; ++t) inner += SW(t, s, ri) * gw[t];
#pragma unroll
                    for (int t = 0; t < NW; ++t) gw[t] = SW(t, s, ri) * (gw[t] - inner);
                    if constexpr (TIED) gw[NT] = ((gw[NT] + gw[NT + 1]) + gw[NT + 2]) + gw[NT + 3];
                    // output channel of weight t (the tied blend logit takes the sum)
                    auto chan = [](int t) { return t < NT ? t : (t < NT + NUP ? NT + (TIED ? 0 : t - NT) : t - NUP + NLUP); };
                    auto skip = [](int t) { return TIED && t > NT && t < NT + NUP; };
                    if (acc_mode) {
#pragma unroll
                        for (int t = 0; t < NW; ++t)
                            if (!skip(t)) st_glogit(gp + chan(t) * hw32, gw[t], true);
                    } else {
#pragma unroll
                        for (int t = 0; t < NW; ++t)
                            if (!skip(t)) st_glogit(gp + chan(t) * hw32, gw[t], false);
                    }
                } else {
                    T inner = (T)0;
                    for (int t = 0; t < NW; ++t) inner += SW(t, s, ri) * gw_of(t);
                    T gb = (T)0;
                    for (int t = 0; t < NW; ++t) {
                        const T gz = SW(t, s, ri) * (gw_of(t) - inner);
                        if (TIED && t >= NT && t < NT + NUP) {
                            gb += gz;
                            if (t == NT + NUP - 1) st_glogit(gp + NT * hw32, gb, acc_mode);
                        } else {
                            const int ch = t < NT ? t : t - NUP + NLUP;
                            st_glogit(gp + ch * hw32, gz, acc_mode);
                        }
                    }
                }
            }
            // -------------------------------------------- B2: gather transpose
            if (qy < H && gx < W) {
                T h[K][CH], hp[PREV ? K : 1][CH];
#pragma unroll
                for (int d = 0; d < K; ++d)
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        h[d][c] = (T)0;
                        if constexpr (PREV) hp[d][c] = (T)0;
                    }
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                    const int rj = ri - dx;
                    T gq[CH];
#pragma unroll
                    for (int c = 0; c < CH; ++c) gq[c] = SG(c, s, rj);
#pragma unroll
                    for (int d = 0; d < K; ++d) {
                        const T wv = SW(d * K + dx + R, s, rj);
#pragma unroll
                        for (int c = 0; c < CH; ++c) h[d][c] += wv * gq[c];
                        if constexpr (PREV) {
                            const T pv = SW(NT + NUP + d * K + dx + R, s, rj);
#pragma unroll
                            for (int c = 0; c < CH; ++c) hp[d][c] += pv * gq[c];
                        }
                    }
                }
                if (gx == 0 || gx == W - 1) {
                    // clamp fold along x: logical columns beyond the border
                    for (int side = 0; side < 2; ++side) {
                        if ((side == 0 && gx != 0) || (side == 1 && gx != W - 1)) continue;
                        for (int e = 1; e <= R; ++e) {
                            const int Pc = side == 0 ? -e : W - 1 + e;
                            for (int dx = -R; dx <= R; ++dx) {
                                const int qx = Pc - dx;
                                if (qx < 0 || qx >= W) continue;
                                const int rj = qx - xr0;
                                for (int d = 0; d < K; ++d) {
                                    const T wv = SW(d * K + dx + R, s, rj);
#pragma unroll
                                    for (int c = 0; c < CH; ++c) h[d][c] += wv * SG(c, s, rj);
                                    if constexpr (PREV) {
                                        const T pv = SW(NT + NUP + d * K + dx + R, s, rj);
#pragma unroll
                                        for (int c = 0; c < CH; ++c) hp[d][c] += pv * SG(c, s, rj);
                                    }
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int d = 0; d < K; ++d) {
                    const int sl = slot(qy + d - R);
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        SACC(s, sl, c, xi) += h[d][c];
                        if constexpr (PREV) SPAC(s, sl, c, xi) += hp[d][c];
                    }
                }
            }
        }
        // ------------------------------------------------ B3: upsample transpose
        if constexpr (UP) {
            if (tid < S * TXC) {
                const int s = tid / TXC, cxi = tid - s * TXC;
                const int qy = qs + s, X = (x0 >> 1) + cxi;
                if (qy < H && X < a.Wc) {
                    T v0[CH], v1[CH];
#pragma unroll
                    for (int c = 0; c < CH; ++c) v0[c] = v1[c] = (T)0;
#pragma unroll
                    for (int k3 = -1; k3 <= 1; ++k3) {
                        const int xx = 2 * X + k3;
                        if (xx < 0 || xx >= W) continue;
                        const int rj = xx - xr0;
                        T gq[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) gq[c] = SG(c, s, rj);
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            if (min((xx + jj) >> 1, a.Wc - 1) != X) continue;
                            const T w0 = SW(NT + jj, s, rj), w1 = SW(NT + 2 + jj, s, rj);
#pragma unroll
                            for (int c = 0; c < CH; ++c) {
                                v0[c] += w0 * gq[c];
                                v1[c] += w1 * gq[c];
                            }
                        }
                    }
                    const int Y0 = min(qy >> 1, a.Hc - 1), Y1 = min((qy + 1) >> 1, a.Hc - 1);
#pragma unroll
                    for (int c = 0; c < CH; ++c) SCAC(s, Y0 & (CR - 1), c, cxi) += v0[c];
#pragma unroll
                    for (int c = 0; c < CH; ++c) SCAC(s, Y1 & (CR - 1), c, cxi) += v1[c];
                }
            }
        }
        __syncthreads();

        // ------------------------------------------------ flush finished rows
        const bool bottom = qs + S >= H;
        const int pend = max(bottom ? H : qs + S - R, next_flush);
        for (int i = tid; i < (pend - next_flush) * TXB; i += BWD_THREADS) {
            const int rr = i / TXB, xi = i - rr * TXB;
            const int P = next_flush + rr, gx = x0 + xi;
            T v[CH], pv[CH];
            auto take = [&](int row) {
                const int sl = slot(row);
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        v[c] += SACC(s, sl, c, xi);
                        SACC(s, sl, c, xi) = (T)0;
                        if constexpr (PREV) {
                            pv[c] += SPAC(s, sl, c, xi);
                            SPAC(s, sl, c, xi) = (T)0;
                        }
                    }
            };
#pragma unroll
            for (int c = 0; c < CH; ++c) v[c] = pv[c] = (T)0;
            take(P);
            if (P == 0)
                for (int e = 1; e <= R; ++e) take(-e);  // fold rows above the image
            if (P == H - 1)
                for (int e = 1; e <= R; ++e) take(H - 1 + e);  // and below it
            if (P < y0 || P >= y1 || gx >= W) continue;
            const long long off = (long long)P * W + gx;
            T* glo = (T*)a.gl_out + b * a.in_b;
            if constexpr (L0) {
                T* gdo = a.gdc_out ? (T*)a.gdc_out + b * a.in_b : nullptr;
                T* gpo = PREV ? (T*)a.gprev_out + b * a.in_b : nullptr;
                const T* up = (const T*)a.gin + b * a.in_b;
                const T* op = a.outp ? (const T*)a.outp + b * a.in_b : nullptr;
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    if (c >= nc) break;
                    const long long o = c * a.in_c + off;
                    if (dem) {
                        const T rd = rcp_dem(demod_clamp(dem[o]));
                        glo[o] = v[c] * rd;
                        if (gdo) {
                            const T x0v = SLIN(c, P, xi + R);
                            T gd = up[o] * (op[o] * rd) - v[c] * x0v * rd;
                            if constexpr (PREV) gd -= pv[c] * SPRV(c, P, xi + R) * rd;
                            gdo[o] = gd;
                        }
                        if constexpr (PREV) gpo[o] = pv[c] * rd;
                    } else {
                        glo[o] = v[c];
                        if constexpr (PREV) gpo[o] = pv[c];
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (c < nc) glo[c * a.in_c + off] = v[c];
            }
        }
        next_flush = pend;

        if constexpr (UP) {
            const int cend = bottom ? a.Hc : (qs + S) >> 1;
            const int own0 = y0 >> 1, own1 = (y1 + 1) >> 1;
            for (int i = tid; i < (cend - cnext) * TXC; i += BWD_THREADS) {
                const int rr = i / TXC, cxi = i - rr * TXC;
                const int Y = cnext + rr, X = (x0 >> 1) + cxi;
                T v[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c) v[c] = (T)0;
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int c = 0; c < CH; ++c) {
                        v[c] += SCAC(s, Y & (CR - 1), c, cxi);
                        SCAC(s, Y & (CR - 1), c, cxi) = (T)0;
                    }
                if (Y < own0 || Y >= own1 || X >= a.Wc) continue;
                T* gc = (T*)a.ghat_c + b * a.c_b + (long long)Y * a.Wc + X;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (c < nc) gc[c * a.c_c] = v[c];
            }
            cnext = cend;
        }
        if (bottom) break;
    }
#undef SW
#undef SG
#undef SLIN
#undef SPRV
#undef SACC
#undef SPAC
#undef SCAC
}

// ===========================================================================
// Pooling (level l -> l+1), count-correct 2x2 mean; level 0 demodulates first
// ===========================================================================
template <typename T>
__global__ void k_pool2(int nc, int H, int W, const T* __restrict__ in, long long in_b,
                        long long in_c, const T* __restrict__ dem, T* __restrict__ out,
                        long long out_b, long long out_c) {
    const int Hc = (H + 1) >> 1, Wc = (W + 1) >> 1;
    const int X = blockIdx.x * blockDim.x + threadIdx.x;
    const int Y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (X >= Wc || Y >= Hc) return;
    const int yb = 2 * Y, xb = 2 * X;
    const bool hy = yb + 1 < H, hx = xb + 1 < W;
    const T rcnt = (hy && hx) ? (T)0.25 : ((hy || hx) ? (T)0.5 : (T)1);  // exact 1/count
    const long long o00 = (long long)yb * W + xb;
    const long long o01 = hx ? o00 + 1 : o00, o10 = hy ? o00 + W : o00, o11 = hy ? o01 + W : o01;
    T v[kMaxCh][4];
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        if (c >= nc) break;
        const T* p = in + b * in_b + c * in_c;
        v[c][0] = p[o00];
        v[c][1] = p[o01];
        v[c][2] = p[o10];
        v[c][3] = p[o11];
        if (dem) {
            const T* d = dem + b * in_b + c * in_c;
            v[c][0] = fdiv(v[c][0], demod_clamp(d[o00]));
            v[c][1] = fdiv(v[c][1], demod_clamp(d[o01]));
            v[c][2] = fdiv(v[c][2], demod_clamp(d[o10]));
            v[c][3] = fdiv(v[c][3], demod_clamp(d[o11]));
        }
    }
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        if (c >= nc) break;
        // pyramid.py:144 sums the 2x2 block (zeros outside the image), then divides
        const T s01 = hx ? v[c][1] : (T)0, s10 = hy ? v[c][2] : (T)0;
        const T s11 = (hx && hy) ? v[c][3] : (T)0;
        out[b * out_b + c * out_c + (long long)Y * Wc + X] = ((v[c][0] + s01) + (s10 + s11)) * rcnt;
    }
}

// ===========================================================================
// Final coarse->fine sweep: g^{L-1} = gL_{L-1}; g^l = pool^T(g^{l+1}) + gL_l;
// then the level-0 combination with the partials written by the level-0
// backward kernel (pyramid.py:415-447).  One thread per level-0 pixel walks
// its ancestor chain, so the per-element arithmetic order equals the
// reference's level-by-level loop.
// ===========================================================================
struct FinalArgs {
    int nc, H, W, levels;
    int dims_h[SSB_MAX_LEVELS], dims_w[SSB_MAX_LEVELS];
    const void* gl[SSB_MAX_LEVELS];  // gL_l for l >= 1 (B, C, H_l, W_l), group-offset
    long long gl_b[SSB_MAX_LEVELS], gl_c[SSB_MAX_LEVELS];
    const void* noisy;
    const void* demod;
    long long in_b, in_c;
    void* g_noisy;  // in: partial, out: final
    void* g_demod;  // in: partial gdc, out: final (masked); may be null
};

template <typename T>
__global__ void k_pyr_final(const FinalArgs a) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (x >= a.W || y >= a.H) return;
    const long long off = (long long)y * a.W + x;
    // pool^T chain: identical for every channel except the gL values
    T pb[kMaxCh];
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) pb[c] = (T)0;
    if (a.levels > 1) {
        const int top = a.levels - 1;
        const long long ot = (long long)(y >> top) * a.dims_w[top] + (x >> top);
        const T* gt = (const T*)a.gl[top] + b * a.gl_b[top];
#pragma unroll
        for (int c = 0; c < kMaxCh; ++c)
            if (c < a.nc) pb[c] = gt[c * a.gl_c[top] + ot];
        for (int l = top - 1; l >= 0; --l) {
            // children count of the level-(l+1) ancestor, at level l
            const int Y = y >> (l + 1), X = x >> (l + 1);
            const bool hy = 2 * Y + 1 < a.dims_h[l], hx = 2 * X + 1 < a.dims_w[l];
            const T rcnt = (hy && hx) ? (T)0.25 : ((hy || hx) ? (T)0.5 : (T)1);
#pragma unroll
            for (int c = 0; c < kMaxCh; ++c) pb[c] = pb[c] * rcnt;  // power-of-two count: exact
            if (l == 0) break;
            const T* gl = (const T*)a.gl[l] + b * a.gl_b[l];
            const long long ol = (long long)(y >> l) * a.dims_w[l] + (x >> l);
#pragma unroll
            for (int c = 0; c < kMaxCh; ++c)
                if (c < a.nc) pb[c] = pb[c] + gl[c * a.gl_c[l] + ol];
        }
    }
    T* __restrict__ gn = (T*)a.g_noisy;
    T* __restrict__ gd = (T*)a.g_demod;
    const T* __restrict__ dm = (const T*)a.demod;
    const T* __restrict__ nz = (const T*)a.noisy;
    T vn[kMaxCh], vd[kMaxCh], vdem[kMaxCh], vx[kMaxCh];
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        if (c >= a.nc) break;
        const long long o = b * a.in_b + c * a.in_c + off;
        vn[c] = gn[o];
        if (dm) {
            vdem[c] = dm[o];
            if (gd) {
                vd[c] = gd[o];
                vx[c] = nz[o];
            }
        }
    }
#pragma unroll
    for (int c = 0; c < kMaxCh; ++c) {
        if (c >= a.nc) break;
        const long long o = b * a.in_b + c * a.in_c + off;
        if (dm) {
            const T rd = frcp(demod_clamp(vdem[c]));
            gn[o] = vn[c] + pb[c] * rd;
            if (gd) {
                const T x0 = vx[c] * rd;
                const T gdc = vd[c] - pb[c] * x0 * rd;
                gd[o] = vdem[c] > (T)kDemodFloor ? gdc : (T)0;
            }
        } else {
            gn[o] = vn[c] + pb[c];
        }
    }
}

}  // namespace ssb
