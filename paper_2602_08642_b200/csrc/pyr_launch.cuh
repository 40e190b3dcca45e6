// Host-side launch sequences for the pyramid filter (one instantiation per k).
#pragma once

#include <string>

#include <type_traits>

#include "pyr_bwd_tma.cuh"
#include "pyr_chain.cuh"
#include "pyr_fwd_tma.cuh"
#include "pyr_kernels.cuh"

namespace ssb {

void set_error(const std::string& msg);
int cuda_check(const char* where);

struct PyrPlan {
    int B, C, H, W, L, K;
    int hl[SSB_MAX_LEVELS], wl[SSB_MAX_LEVELS];
    int nlog[SSB_MAX_LEVELS];
    size_t esz;    // image element size
    size_t lgesz;  // logit element size
    // tape: pooled L^l and Lhat^l for l >= 1 (byte offsets)
    size_t pool_off[SSB_MAX_LEVELS], lhat_off[SSB_MAX_LEVELS], tape_bytes;
    // workspace: ghat^l and gL_l for l >= 1
    size_t ghat_off[SSB_MAX_LEVELS], gl_off[SSB_MAX_LEVELS], ws_bytes;
    // tape (float32 plans): per-level base-2 log-sum-exp of the softmax, B x h_l x w_l floats
    size_t lse_off[SSB_MAX_LEVELS];
};

int make_plan(const ssb_pyr_desc* d, PyrPlan* p);

inline long long lvl_elems(const PyrPlan& p, int l) { return (long long)p.hl[l] * p.wl[l]; }

inline int pick_segment(int strips, int H, int B);

template <typename TL>
constexpr CUtensorMapDataType tma_dtype() {
    return sizeof(TL) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
}

// TMA-pipelined level forward (fp32 images, fp32/bf16 logits, demodulated
// level 0, the temporal group on the one-pixel-per-thread path); returns
// false if the tensors are not TMA-addressable.
template <int K, typename TL, bool L0, bool UP, bool TIED, bool PREV = false>
bool launch_fwd_tma(const FwdLevel& a0, cudaStream_t s) {
    using SH = FwdTmaShape<K, TL, L0, UP, TIED, PREV>;
    if (L0 && !a0.demod) return false;
    if (PREV && (!a0.prev || K == 7)) return false;  // (k = 7: 102 weights per pixel exceed the registers)
    if (const char* e = getenv("SSB_NO_TMA")) {
        if (e[0] == '1') return false;
    }
    const long long plane = (long long)a0.H * a0.W;
    auto base = [&](const void* p, long long pl) {
        return p ? (const void*)((const float*)p - (long long)a0.c0 * pl) : nullptr;
    };
    FwdTmaMaps mp;
    const CUtensorMapDataType f32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    bool ok = make_tma_map_4d(&mp.lg, a0.logits, tma_dtype<TL>(), sizeof(TL), a0.W, a0.H, a0.nlog,
                              a0.batch, SH::TXF, SH::S, SH::NLOG) &&
              make_tma_map_4d(&mp.lin, base(a0.lin, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                              SH::RX, SH::S, 3);
    if (ok && L0)
        ok = make_tma_map_4d(&mp.dem, base(a0.demod, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                             SH::RX, SH::S, 3);
    if (ok && UP)
        ok = make_tma_map_4d(&mp.lhc, base(a0.lhat_c, (long long)a0.Hc * a0.Wc), f32, 4, a0.Wc,
                             a0.Hc, a0.ctot, a0.batch, SH::CB, SH::CROWS, 3);
    if (ok && PREV)
        ok = make_tma_map_4d(&mp.prv, base(a0.prev, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                             SH::RX, SH::S, 3);
    if (!ok) return false;
    auto kern = k_pyr_fwd_tma<K, TL, L0, UP, TIED, PREV>;
    static std::atomic<unsigned long long> attr_mask{0};
    smem_attr_once(attr_mask, (const void*)kern, (int)SH::SMEM);
    FwdLevel a = a0;
    const int strips = (a.W + SH::TXF - 1) / SH::TXF;
    a.seg_h = pick_segment(strips, a.H, a.batch);
    dim3 grid(strips, (a.H + a.seg_h - 1) / a.seg_h, a.batch);
    SSB_LAUNCH(s, kern<<<grid, SH::NTH, SH::SMEM, s>>>(a, mp));
    return true;
}

template <int K, typename TL, typename T, bool L0, bool UP, bool TIED, bool PREV>
void launch_fwd_one(const FwdLevel& a, int B, cudaStream_t s) {
    if constexpr (std::is_same<T, float>::value && !std::is_same<TL, double>::value) {
        if (launch_fwd_tma<K, TL, L0, UP, TIED, PREV>(a, s)) return;
    }
    dim3 block(FWD_TX, FWD_TY);
    dim3 grid((a.W + FWD_TX - 1) / FWD_TX, (a.H + FWD_TY - 1) / FWD_TY, B);
    SSB_LAUNCH(s, k_pyr_fwd<K, TL, T, L0, UP, TIED, PREV><<<grid, block, 0, s>>>(a));
}

inline int pick_segment(int strips, int H, int B) {
    // balanced row segments of <= SSB_SEG_ROWS (default 128) rows, a multiple
    // of 4, keeping >= ~8 CTAs per SM of work.  Measured (tools/seg_sweep.sh,
    // c4a): 48 -> 7719, 96 -> 7798, 128 -> 7886, 192 -> 7630, 256 -> 7250
    // Mpix/s -- longer walks amortise the prologue but spread the co-resident
    // CTAs over more rows of every logit plane.  SSB_MIN_CTAS (default 8 per
    // SM): c3 296 -> 4282, 592 -> 4371, 1184 -> 4413, 2368 -> 4342 Mpix/s
    static const int target = [] {
        const char* e = getenv("SSB_SEG_ROWS");
        const int v = e ? atoi(e) : 128;
        return v >= 16 ? v : 128;
    }();
    static const long long min_ctas = [] {
        const char* e = getenv("SSB_MIN_CTAS");
        const long long v = e ? atoll(e) : 148 * 8;
        return v >= 1 ? v : 148 * 8;
    }();
    // levels of < 4 Mpx (the coarse levels of one 4K frame, c2's frames):
    // SSB_MIN_CTAS_SMALL (experiment; default: the same target)
    static const long long min_small = [] {
        const char* e = getenv("SSB_MIN_CTAS_SMALL");
        const long long v = e ? atoll(e) : 0;
        return v >= 1 ? v : 0;
    }();
    const bool small = (long long)strips * 64 * H * B < (4ll << 20);
    const long long want = (small && min_small) ? min_small : min_ctas;
    int nseg = (H + target - 1) / target;
    while ((long long)strips * nseg * B < want && (H + nseg - 1) / nseg > 16) nseg *= 2;
    const int seg = (H + nseg - 1) / nseg;
    return (seg + 3) & ~3;
}

// TMA-pipelined level backward (fp32 images, fp32/bf16 logits, no temporal
// group, demodulated level 0); returns false if the tensors are not
// TMA-addressable.
inline bool tma_disabled() {
    const char* e = getenv("SSB_NO_TMA");
    return e && e[0] == '1';
}

template <int K, typename TL, bool L0, bool UP, bool TIED, bool CH = false, int SS = 4, int NST = 2, int TXO = 0,
          int MODE = 0>
bool prepare_bwd_tma(const BwdLevel& a0, TmaMaps& mp) {
    using SH = TmaShape<K, TL, L0, UP, TIED, CH, SS, NST, TXO, MODE>;
    // needs the forward output (level 0) / Lhat^l for the softmax-backward inner product
    if ((L0 && !a0.demod) || !a0.outp || (SH::LSW && !a0.lse) || tma_disabled()) return false;
    const long long plane = (long long)a0.H * a0.W;
    auto base = [&](const void* p, long long pl) {
        return p ? (const void*)((const float*)p - (long long)a0.c0 * pl) : nullptr;
    };
    const CUtensorMapDataType f32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    bool ok = make_tma_map_4d(&mp.lg, a0.logits, tma_dtype<TL>(), sizeof(TL), a0.W, a0.H, a0.nlog,
                              a0.batch, SH::RX, SH::S, SH::NLOG) &&
              make_tma_map_4d(&mp.lin, base(a0.lin, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                              SH::RXI, SH::S, 3) &&
              make_tma_map_4d(&mp.up, base(a0.gin, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                              SH::RXI, SH::S, 3);
    if (ok)
        ok = make_tma_map_4d(&mp.out, base(a0.outp, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                             SH::RXI, SH::S, 3);
    if (ok && L0)
        ok = make_tma_map_4d(&mp.dem, base(a0.demod, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                             SH::RXI, SH::S, 3);
    if (ok && UP)
        ok = make_tma_map_4d(&mp.lhc, base(a0.lhat_c, (long long)a0.Hc * a0.Wc), f32, 4, a0.Wc,
                             a0.Hc, a0.ctot, a0.batch, SH::CB, SH::CROWS, 3);
    if (ok && SH::LSW)  // the forward's log-sum-exp, (W, H, 1, B)
        ok = make_tma_map_4d(&mp.lse, a0.lse, f32, 4, a0.W, a0.H, 1, a0.batch, SH::RXI, SH::S, 1);
    if (ok && SH::TP && a0.gdc_out)  // temporal pass: g_demod as level 0 wrote it
        ok = make_tma_map_4d(&mp.gd, base(a0.gdc_out, plane), f32, 4, a0.W, a0.H, a0.ctot, a0.batch,
                                           SH::RXI, SH::S, 3);
    if (ok && CH)
        ok = a0.t1 && make_tma_map_4d(&mp.t1, base(a0.t1, (long long)a0.Hc * a0.Wc), f32, 4, a0.Wc, a0.Hc,
                                      a0.ctot, a0.batch, SH::CB, SH::CT, 3);
    return ok;
}

// strip width of the k = 5 fp32 backward per level width: the default 60
// own columns tile 1080p-family widths exactly; for others (c2's 256 / 128 /
// 64 / 32) the last strip can be mostly empty -- pick the width minimising
// strips x (own + 8 halo columns) among the instantiated 60 / 52 / 44 / 36
inline int pick_bwd_strip(int W) {
    static const bool off = [] {
        const char* e = getenv("SSB_BWD_STRIP60");
        return e && e[0] == '1';
    }();
    if (off) return 0;
    const int cand[4] = {60, 52, 44, 36};
    int best = 0;
    long long bc = 0;
    for (int t : cand) {
        const long long c = (long long)((W + t - 1) / t) * (t + 8);
        if (best == 0 || c < bc) {
            best = t;
            bc = c;
        }
    }
    return best == 60 ? 0 : best;
}

template <int K, typename TL, bool L0, bool UP, bool TIED, bool CH = false, int TXO = 0>
bool launch_bwd_tma(const BwdLevel& a0, cudaStream_t s) {
    using SH = TmaShape<K, TL, L0, UP, TIED, CH, 4, 2, TXO>;
    TmaMaps mp;
    if (!prepare_bwd_tma<K, TL, L0, UP, TIED, CH, 4, 2, TXO>(a0, mp)) return false;
    auto kern = k_pyr_bwd_tma<K, TL, L0, UP, TIED, CH, 4, 2, TXO>;
    static std::atomic<unsigned long long> attr_mask{0};
    smem_attr_once(attr_mask, (const void*)kern, (int)SH::SMEM);
    BwdLevel a = a0;
    const int strips = (a.W + SH::TXB - 1) / SH::TXB;
    a.seg_h = pick_segment(strips, a.H, a.batch);
    dim3 grid(strips, (a.H + a.seg_h - 1) / a.seg_h, a.batch);
    SSB_LAUNCH(s, kern<<<grid, 256, SH::SMEM, s>>>(a, mp));
    return true;
}

template <int K, typename TL, typename T, bool L0, bool UP, bool TIED, bool PREV>
void launch_bwd_one(const BwdLevel& a0, int B, cudaStream_t s) {
    if constexpr (std::is_same<T, float>::value && !std::is_same<TL, double>::value && !PREV) {
        if constexpr (K == 5 && std::is_same<TL, float>::value) {
            switch (pick_bwd_strip(a0.W)) {
                case 52: if (launch_bwd_tma<K, TL, L0, UP, TIED, false, 52>(a0, s)) return; break;
                case 44: if (launch_bwd_tma<K, TL, L0, UP, TIED, false, 44>(a0, s)) return; break;
                case 36: if (launch_bwd_tma<K, TL, L0, UP, TIED, false, 36>(a0, s)) return; break;
                default: break;
            }
        }
        if (launch_bwd_tma<K, TL, L0, UP, TIED>(a0, s)) return;
    }
    using SH = BwdShape<K, UP, PREV, T>;
    auto kern = k_pyr_bwd<K, TL, T, L0, UP, TIED, PREV>;
    static std::atomic<unsigned long long> attr_mask{0};
    smem_attr_once(attr_mask, (const void*)kern, (int)SH::SMEM);
    BwdLevel a = a0;
    const int strips = (a.W + SH::TXB - 1) / SH::TXB;
    a.seg_h = pick_segment(strips, a.H, B);
    dim3 grid(strips, (a.H + a.seg_h - 1) / a.seg_h, B);
    SSB_LAUNCH(s, kern<<<grid, BWD_THREADS, SH::SMEM, s>>>(a));
}

template <int K, typename TL, typename T>
void dispatch_fwd(const FwdLevel& a, int B, bool l0, bool up, bool tied, bool prev,
                  cudaStream_t s) {
    if (l0) {
        if (up) {
            if (tied) {
                if (prev) launch_fwd_one<K, TL, T, true, true, true, true>(a, B, s);
                else launch_fwd_one<K, TL, T, true, true, true, false>(a, B, s);
            } else {
                if (prev) launch_fwd_one<K, TL, T, true, true, false, true>(a, B, s);
                else launch_fwd_one<K, TL, T, true, true, false, false>(a, B, s);
            }
        } else {
            if (prev) launch_fwd_one<K, TL, T, true, false, false, true>(a, B, s);
            else launch_fwd_one<K, TL, T, true, false, false, false>(a, B, s);
        }
    } else if (up) {
        if (tied) launch_fwd_one<K, TL, T, false, true, true, false>(a, B, s);
        else launch_fwd_one<K, TL, T, false, true, false, false>(a, B, s);
    } else {
        launch_fwd_one<K, TL, T, false, false, false, false>(a, B, s);
    }
}

template <int K, typename TL, typename T>
void dispatch_bwd(const BwdLevel& a, int B, bool l0, bool up, bool tied, bool prev,
                  cudaStream_t s) {
    if (l0) {
        if (up) {
            if (tied) {
                if (prev) launch_bwd_one<K, TL, T, true, true, true, true>(a, B, s);
                else launch_bwd_one<K, TL, T, true, true, true, false>(a, B, s);
            } else {
                if (prev) launch_bwd_one<K, TL, T, true, true, false, true>(a, B, s);
                else launch_bwd_one<K, TL, T, true, true, false, false>(a, B, s);
            }
        } else {
            if (prev) launch_bwd_one<K, TL, T, true, false, false, true>(a, B, s);
            else launch_bwd_one<K, TL, T, true, false, false, false>(a, B, s);
        }
    } else if (up) {
        if (tied) launch_bwd_one<K, TL, T, false, true, true, false>(a, B, s);
        else launch_bwd_one<K, TL, T, false, true, false, false>(a, B, s);
    } else {
        launch_bwd_one<K, TL, T, false, false, false, false>(a, B, s);
    }
}

template <typename T>
void launch_pool(int B, int nc, int H, int W, const T* in, long long in_b, long long in_c,
                 const T* dem, T* out, long long out_b, long long out_c, cudaStream_t s) {
    const int Hc = (H + 1) >> 1, Wc = (W + 1) >> 1;
    dim3 block(32, 8);
    dim3 grid((Wc + 31) / 32, (Hc + 7) / 8, B);
    SSB_LAUNCH(s, k_pool2<T><<<grid, block, 0, s>>>(nc, H, W, in, in_b, in_c, dem, out, out_b, out_c));
}

// float32, 3 channels, no history, demodulated, >= 2 levels: the backward
// runs level 0 last (pyr_chain.cuh) from the forward's log-sum-exp
inline bool chain_path(const ssb_pyr_desc* d, const PyrPlan& p, const void* demod) {
    if (p.esz != 4 || p.C != 3 || !demod || p.L < 2 || tma_disabled()) return false;
    const char* e = getenv("SSB_NO_CHAIN");
    return !(e && e[0] == '1');
}

template <int K, typename TL, typename T>
int run_forward(const ssb_pyr_desc* d, const PyrPlan& p, const ssb_pyr_fwd_io* io, void* tape,
                cudaStream_t s) {
    char* tp = (char*)tape;
    const bool tied = d->blend_mode == SSB_BLEND_TIED;
    const long long img_b = (long long)p.C * p.H * p.W;
    for (int c0 = 0; c0 < p.C; c0 += kMaxCh) {
        const int nc = p.C - c0 < kMaxCh ? p.C - c0 : kMaxCh;
        const long long coff0 = (long long)c0 * p.H * p.W;
        const T* noisy = (const T*)io->noisy + coff0;
        const T* dem = io->demod ? (const T*)io->demod + coff0 : nullptr;
        // pooled pyramid of the demodulated input
        for (int l = 1; l < p.L; ++l) {
            const long long e_prev = lvl_elems(p, l - 1), e_l = lvl_elems(p, l);
            const T* src = l == 1 ? noisy
                                  : (const T*)(tp + p.pool_off[l - 1]) + (long long)c0 * e_prev;
            T* dst = (T*)(tp + p.pool_off[l]) + (long long)c0 * e_l;
            const long long sb = l == 1 ? img_b : (long long)p.C * e_prev;
            launch_pool<T>(p.B, nc, p.hl[l - 1], p.wl[l - 1], src, sb, e_prev,
                           l == 1 ? dem : nullptr, dst, (long long)p.C * e_l, e_l, s);
        }
        // coarse -> fine
        for (int l = p.L - 1; l >= 0; --l) {
            FwdLevel a{};
            a.nc = nc;
            a.H = p.hl[l];
            a.W = p.wl[l];
            a.c0 = c0;
            a.ctot = p.C;
            a.batch = p.B;
            a.nlog = p.nlog[l];
            const long long e_l = lvl_elems(p, l);
            a.logits = io->logits[l];
            a.lg_b = (long long)p.nlog[l] * e_l;
            a.in_b = (long long)p.C * e_l;
            a.in_c = e_l;
            if (l == 0) {
                a.lin = noisy;
                a.demod = dem;
                a.prev = io->prev ? (const T*)io->prev + coff0 : nullptr;
                a.out = (T*)io->out + coff0;
            } else {
                a.lin = (const T*)(tp + p.pool_off[l]) + (long long)c0 * e_l;
                a.out = (T*)(tp + p.lhat_off[l]) + (long long)c0 * e_l;
            }
            // the log-sum-exp is channel independent: written once (group 0);
            // read by k_up_transpose (level 0) and the k = 7 backward (LSW)
            a.lse = (p.esz == 4 && c0 == 0 && (l == 0 || K >= 7)) ? (void*)(tp + p.lse_off[l]) : nullptr;
            const bool up = l < p.L - 1;
            if (up) {
                const long long e_c = lvl_elems(p, l + 1);
                a.Hc = p.hl[l + 1];
                a.Wc = p.wl[l + 1];
                a.lhat_c = (const T*)(tp + p.lhat_off[l + 1]) + (long long)c0 * e_c;
                a.c_b = (long long)p.C * e_c;
                a.c_c = e_c;
            }
            dispatch_fwd<K, TL, T>(a, p.B, l == 0, up, tied, l == 0 && d->has_prev, s);
        }
    }
    return cuda_check("ssb_pyr_forward");
}

// level-b backward descriptor (channel group 0, C = 3) shared by both orders
template <typename T>
BwdLevel bwd_level(const ssb_pyr_desc* d, const PyrPlan& p, const ssb_pyr_bwd_io* io, const char* tp,
                   char* wp, int l, bool want, int accum) {
    BwdLevel a{};
    a.nc = p.C < kMaxCh ? p.C : kMaxCh;
    a.H = p.hl[l];
    a.W = p.wl[l];
    a.c0 = 0;
    a.ctot = p.C;
    a.batch = p.B;
    a.nlog = p.nlog[l];
    const long long e_l = lvl_elems(p, l);
    a.want_params = want ? 1 : 0;
    a.accum = accum;
    a.logits = io->logits[l];
    a.lg_b = (long long)p.nlog[l] * e_l;
    a.glogits = want ? io->g_logits[l] : nullptr;
    a.in_b = (long long)p.C * e_l;
    a.in_c = e_l;
    a.lse = p.esz == 4 ? (const float*)(tp + p.lse_off[l]) : nullptr;
    if (l == 0) {
        a.lin = io->noisy;
        a.demod = io->demod;
        a.gin = io->upstream;
        a.outp = io->out;
        a.gl_out = io->g_noisy;
        a.gdc_out = io->g_demod;
    } else {
        a.lin = tp + p.pool_off[l];
        a.outp = tp + p.lhat_off[l];
        a.gin = wp + p.ghat_off[l];
        a.gl_out = wp + p.gl_off[l];
    }
    if (l < p.L - 1) {
        const long long e_c = lvl_elems(p, l + 1);
        a.Hc = p.hl[l + 1];
        a.Wc = p.wl[l + 1];
        a.lhat_c = tp + p.lhat_off[l + 1];
        a.ghat_c = wp + p.ghat_off[l + 1];
        a.c_b = (long long)p.C * e_c;
        a.c_c = e_c;
    }
    return a;
}

// backward with level 0 LAST (pyr_chain.cuh): ghat^1 from the up-transpose
// pre-pass, levels 1..L-1, the level-1 pool chain, then level 0 writing the
// final g_noisy / g_demod (no coarse->fine sweep kernel).  Returns 1 without
// launching anything if level 0 is not TMA-addressable.
// SSB_BWD_S8=1 (experiment): the level-0 kernel with 8-row steps, 512 threads
inline bool bwd_s8() {  // read per call (tests switch it in-process, like SSB_NO_TMA)
    const char* e = getenv("SSB_BWD_S8");
    return e && e[0] == '1';
}

// MODE = kBwdLsw with history: level 0's denoise / upsample taps from the
// log-sum-exp of all its logits, then the temporal pass (kBwdTp)
template <int K, typename TL, bool TIED, int SS, int NST = 2, int TXO = 0, int MODE = 0>
int run_backward_chain_ss(const ssb_pyr_desc* d, const PyrPlan& p, const ssb_pyr_bwd_io* io, const void* tape,
                          void* ws, cudaStream_t s) {
    const char* tp = (const char*)tape;
    char* wp = (char*)ws;
    const bool want = io->g_logits[0] != nullptr;
    const int accum = io->accumulate_logits ? 1 : 0;
    BwdLevel a0 = bwd_level<float>(d, p, io, tp, wp, 0, want, accum);
    a0.t1 = wp + p.gl_off[1];
    TmaMaps mp0;
    if (!prepare_bwd_tma<K, TL, true, true, TIED, true, SS, NST, TXO, MODE>(a0, mp0)) return 1;
    // the temporal group (history): same level-0 walk over the warped
    // history with the temporal logits (channels K*K + 4 ..; + 1 tied)
    constexpr bool HIST = (MODE & kBwdLsw) != 0;
    BwdLevel at = a0;
    TmaMaps mpt;
    if constexpr (HIST) {
        if (!d->has_prev || !io->prev || !io->g_prev) return 1;
        at.lin = io->prev;
        at.gl_out = io->g_prev;
        at.t1 = nullptr;
        at.lg_c0 = K * K + (TIED ? 1 : 4);
        at.glogits = want ? (void*)((TL*)io->g_logits[0] + (long long)at.lg_c0 * p.H * p.W) : nullptr;
        if (!prepare_bwd_tma<K, TL, true, false, false, false, SS, NST, TXO, kBwdLsw | kBwdTp>(at, mpt)) return 1;
    }
    {
        UpTransposeArgs u{};
        u.H = p.H;
        u.W = p.W;
        u.Hc = p.hl[1];
        u.Wc = p.wl[1];
        u.nlog = p.nlog[0];
        u.logits = io->logits[0];
        u.lg_b = (long long)p.nlog[0] * lvl_elems(p, 0);
        u.lse = (const float*)(tp + p.lse_off[0]);
        u.up = (const float*)io->upstream;
        u.demod = (const float*)io->demod;
        u.ghat = (float*)(wp + p.ghat_off[1]);
        dim3 grid((u.Wc + UPT_X - 1) / UPT_X, (u.Hc + UPT_Y - 1) / UPT_Y, p.B);
        SSB_LAUNCH(s, (k_up_transpose<K * K, TIED, TL><<<grid, dim3(UPT_X, UPT_Y), 0, s>>>(u)));
    }
    for (int l = 1; l < p.L; ++l) {
        BwdLevel a = bwd_level<float>(d, p, io, tp, wp, l, want, accum);
        dispatch_bwd<K, TL, float>(a, p.B, false, l < p.L - 1, TIED, false, s);
    }
    if (p.L >= 3) {
        ChainArgs c{};
        c.levels = p.L;
        for (int l = 0; l < p.L; ++l) {
            c.dims_h[l] = p.hl[l];
            c.dims_w[l] = p.wl[l];
            c.gl[l] = l >= 1 ? (float*)(wp + p.gl_off[l]) : nullptr;
        }
        dim3 grid((p.wl[1] + 127) / 128, (p.hl[1] + 7) / 8, p.B);
        SSB_LAUNCH(s, k_pool_chain<<<grid, dim3(32, 8), 0, s>>>(c));
    }
    using SH = TmaShape<K, TL, true, true, TIED, true, SS, NST, TXO, MODE>;
    auto kern = k_pyr_bwd_tma<K, TL, true, true, TIED, true, SS, NST, TXO, MODE>;
    static std::atomic<unsigned long long> attr_mask{0};
    smem_attr_once(attr_mask, (const void*)kern, (int)SH::SMEM);
    const int strips = (a0.W + SH::TXB - 1) / SH::TXB;
    a0.seg_h = pick_segment(strips, a0.H, a0.batch);
    dim3 grid(strips, (a0.H + a0.seg_h - 1) / a0.seg_h, a0.batch);
    SSB_LAUNCH(s, kern<<<grid, SH::NTH, SH::SMEM, s>>>(a0, mp0));
    if constexpr (HIST) {
        // after level 0: its g_demod term joins the value level 0 wrote
        using SHT = TmaShape<K, TL, true, false, false, false, SS, NST, TXO, kBwdLsw | kBwdTp>;
        auto kt = k_pyr_bwd_tma<K, TL, true, false, false, false, SS, NST, TXO, kBwdLsw | kBwdTp>;
        static std::atomic<unsigned long long> attr_t{0};
        smem_attr_once(attr_t, (const void*)kt, (int)SHT::SMEM);
        const int st = (at.W + SHT::TXB - 1) / SHT::TXB;
        at.seg_h = pick_segment(st, at.H, at.batch);
        dim3 gt(st, (at.H + at.seg_h - 1) / at.seg_h, at.batch);
        SSB_LAUNCH(s, kt<<<gt, SHT::NTH, SHT::SMEM, s>>>(at, mpt));
    }
    return cuda_check("ssb_pyr_backward");
}

// SSB_BWD0=<stages>,<own columns> (experiment): level-0 kernel ring depth and
// strip width among the instantiated variants (0 = the default)
inline int bwd0_variant() {
    const char* e = getenv("SSB_BWD0");
    if (!e) return 0;
    int nst = 0, txo = 0;
    if (sscanf(e, "%d,%d", &nst, &txo) < 1) return 0;
    return nst * 1000 + txo;
}

template <int K, typename TL, bool TIED>
int run_backward_chain(const ssb_pyr_desc* d, const PyrPlan& p, const ssb_pyr_bwd_io* io, const void* tape,
                       void* ws, cudaStream_t s) {
    if (d->has_prev) return run_backward_chain_ss<K, TL, TIED, 4, 2, 0, kBwdLsw>(d, p, io, tape, ws, s);
    if constexpr (K == 5 && std::is_same<TL, float>::value) {
        if (bwd_s8()) return run_backward_chain_ss<K, TL, TIED, 8>(d, p, io, tape, ws, s);
#ifdef SSB_BWD_VARIANTS
        switch (bwd0_variant()) {
            // measured (r02, c4a bwd_l0 8.37 ms at 2,60): 3,40 10.31 ms; 3,32
            // / 2,32 / 4,32 ~10.4-13.4 ms -- narrower strips double the
            // barriers per pixel and the kernel is issue-bound, not ring-depth
            // bound (profiles/r02_variants.txt)
            case 3040: return run_backward_chain_ss<K, TL, TIED, 4, 3, 40>(d, p, io, tape, ws, s);
            default: break;
        }
#endif
        switch (pick_bwd_strip(p.W)) {
            case 52: return run_backward_chain_ss<K, TL, TIED, 4, 2, 52>(d, p, io, tape, ws, s);
            case 44: return run_backward_chain_ss<K, TL, TIED, 4, 2, 44>(d, p, io, tape, ws, s);
            case 36: return run_backward_chain_ss<K, TL, TIED, 4, 2, 36>(d, p, io, tape, ws, s);
            default: break;
        }
    }
    if constexpr (K == 7 && std::is_same<TL, __nv_bfloat16>::value) {
#ifdef SSB_BWD_VARIANTS
        switch (bwd0_variant()) {
            // measured (r02, c3 bwd_l0 0.880 ms at 2,32): 3,32 1.222 ms (1 CTA/SM), 3,24 1.475 ms
            case 3000: return run_backward_chain_ss<K, TL, TIED, 4, 3, 0>(d, p, io, tape, ws, s);
            default: break;
        }
#endif
    }
    return run_backward_chain_ss<K, TL, TIED, 4>(d, p, io, tape, ws, s);
}

template <int K, typename TL, typename T>
int run_backward(const ssb_pyr_desc* d, const PyrPlan& p, const ssb_pyr_bwd_io* io,
                 const void* tape, void* ws, cudaStream_t s) {
    const char* tp = (const char*)tape;
    char* wp = (char*)ws;
    const bool tied = d->blend_mode == SSB_BLEND_TIED;
    const bool want = io->g_logits[0] != nullptr;
    if constexpr (std::is_same<T, float>::value && !std::is_same<TL, double>::value) {
        if (chain_path(d, p, io->demod) && io->out) {
            const int rc = tied ? run_backward_chain<K, TL, true>(d, p, io, tape, ws, s)
                                : run_backward_chain<K, TL, false>(d, p, io, tape, ws, s);
            if (rc != 1) return rc;  // 1: not TMA-addressable, take the general order below
        }
    }
    for (int c0 = 0; c0 < p.C; c0 += kMaxCh) {
        const int nc = p.C - c0 < kMaxCh ? p.C - c0 : kMaxCh;
        const long long coff0 = (long long)c0 * p.H * p.W;
        const int accum = (io->accumulate_logits || c0 > 0) ? 1 : 0;
        for (int l = 0; l < p.L; ++l) {
            BwdLevel a{};
            a.nc = nc;
            a.H = p.hl[l];
            a.W = p.wl[l];
            a.c0 = c0;
            a.ctot = p.C;
            a.batch = p.B;
            a.nlog = p.nlog[l];
            const long long e_l = lvl_elems(p, l);
            a.want_params = want ? 1 : 0;
            a.accum = accum;
            a.logits = io->logits[l];
            a.lg_b = (long long)p.nlog[l] * e_l;
            a.glogits = want ? io->g_logits[l] : nullptr;
            a.in_b = (long long)p.C * e_l;
            a.in_c = e_l;
            a.lse = p.esz == 4 ? (const float*)(tp + p.lse_off[l]) : nullptr;
            if (l == 0) {
                a.lin = (const T*)io->noisy + coff0;
                a.demod = io->demod ? (const T*)io->demod + coff0 : nullptr;
                a.prev = io->prev ? (const T*)io->prev + coff0 : nullptr;
                a.gin = (const T*)io->upstream + coff0;
                a.outp = io->out ? (const T*)io->out + coff0 : nullptr;
                a.gl_out = (T*)io->g_noisy + coff0;
                a.gdc_out = (io->g_demod && io->demod) ? (T*)io->g_demod + coff0 : nullptr;
                a.gprev_out = io->g_prev ? (T*)io->g_prev + coff0 : nullptr;
            } else {
                a.lin = (const T*)(tp + p.pool_off[l]) + (long long)c0 * e_l;
                a.outp = (const T*)(tp + p.lhat_off[l]) + (long long)c0 * e_l;  // Lhat^l
                a.gin = (const T*)(wp + p.ghat_off[l]) + (long long)c0 * e_l;
                a.gl_out = (T*)(wp + p.gl_off[l]) + (long long)c0 * e_l;
            }
            const bool up = l < p.L - 1;
            if (up) {
                const long long e_c = lvl_elems(p, l + 1);
                a.Hc = p.hl[l + 1];
                a.Wc = p.wl[l + 1];
                a.lhat_c = (const T*)(tp + p.lhat_off[l + 1]) + (long long)c0 * e_c;
                a.ghat_c = (T*)(wp + p.ghat_off[l + 1]) + (long long)c0 * e_c;
                a.c_b = (long long)p.C * e_c;
                a.c_c = e_c;
            }
            dispatch_bwd<K, TL, T>(a, p.B, l == 0, up, tied, l == 0 && d->has_prev, s);
        }
        FinalArgs f{};
        f.nc = nc;
        f.H = p.H;
        f.W = p.W;
        f.levels = p.L;
        for (int l = 0; l < p.L; ++l) {
            f.dims_h[l] = p.hl[l];
            f.dims_w[l] = p.wl[l];
            if (l >= 1) {
                const long long e_l = lvl_elems(p, l);
                f.gl[l] = (const T*)(wp + p.gl_off[l]) + (long long)c0 * e_l;
                f.gl_b[l] = (long long)p.C * e_l;
                f.gl_c[l] = e_l;
            }
        }
        f.noisy = (const T*)io->noisy + coff0;
        f.demod = io->demod ? (const T*)io->demod + coff0 : nullptr;
        f.in_b = (long long)p.C * p.H * p.W;
        f.in_c = (long long)p.H * p.W;
        f.g_noisy = (T*)io->g_noisy + coff0;
        f.g_demod = (io->g_demod && io->demod) ? (T*)io->g_demod + coff0 : nullptr;
        dim3 block(32, 8);
        dim3 grid((p.W + 31) / 32, (p.H + 7) / 8, p.B);
        SSB_LAUNCH(s, k_pyr_final<T><<<grid, block, 0, s>>>(f));
    }
    return cuda_check("ssb_pyr_backward");
}

// one level on caller-laid-out buffers (row bands): the same dispatch as
// run_forward, per channel group
template <int K, typename TL, typename T>
int run_forward_level(const ssb_pyr_level_desc* d, const void* img, const void* demod, const void* logits,
                      const void* coarse, void* out, cudaStream_t s) {
    const bool tied = d->blend_mode == SSB_BLEND_TIED;
    const bool up = d->has_coarse != 0;
    const long long e_l = (long long)d->height * d->width;
    const long long e_c = up ? (long long)d->coarse_height * d->coarse_width : 0;
    const int nlog = K * K + (up ? (tied ? 1 : 4) : 0);
    for (int c0 = 0; c0 < d->channels; c0 += kMaxCh) {
        const int nc = d->channels - c0 < kMaxCh ? d->channels - c0 : kMaxCh;
        FwdLevel a{};
        a.nc = nc;
        a.H = d->height;
        a.W = d->width;
        a.c0 = c0;
        a.ctot = d->channels;
        a.batch = d->batch;
        a.nlog = nlog;
        a.logits = logits;
        a.lg_b = (long long)nlog * e_l;
        a.in_b = (long long)d->channels * e_l;
        a.in_c = e_l;
        a.lin = (const T*)img + (long long)c0 * e_l;
        a.demod = demod ? (const T*)demod + (long long)c0 * e_l : nullptr;
        a.out = (T*)out + (long long)c0 * e_l;
        if (up) {
            a.Hc = d->coarse_height;
            a.Wc = d->coarse_width;
            a.lhat_c = (const T*)coarse + (long long)c0 * e_c;
            a.c_b = (long long)d->channels * e_c;
            a.c_c = e_c;
        }
        dispatch_fwd<K, TL, T>(a, d->batch, demod != nullptr, up, tied, false, s);
    }
    return cuda_check("ssb_pyr_forward_level");
}

// declarations for the TUs that only call them (pyr_api.cu): no implicit
// instantiation there -- each (k, logit dtype) is compiled once, in its own TU
#define SSB_EXTERN_PYR(K, TL, T)                                                           \
    extern template int run_forward<K, TL, T>(const ssb_pyr_desc*, const PyrPlan&,         \
                                              const ssb_pyr_fwd_io*, void*, cudaStream_t); \
    extern template int run_backward<K, TL, T>(const ssb_pyr_desc*, const PyrPlan&,        \
                                               const ssb_pyr_bwd_io*, const void*, void*, cudaStream_t); \
    extern template int run_forward_level<K, TL, T>(const ssb_pyr_level_desc*, const void*, const void*, \
                                                    const void*, const void*, void*, cudaStream_t);

#define SSB_INSTANTIATE_PYR(K, TL, T)                                                       \
    template int run_forward<K, TL, T>(const ssb_pyr_desc*, const PyrPlan&,                 \
                                       const ssb_pyr_fwd_io*, void*, cudaStream_t);         \
    template int run_backward<K, TL, T>(const ssb_pyr_desc*, const PyrPlan&,                \
                                        const ssb_pyr_bwd_io*, const void*, void*, cudaStream_t); \
    template int run_forward_level<K, TL, T>(const ssb_pyr_level_desc*, const void*, const void*,  \
                                             const void*, const void*, void*, cudaStream_t);

}  // namespace ssb
