/*
 * ssb_api.h -- C ABI of libssb200.so, the B200 (sm_100a) hot path of the
 * sparse-sampler pipeline (arXiv 2602.08642).
 *
 * The reference (`/root/reference/pkg/src/sparse_sampler`) is pure Python; its
 * "plugin interface" for this path is a set of module-level numpy functions.
 * Each entry point below names the reference function(s) it replaces
 * (file:line).  The Python host mirror lives in paper_2602_08642_b200/ (ops.py
 * for torch tensors, compat/ for the reference's exact numpy signatures);
 * INTEGRATION.md shows the ctypes binding.
 *
 * Conventions
 *  - Caller owns all device memory: the library never allocates or frees, so
 *    every call is CUDA-graph capturable.  Workspace sizes come from the
 *    *_bytes queries.
 *  - Every call launches only on `stream` and never synchronises the host.
 *  - Return value: SSB_OK or a negative SSB_E* code; ssb_last_error() returns
 *    a thread-local message for the last failure.  No C++ exception crosses
 *    the boundary.
 *  - Images are planar, contiguous (B, C, H, W); level-l logits are
 *    (B, C_l, H_l, W_l) with H_l = ceil(H / 2^l).  Scalars are host values.
 */
#ifndef SSB_API_H
#define SSB_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ssb_stream_t; /* == cudaStream_t */

#define SSB_VERSION 1
#define SSB_MAX_LEVELS 8

enum { SSB_OK = 0, SSB_EINVAL = -1, SSB_ECUDA = -2, SSB_EUNSUPPORTED = -3 };
enum { SSB_F32 = 0, SSB_BF16 = 1, SSB_F64 = 2 };
enum { SSB_BLEND_NATIVE = 0, SSB_BLEND_TIED = 1 };

int ssb_version(void);
const char* ssb_last_error(void);

/* Measurement hooks (bench/profiling only; not needed for computation).
 * ssb_launch_count: kernels launched by this process so far.
 * ssb_set_launch_events: while `events` is non-NULL, the i-th kernel this
 * thread launches is bracketed by cudaEventRecord(events[2i]) and
 * cudaEventRecord(events[2i+1]) on its stream, for i < capacity; *count
 * receives the number bracketed.  Pass NULL to disable. */
unsigned long long ssb_launch_count(void);
int ssb_set_launch_events(void* const* events, int capacity, int* count);

/* ------------------------------------------------------------------------
 * (c) gather pyramid filter -- replaces pyramid.py `reconstruct_core`
 * (:292-345), `reconstruct` (:348-359) and `reconstruct_backward` (:362-449),
 * generalised to odd k in {3,5,7} and 1 <= L <= SSB_MAX_LEVELS.
 *
 * Level-l logit channels (ssb_pyr_logit_channels): k*k denoise taps
 * (dy-major), then the upsample group if l < L-1 (4 logits native, 1 logit
 * tied), then k*k temporal taps at l = 0 iff has_prev.  The reference layout
 * always carries the temporal group at level 0 (pyramid.py:41-43); with no
 * history it is unread, so the device layout omits it.
 * ---------------------------------------------------------------------- */
typedef struct ssb_pyr_desc {
    int32_t batch, channels, height, width; /* channels: any C >= 1 */
    int32_t levels, ksize;
    int32_t image_dtype; /* SSB_F32 | SSB_F64: noisy/demod/prev/out/upstream/grads */
    int32_t logit_dtype; /* SSB_F32 | SSB_BF16 (with F32 images) | SSB_F64 (with F64 images) */
    int32_t has_prev;    /* temporal group at level 0 */
    int32_t has_demod;   /* demodulation by max(d, 1e-3) */
    int32_t blend_mode;  /* SSB_BLEND_NATIVE | SSB_BLEND_TIED */
    int32_t reserved;
} ssb_pyr_desc;

typedef struct ssb_pyr_fwd_io {
    const void* noisy; /* (B,C,H,W) */
    const void* demod; /* (B,C,H,W), or NULL iff !has_demod */
    const void* prev;  /* (B,C,H,W) warped history, or NULL iff !has_prev */
    const void* logits[SSB_MAX_LEVELS];
    void* out; /* (B,C,H,W) remodulated output (not clamped, like reconstruct_core) */
} ssb_pyr_fwd_io;

typedef struct ssb_pyr_bwd_io {
    const void* noisy;
    const void* demod;
    const void* prev;
    const void* logits[SSB_MAX_LEVELS];
    const void* out;      /* forward output (the tape's out_pre = out / max(d,1e-3)) */
    const void* upstream; /* (B,C,H,W) */
    void* g_logits[SSB_MAX_LEVELS]; /* all NULL => want_param_grads = False */
    void* g_noisy;                  /* required */
    void* g_demod;                  /* w.r.t. d (g_theta = g_d * d); NULL to skip */
    void* g_prev;                   /* required iff has_prev */
    int32_t accumulate_logits;      /* 1: g_logits += (for callers summing frames) */
    int32_t reserved;
} ssb_pyr_bwd_io;

int ssb_pyr_logit_channels(const ssb_pyr_desc* d, int level);
int ssb_pyr_level_dims(const ssb_pyr_desc* d, int level, int32_t* h, int32_t* w);
/* tape = pooled levels L^1..L^{L-1} and partial reconstructions Lhat^1..Lhat^{L-1} */
int ssb_pyr_tape_bytes(const ssb_pyr_desc* d, size_t* bytes);
/* backward scratch: per-level gradients for l >= 1 */
int ssb_pyr_workspace_bytes(const ssb_pyr_desc* d, size_t* bytes);
int ssb_pyr_forward(const ssb_pyr_desc* d, const ssb_pyr_fwd_io* io, void* tape,
                    ssb_stream_t stream);
int ssb_pyr_backward(const ssb_pyr_desc* d, const ssb_pyr_bwd_io* io, const void* tape,
                     void* workspace, ssb_stream_t stream);

/* Primitives behind the reference's surface helpers (same math, planar). */
/* normalize_kernels (pyramid.py:93-109): joint softmax over the first `active`
 * of C channels per pixel; channels >= active get weight exactly 0. */
int ssb_softmax_channels(int dtype, int B, int C, int H, int W, int active,
                         const void* logits, void* weights, ssb_stream_t stream);
/* gather5 (pyramid.py:184-187) for k x k: weights (B, k*k, H, W) */
int ssb_gather(int dtype, int B, int C, int H, int W, int ksize, const void* image,
               const void* weights, void* out, ssb_stream_t stream);
/* upsample2 (pyramid.py:234-241): weights (B, 4, Hf, Wf), coarse (B, C, Hc, Wc) */
int ssb_upsample2(int dtype, int B, int C, int Hc, int Wc, int Hf, int Wf, const void* coarse,
                  const void* weights, void* out, ssb_stream_t stream);
/* _avgpool2 (pyramid.py:140-149): out (B, C, ceil(H/2), ceil(W/2)) */
int ssb_avgpool2(int dtype, int B, int C, int H, int W, const void* in, void* out,
                 ssb_stream_t stream);

/* ------------------------------------------------------------------------
 * (a) sample placement -- replaces rng.py `uniform_grid[_batch]` (:57-63,
 * :73-81), density.py `normalize_density` (:55-65), `allocate` (:209-233),
 * `holdout_taken` (:196-206), estimators.py `stochastic_core` (:90-133),
 * `_bank_inputs`/`_stochastic_estimate` (:136-149).  All decision
 * arithmetic is float64 so counts and masks are bit-exact.
 * ---------------------------------------------------------------------- */
enum { SSB_RULE_STOCHASTIC = 0, SSB_RULE_RELAXED = 1, SSB_RULE_GUMBEL = 2 };
enum {
    SSB_VAR_STOCHASTIC = 0,
    SSB_VAR_RELAXED = 1,
    SSB_VAR_STRAIGHT_THROUGH = 2,
    SSB_VAR_GUMBEL = 3
};

/* u[b, y, x] = uniform(seed, frame_b, x, y, stream_id), f64 (B, H, W), where
 * frame_b = frames[b] if `frames` (device, B x i64) is non-NULL, else frame0 + b. */
int ssb_uniform_grid(uint64_t seed, int64_t frame0, const int64_t* frames, int B, int H, int W,
                     uint64_t stream_id, double* u, ssb_stream_t stream);

/* one variate of the same hash (rng.pixel_uniform, rng.py:51-54) */
int ssb_uniform_at(uint64_t seed, int64_t frame, int64_t x, int64_t y, uint64_t stream_id, double* u,
                   ssb_stream_t stream);

/* normalize_density: spp = budget/8 + 7/8*budget*N*softmax(scores) per frame.
 * scores f64 (B, H, W); workspace from ssb_density_workspace_bytes (also
 * sized for ssb_place: its partial pairs and per-frame column hashes). */
int ssb_density_workspace_bytes(int B, int H, int W, size_t* bytes);
int ssb_normalize_density(int B, int H, int W, const double* scores, double budget,
                          double* spp, void* workspace, ssb_stream_t stream);

typedef struct ssb_alloc_desc {
    int32_t B, H, W;
    int32_t rule;     /* SSB_RULE_* */
    int32_t dithered; /* 0: u from the allocation stream; 1: u from the rank mask */
    int32_t mask_size;
    uint64_t seed;
    int64_t frame0; /* batch element b uses frame0 + b */
    double gumbel_temp;
} ssb_alloc_desc;

/* allocate: base = floor(spp) (i64), frac, u, taken (u8).  `rank` (T*T i64,
 * device) only for dithered mode.  Any output pointer may be NULL. */
int ssb_allocate(const ssb_alloc_desc* d, const double* spp, const int64_t* rank, int64_t* base,
                 double* frac, double* u, uint8_t* taken, ssb_stream_t stream);

typedef struct ssb_estimate_desc {
    int32_t B, H, W;
    int32_t variant;  /* SSB_VAR_* */
    int32_t capacity; /* bank samples per pixel S */
    int32_t reserved;
    double lam, gumbel_temp, density_floor;
} ssb_estimate_desc;

/* stochastic_core: spp/frac/u (B,H,W) f64; base_sum/holdout (B,H,W,3) f64;
 * outputs noisy/grad/contrib (B,H,W,3) f64 and drawn (B,H,W) u8. */
int ssb_stochastic_core(const ssb_estimate_desc* d, const double* spp, const double* frac,
                        const double* u, const double* base_sum, const double* holdout,
                        double* noisy, double* grad, double* contrib, uint8_t* drawn,
                        ssb_stream_t stream);

/* _stochastic_estimate with the bank read fused: samples (B,H,W,S,3) f64
 * (SampleBank layout).  noisy is clamped at 0 like the RadianceImage result;
 * used = min(base, S-1) + drawn.  noisy32 (B,3,H,W) f32 planar is the fused
 * filter input (may be NULL); any other output may be NULL. */
int ssb_estimate(const ssb_estimate_desc* d, const double* spp, const int64_t* base,
                 const double* frac, const double* u, const double* samples, double* noisy,
                 double* grad, double* contrib, int64_t* used, float* noisy32,
                 ssb_stream_t stream);

/* Fused inference placement (scores -> spp -> counts -> mask -> accumulated
 * radiance) for the filter: scores f32 (B,H,W); bank f32 planar (B,S,3,H,W);
 * writes noisy (B,3,H,W) f32 and optionally spp f32, taken u8.  Decisions
 * (floor, u < frac) are made in float64 from the float64 spp. */
typedef struct ssb_place_desc {
    int32_t B, H, W, capacity;
    int32_t variant; /* SSB_VAR_* (ssb_place_fused: SSB_VAR_STOCHASTIC only) */
    int32_t reserved;
    uint64_t seed;
    int64_t frame0;
    double budget;
} ssb_place_desc;
int ssb_place_fused(const ssb_place_desc* d, const float* scores, const float* bank,
                    float* noisy, float* spp_out, uint8_t* taken_out, void* workspace,
                    ssb_stream_t stream);

/* The fused placement for every stochastic estimator variant (the training
 * default is "relaxed", optimize.py:53): normalize_density -> allocate
 * (take_rule(variant)) -> _stochastic_estimate over a materialised bank
 * (density.py:55-65,209-233; estimators.py:90-149), two launches (per-block
 * (max, sum) partials of the frame softmax; one pass that finishes the
 * partials in every CTA in a fixed order and places the samples).  Decisions
 * are exact: u = (h >> 11) 2^-53 is compared as the integer h >> 11 against
 * frac 2^53 (stochastic) or (1 - frac) 2^53 (relaxed) in float64, the
 * estimator values are float64 and stored float32.  Outputs (B,3,H,W) f32
 * planar: noisy (>= 0, required), grad = d noisy / d density (optional);
 * (B,H,W): spp f32, taken u8 (the allocation's holdout_taken for
 * take_rule(variant)), drawn u8 (the estimator's drawn mask), all optional.
 * workspace: ssb_density_workspace_bytes. */
typedef struct ssb_place_cfg {
    double lam, gumbel_temp, density_floor; /* EstimatorConfig (estimators.py:44-59) */
} ssb_place_cfg;
typedef struct ssb_place_io {
    const float* scores; /* (B,H,W) */
    const float* bank;   /* (B,S,3,H,W): sample j of channel c at [(b*S + j)*3 + c] */
    float* noisy;
    float* grad;
    float* spp;
    uint8_t* taken;
    uint8_t* drawn;
} ssb_place_io;
int ssb_place(const ssb_place_desc* d, const ssb_place_cfg* cfg, const ssb_place_io* io, void* workspace,
              ssb_stream_t stream);

/* Small frames (BASELINE c0): the inference path -- the stochastic fused
 * placement (as ssb_place_fused, capacity 2: identical noisy) followed by
 * reconstruct_core (pyramid.py:292-345) with demod, native blend, 3
 * channels, float32 -- in ONE cooperative kernel with grid-wide barriers
 * between the stages (the partial pairs and their fold, place, one pooled
 * level per barrier, one forward level per barrier) instead of eight
 * dependent launches.  logits[l] (B, k^2 (+4 below the top level), H_l, W_l).
 * Returns SSB_EUNSUPPORTED outside B <= 8, B*H*W <= 2^20, W % 4 == 0, k in
 * {3,5,7} (the caller then runs ssb_place_fused + ssb_pyr_forward).  No tape:
 * inference only. */
int ssb_infer_small_workspace_bytes(int B, int H, int W, int levels, size_t* bytes);
int ssb_infer_small(const ssb_place_desc* pd, const float* scores, const float* bank, const float* demod,
                    int levels, int ksize, const float* const* logits, float* noisy, float* out,
                    void* workspace, ssb_stream_t stream);

/* ------------------------------------------------------------------------
 * Row bands: one 8K frame split into G row bands,
 * one per GPU, exchanging only r rows of each pooled level and one Lhat row
 * per level with the neighbours (paper_2602_08642_b200/bands.py).  The band
 * runs the pyramid level by level on caller-laid-out, row-extended buffers:
 *
 * ssb_pyr_forward_level -- one level of reconstruct_core (pyramid.py:321-338)
 * on planar buffers of the SAME geometry (B, C, H, W) for img / demod / out
 * and (B, C_l, H, W) for the logits: out = gather_k(img', w[:k^2]) +
 * upsample2(coarse, w[k^2:]) with w = softmax(logits) and img' = img /
 * max(demod, 1e-3), out *= max(demod, 1e-3) when demod != NULL (level 0);
 * coarse (B, C, Hc, Wc), parent(y) = min((y + i) / 2, Hc - 1), NULL at the
 * coarsest level (has_coarse = 0).  The same fused kernels as ssb_pyr_forward:
 * every output pixel is bit-identical to the full-frame call's. */
typedef struct ssb_pyr_level_desc {
    int32_t batch, channels, height, width, ksize;
    int32_t image_dtype, logit_dtype, blend_mode;
    int32_t has_coarse, coarse_height, coarse_width;
    int32_t reserved;
} ssb_pyr_level_desc;
int ssb_pyr_forward_level(const ssb_pyr_level_desc* d, const void* img, const void* demod, const void* logits,
                          const void* coarse, void* out, ssb_stream_t stream);
/* count-correct 2x2 pooling (pyramid.py:140-149) on strided planar views
 * (element strides per channel plane and per batch item), demodulating on
 * load when demod != NULL (x0 = in / max(demod, 1e-3), same strides as in):
 * the kernel of ssb_pyr_forward's pyramid build, so bands pool bit-identically */
int ssb_pool2_strided(int dtype, int B, int C, int H, int W, const void* in, long long in_c, long long in_b,
                      const void* demod, void* out, long long out_c, long long out_b, ssb_stream_t stream);
/* halo transport over peer memory (NVLink P2P stores; the destination may be
 * another GPU's buffer mapped into this process through CUDA IPC, peer access
 * enabled with ssb_enable_peer): copy `planes` planes of `rows` x `row_elems`
 * elements (esz bytes each; source / destination plane pitches in elements),
 * then a system-scope release store of `value` into *flag.  ssb_flag_wait
 * blocks `stream` (one spinning thread, acquire loads) until *flag >= value.
 * Generation counters make the flags reusable without resets. */
int ssb_halo_put(void* dst, long long dst_pitch, const void* src, long long src_pitch, int planes, int rows,
                 int row_elems, int esz, int* flag, int value, ssb_stream_t stream);
int ssb_flag_wait(const int* flag, int value, ssb_stream_t stream);
int ssb_enable_peer(int device, int peer);

/* ------------------------------------------------------------------------
 * Temporal path -- replaces images.py `warp_array`
 * (:88-119) and `warp_backward` (:122-147).  Planar: prev/out/grad (B,C,H,W),
 * motion (B,2,H,W) = (mx, my), validity (B,H,W) (may be NULL).  dtype
 * SSB_F32 | SSB_F64.  The transpose is a deterministic gather in the
 * reference's summation order (float64: bit-exact) for any motion: frames with
 * max |motion| + 1 > 16 take an O(HW) segment-candidate path instead of the
 * per-pixel scan; workspace: ssb_warp_backward_workspace_bytes(B, H, W).
 * ---------------------------------------------------------------------- */
int ssb_warp(int dtype, int B, int C, int H, int W, const void* prev, const void* motion,
             void* out, void* validity, ssb_stream_t stream);
int ssb_warp_backward_workspace_bytes(int B, int H, int W, size_t* bytes);
int ssb_warp_backward(int dtype, int B, int C, int H, int W, const void* grad_out,
                      const void* motion, void* grad_prev, void* workspace, ssb_stream_t stream);

/* ------------------------------------------------------------------------
 * Estimator backward to the density scores --
 * replaces optimize.py:244-251 (g_spp = sum_f sum_c g_input * grad_density,
 * scipy gaussian_filter(sigma, mode="nearest"), then 7/8*budget*N *
 * density.softmax_backward(softmax(scores), g_spp), density.py:43-52).
 * g_input / grad_density (B,F,C,H,W) planar, scores and g_scores (B,H,W);
 * dtype SSB_F32 | SSB_F64 (float64 arithmetic inside).  sigma = 0: no blur.
 * ---------------------------------------------------------------------- */
int ssb_score_grad_workspace_bytes(int B, int H, int W, size_t* bytes);
int ssb_score_grad(int dtype, int B, int F, int C, int H, int W, const void* g_input,
                   const void* grad_density, const void* scores, double budget, double sigma,
                   void* g_scores, void* workspace, ssb_stream_t stream);

/* ------------------------------------------------------------------------
 * Tonemap + loss epilogue -- replaces tonemap.py
 * `tonemap_array` (:87-88) / `tonemap_backward` (:95-118) and losses.py
 * `spatial_loss` / `temporal_loss` / `combined_loss` (:58-91) with the loss
 * gradients of optimize.py:219-231.  Images (B,3,H,W), maps (B,H,W); tmo =
 * {exposure, contrast, saturation, toe, shoulder} (host doubles).
 * ssb_losses: ldr0_w/ref_w (history) and validity/mask may be NULL; any
 * output may be NULL; losses = B x {spatial, temporal, combined} (device
 * doubles, needs the workspace).
 * ---------------------------------------------------------------------- */
int ssb_tonemap(int dtype, int B, int H, int W, const double* tmo, const void* radiance, void* ldr,
                ssb_stream_t stream);
int ssb_tonemap_backward(int dtype, int B, int H, int W, const double* tmo, const void* radiance,
                         const void* upstream, void* grad, ssb_stream_t stream);
int ssb_losses_workspace_bytes(int B, size_t* bytes);
int ssb_losses(int dtype, int B, int H, int W, const void* ldr1, const void* ref, const void* ldr0_w,
               const void* ref_w, const void* validity, const void* mask, void* sp_map, void* tm_map,
               void* cb_map, double* losses, void* g_ldr1, void* g_ldr0_w, void* workspace,
               ssb_stream_t stream);

/* The evaluate_step epilogue fused (optimize.py:219-231 over tonemap.py and
 * losses.py): tonemap(radiance) -> losses vs ref (+ warped history) -> the
 * loss gradient w.r.t. the LDR frame -> chained through the tonemap, in one
 * pass.  Equals ssb_tonemap + ssb_losses(g_ldr1, g_ldr0_w) +
 * ssb_tonemap_backward (float64: bit-identical).  grad_radiance required;
 * ldr (the tonemapped frame), losses (needs the ssb_losses workspace) and
 * g_ldr0_w optional; ldr0_w/ref_w/validity/mask as in ssb_losses. */
int ssb_epilogue(int dtype, int B, int H, int W, const double* tmo, const void* radiance, const void* ref,
                 const void* ldr0_w, const void* ref_w, const void* validity, const void* mask, void* ldr,
                 double* losses, void* grad_radiance, void* g_ldr0_w, void* workspace, ssb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SSB_API_H */
