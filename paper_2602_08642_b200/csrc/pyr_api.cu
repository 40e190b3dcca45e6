// C ABI of the pyramid filter + the reference's surface primitives.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "pyr_launch.cuh"
#include "tma.cuh"

#include <mutex>

namespace ssb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_check(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(where) + ": " + cudaGetErrorString(e));
        return SSB_ECUDA;
    }
    return SSB_OK;
}

// ---- launch accounting (see ssb_set_launch_events) ----
static std::atomic<unsigned long long> g_launches{0};
struct LaunchHook {
    cudaEvent_t const* ev = nullptr;
    int cap = 0;
    int* count = nullptr;
};
static thread_local LaunchHook g_hook;

void launch_begin(cudaStream_t s) {
    if (g_hook.ev && *g_hook.count < g_hook.cap) cudaEventRecord(g_hook.ev[2 * *g_hook.count], s);
}

void launch_end(cudaStream_t s) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (g_hook.ev && *g_hook.count < g_hook.cap) {
        cudaEventRecord(g_hook.ev[2 * *g_hook.count + 1], s);
        ++*g_hook.count;
    }
}

// ---- TMA tensor maps (driver entry point fetched once through the runtime) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool make_tma_map_4d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int esz,
                     long long W, long long H, long long C, long long B, int box_w, int box_h,
                     int box_c) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || !base || ((uintptr_t)base & 15)) return false;
    const cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)B};
    const cuuint64_t strides[3] = {(cuuint64_t)(W * esz), (cuuint64_t)(W * H * esz),
                                   (cuuint64_t)(W * H * C * esz)};
    for (int i = 0; i < 3; ++i)
        if (strides[i] % 16 || strides[i] >= (1ull << 40)) return false;
    if ((box_w * esz) % 16 || box_w > 256 || box_h > 256 || box_c > 256) return false;
    const cuuint32_t box[4] = {(cuuint32_t)box_w, (cuuint32_t)box_h, (cuuint32_t)box_c, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, dtype, 4, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// SSB_DEBUG_SYNC=1: synchronise after every launch and report the first
// failing kernel by name (debugging aid; never set in measurements)
void launch_debug_check(cudaStream_t s, const char* what) {
    static const bool on = [] {
        const char* e = getenv("SSB_DEBUG_SYNC");
        return e && e[0] == '1';
    }();
    if (!on) return;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "[ssb] kernel failed: %s\n  -> %s\n", what, cudaGetErrorString(e));
        fflush(stderr);
    }
}

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

static int logit_channels(const ssb_pyr_desc* d, int l) {
    const int taps = d->ksize * d->ksize;
    int n = taps;
    if (l < d->levels - 1) n += d->blend_mode == SSB_BLEND_TIED ? 1 : 4;
    if (l == 0 && d->has_prev) n += taps;
    return n;
}

int make_plan(const ssb_pyr_desc* d, PyrPlan* p) {
    if (!d) {
        set_error("null descriptor");
        return SSB_EINVAL;
    }
    if (d->batch < 1 || d->channels < 1 || d->height < 1 || d->width < 1) {
        set_error("batch, channels, height and width must be >= 1");
        return SSB_EINVAL;
    }
    if (d->levels < 1 || d->levels > SSB_MAX_LEVELS) {
        set_error("levels must be in [1, SSB_MAX_LEVELS]");
        return SSB_EINVAL;
    }
    if (d->ksize != 3 && d->ksize != 5 && d->ksize != 7) {
        set_error("ksize must be 3, 5 or 7");
        return SSB_EUNSUPPORTED;
    }
    if (d->blend_mode != SSB_BLEND_NATIVE && d->blend_mode != SSB_BLEND_TIED) {
        set_error("unknown blend_mode");
        return SSB_EINVAL;
    }
    const bool ok_types = (d->image_dtype == SSB_F32 &&
                           (d->logit_dtype == SSB_F32 || d->logit_dtype == SSB_BF16)) ||
                          (d->image_dtype == SSB_F64 && d->logit_dtype == SSB_F64);
    if (!ok_types) {
        set_error("supported (image, logit) dtypes: (f32, f32), (f32, bf16), (f64, f64)");
        return SSB_EUNSUPPORTED;
    }
    p->B = d->batch;
    p->C = d->channels;
    p->H = d->height;
    p->W = d->width;
    p->L = d->levels;
    p->K = d->ksize;
    p->esz = d->image_dtype == SSB_F64 ? 8 : 4;
    p->lgesz = d->logit_dtype == SSB_F64 ? 8 : (d->logit_dtype == SSB_BF16 ? 2 : 4);
    p->hl[0] = d->height;
    p->wl[0] = d->width;
    for (int l = 1; l < p->L; ++l) {
        p->hl[l] = (p->hl[l - 1] + 1) / 2;
        p->wl[l] = (p->wl[l - 1] + 1) / 2;
    }
    size_t t = 0, w = 0;
    for (int l = 0; l < p->L; ++l) {
        p->nlog[l] = logit_channels(d, l);
        p->pool_off[l] = p->lhat_off[l] = p->ghat_off[l] = p->gl_off[l] = 0;
        if (l == 0) continue;
        const size_t bytes = align256((size_t)p->B * p->C * p->hl[l] * p->wl[l] * p->esz);
        p->pool_off[l] = t;
        t += bytes;
        p->lhat_off[l] = t;
        t += bytes;
        p->ghat_off[l] = w;
        w += bytes;
        p->gl_off[l] = w;
        w += bytes;
    }
    // float32: per-level base-2 log-sum-exp of the softmax (the TMA backward
    // kernels evaluate their weights from it; k_up_transpose reads level 0)
    for (int l = 0; l < p->L; ++l) {
        p->lse_off[l] = 0;
        if (p->esz == 4 && (l == 0 || p->K >= 7)) {
            p->lse_off[l] = t;
            t += align256((size_t)p->B * p->hl[l] * p->wl[l] * sizeof(float));
        }
    }
    // kernels address channels of one frame with 32-bit offsets
    if ((unsigned long long)p->nlog[0] * (unsigned long long)p->H * (unsigned long long)p->W >=
        (1ull << 32)) {
        set_error("frame too large: logit channels * H * W must stay below 2^32 per frame");
        return SSB_EUNSUPPORTED;
    }
    p->tape_bytes = t;
    p->ws_bytes = w;
    return SSB_OK;
}

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_version(void) { return SSB_VERSION; }

const char* ssb_last_error(void) { return g_last_error.c_str(); }

unsigned long long ssb_launch_count(void) { return g_launches.load(); }

int ssb_set_launch_events(void* const* events, int capacity, int* count) {
    if (events && (capacity < 0 || !count)) {
        set_error("ssb_set_launch_events: need capacity >= 0 and a count pointer");
        return SSB_EINVAL;
    }
    g_hook.ev = reinterpret_cast<cudaEvent_t const*>(events);
    g_hook.cap = events ? capacity : 0;
    g_hook.count = events ? count : nullptr;
    if (count) *count = 0;
    return SSB_OK;
}

int ssb_pyr_logit_channels(const ssb_pyr_desc* d, int level) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (level < 0 || level >= p.L) {
        set_error("level out of range");
        return SSB_EINVAL;
    }
    return p.nlog[level];
}

int ssb_pyr_level_dims(const ssb_pyr_desc* d, int level, int32_t* h, int32_t* w) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (level < 0 || level >= p.L || !h || !w) {
        set_error("level out of range or null output");
        return SSB_EINVAL;
    }
    *h = p.hl[level];
    *w = p.wl[level];
    return SSB_OK;
}

int ssb_pyr_tape_bytes(const ssb_pyr_desc* d, size_t* bytes) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (!bytes) {
        set_error("null output");
        return SSB_EINVAL;
    }
    *bytes = p.tape_bytes;
    return SSB_OK;
}

int ssb_pyr_workspace_bytes(const ssb_pyr_desc* d, size_t* bytes) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (!bytes) {
        set_error("null output");
        return SSB_EINVAL;
    }
    *bytes = p.ws_bytes;
    return SSB_OK;
}

}  // extern "C"

namespace ssb {
SSB_EXTERN_PYR(3, float, float)
SSB_EXTERN_PYR(3, __nv_bfloat16, float)
SSB_EXTERN_PYR(3, double, double)
SSB_EXTERN_PYR(5, float, float)
SSB_EXTERN_PYR(5, __nv_bfloat16, float)
SSB_EXTERN_PYR(5, double, double)
SSB_EXTERN_PYR(7, float, float)
SSB_EXTERN_PYR(7, __nv_bfloat16, float)
SSB_EXTERN_PYR(7, double, double)

template <typename Fn>
static int by_types(const ssb_pyr_desc* d, Fn&& fn) {
    // fn.template operator()<K, TL, T>() dispatched on (ksize, logit dtype)
    switch (d->ksize) {
#define CASE_K(KV)                                                                   \
    case KV:                                                                         \
        if (d->logit_dtype == SSB_F32) return fn.template call<KV, float, float>();  \
        if (d->logit_dtype == SSB_BF16)                                              \
            return fn.template call<KV, __nv_bfloat16, float>();                     \
        return fn.template call<KV, double, double>();
        CASE_K(3)
        CASE_K(5)
        CASE_K(7)
#undef CASE_K
    }
    set_error("unsupported ksize");
    return SSB_EUNSUPPORTED;
}

struct FwdCall {
    const ssb_pyr_desc* d;
    const PyrPlan* p;
    const ssb_pyr_fwd_io* io;
    void* tape;
    cudaStream_t s;
    template <int K, typename TL, typename T>
    int call() { return run_forward<K, TL, T>(d, *p, io, tape, s); }
};

struct BwdCall {
    const ssb_pyr_desc* d;
    const PyrPlan* p;
    const ssb_pyr_bwd_io* io;
    const void* tape;
    void* ws;
    cudaStream_t s;
    template <int K, typename TL, typename T>
    int call() { return run_backward<K, TL, T>(d, *p, io, tape, ws, s); }
};
}  // namespace ssb

extern "C" {

int ssb_pyr_forward(const ssb_pyr_desc* d, const ssb_pyr_fwd_io* io, void* tape,
                    ssb_stream_t stream) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (!io || !io->noisy || !io->out) {
        set_error("ssb_pyr_forward: noisy and out are required");
        return SSB_EINVAL;
    }
    if ((d->has_demod != 0) != (io->demod != nullptr) || (d->has_prev != 0) != (io->prev != nullptr)) {
        set_error("ssb_pyr_forward: demod/prev pointers must match has_demod/has_prev");
        return SSB_EINVAL;
    }
    for (int l = 0; l < p.L; ++l)
        if (!io->logits[l]) {
            set_error("ssb_pyr_forward: missing logits for a level");
            return SSB_EINVAL;
        }
    if (p.L > 1 && !tape) {
        set_error("ssb_pyr_forward: tape required for levels > 1");
        return SSB_EINVAL;
    }
    FwdCall c{d, &p, io, tape, (cudaStream_t)stream};
    return by_types(d, c);
}

int ssb_pyr_forward_level(const ssb_pyr_level_desc* d, const void* img, const void* demod, const void* logits,
                          const void* coarse, void* out, ssb_stream_t stream) {
    if (!d || !img || !logits || !out || d->batch < 1 || d->channels < 1 || d->height < 1 || d->width < 1) {
        set_error("ssb_pyr_forward_level: bad arguments");
        return SSB_EINVAL;
    }
    if (d->has_coarse && (!coarse || d->coarse_height < 1 || d->coarse_width < 1)) {
        set_error("ssb_pyr_forward_level: has_coarse needs the coarse level and its dims");
        return SSB_EINVAL;
    }
    if (d->ksize != 3 && d->ksize != 5 && d->ksize != 7) {
        set_error("unsupported ksize");
        return SSB_EUNSUPPORTED;
    }
    const bool f64 = d->image_dtype == SSB_F64;
    if (f64 != (d->logit_dtype == SSB_F64) || (d->image_dtype != SSB_F32 && !f64)) {
        set_error("ssb_pyr_forward_level: images f32 with f32/bf16 logits, or f64 with f64");
        return SSB_EUNSUPPORTED;
    }
    if ((long long)d->channels * d->height * d->width >= (1ll << 32)) {
        set_error("ssb_pyr_forward_level: C*H*W must be < 2^32 per frame");
        return SSB_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const void* dm = d->has_coarse ? coarse : nullptr;
    switch (d->ksize) {
#define LEVEL_K(KV)                                                                                          \
    case KV:                                                                                                 \
        if (d->logit_dtype == SSB_F32) return run_forward_level<KV, float, float>(d, img, demod, logits, dm, out, s); \
        if (d->logit_dtype == SSB_BF16)                                                                      \
            return run_forward_level<KV, __nv_bfloat16, float>(d, img, demod, logits, dm, out, s);          \
        return run_forward_level<KV, double, double>(d, img, demod, logits, dm, out, s);
        LEVEL_K(3)
        LEVEL_K(5)
        LEVEL_K(7)
#undef LEVEL_K
    }
    return SSB_EUNSUPPORTED;
}

int ssb_pool2_strided(int dtype, int B, int C, int H, int W, const void* in, long long in_c, long long in_b,
                      const void* demod, void* out, long long out_c, long long out_b, ssb_stream_t stream) {
    if (B < 1 || C < 1 || H < 1 || W < 1 || !in || !out || in_c < (long long)H * W || out_c < 1) {
        set_error("ssb_pool2_strided: bad arguments");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    for (int c0 = 0; c0 < C; c0 += kMaxCh) {
        const int nc = C - c0 < kMaxCh ? C - c0 : kMaxCh;
        if (dtype == SSB_F32)
            launch_pool<float>(B, nc, H, W, (const float*)in + c0 * in_c, in_b, in_c,
                               demod ? (const float*)demod + c0 * in_c : nullptr, (float*)out + c0 * out_c, out_b, out_c, s);
        else if (dtype == SSB_F64)
            launch_pool<double>(B, nc, H, W, (const double*)in + c0 * in_c, in_b, in_c,
                                demod ? (const double*)demod + c0 * in_c : nullptr, (double*)out + c0 * out_c, out_b,
                                out_c, s);
        else {
            set_error("ssb_pool2_strided: dtype must be f32 or f64");
            return SSB_EUNSUPPORTED;
        }
    }
    return cuda_check("ssb_pool2_strided");
}

int ssb_pyr_backward(const ssb_pyr_desc* d, const ssb_pyr_bwd_io* io, const void* tape,
                     void* workspace, ssb_stream_t stream) {
    PyrPlan p;
    int rc = make_plan(d, &p);
    if (rc) return rc;
    if (!io || !io->noisy || !io->upstream || !io->g_noisy) {
        set_error("ssb_pyr_backward: noisy, upstream and g_noisy are required");
        return SSB_EINVAL;
    }
    if ((d->has_demod != 0) != (io->demod != nullptr) || (d->has_prev != 0) != (io->prev != nullptr)) {
        set_error("ssb_pyr_backward: demod/prev pointers must match has_demod/has_prev");
        return SSB_EINVAL;
    }
    if (d->has_prev && !io->g_prev) {
        set_error("ssb_pyr_backward: g_prev required when has_prev");
        return SSB_EINVAL;
    }
    const bool want = io->g_logits[0] != nullptr;
    for (int l = 0; l < p.L; ++l) {
        if (!io->logits[l] || (want && !io->g_logits[l])) {
            set_error("ssb_pyr_backward: logits (and g_logits when wanted) needed per level");
            return SSB_EINVAL;
        }
    }
    if (io->g_demod && d->has_demod && !io->out) {
        set_error("ssb_pyr_backward: forward output required for the demod gradient");
        return SSB_EINVAL;
    }
    if (p.L > 1 && (!tape || !workspace)) {
        set_error("ssb_pyr_backward: tape and workspace required for levels > 1");
        return SSB_EINVAL;
    }
    BwdCall c{d, &p, io, tape, workspace, (cudaStream_t)stream};
    return by_types(d, c);
}


#ifdef SSB_ROLE_TIMING
// experiment build only (not in ssb_api.h): this TU's copy of the backward
// kernel's per-role cycle counters (tools/role_timing.py sums every TU)
int ssb_debug_role_cycles0(unsigned long long* out8) { return ssb::role_cycles_read(out8); }
#endif

}  // extern "C"
