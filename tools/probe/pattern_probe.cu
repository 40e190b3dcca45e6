// Memory-pattern ceiling of the level-0 backward (c4a shape): the same TMA
// box stream per CTA -- column strips of 60 (+2x4 halo) columns, row segments
// of 120 rows walked in steps of 4 rows, per step the boxes of 29 logit planes,
// noisy, demod, upstream, forward output (3 planes each) and the coarse T1
// rows, double buffered and issued one step ahead -- and the same write
// stream (29 logit-gradient planes + g_noisy + g_demod, 16-B streaming stores
// of the own 60 columns), with no arithmetic.  Its bandwidth bounds what the
// real kernel can reach with this access pattern.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DPS=4 -DNST=2 -DMINB=2] \
//        pattern_probe.cu -o pattern_probe -lcuda
//   ./pattern_probe [frames]
// PS = rows per step, NST = TMA stages (prefetch NST - 1 steps ahead), MINB = CTAs per SM,
// NTHR = threads per CTA (the store stream's issuers)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#ifndef PS
#define PS 4
#endif
#ifndef NST
#define NST 2
#endif
#ifndef MINB
#define MINB 2
#endif
#ifndef NTHR
#define NTHR 256
#endif
#ifndef PTXB  // own columns per strip (multiple of 4)
#define PTXB 60
#endif
#ifndef PSEG
#define PSEG 120
#endif
constexpr int NLOG = 29, S = PS, TXB = PTXB, RX = TXB + 8, RA = 4, SEG = PSEG, CB = ((TXB / 2 + 4 + 3) / 4) * 4, CT = S;
constexpr int NQ = TXB / 4;
constexpr int al32(int n) { return (n + 31) & ~31; }  // TMA destinations 128-B aligned
constexpr int LGF = al32(NLOG * S * RX), IMF = al32(3 * S * RX), T1F = al32(3 * CT * CB);
constexpr int STAGE = LGF + 4 * IMF + T1F;  // floats per stage
constexpr uint32_t TX = (NLOG * S * RX + 4 * 3 * S * RX + 3 * CT * CB) * 4;  // exact box bytes

struct Maps {
    CUtensorMap lg, img[4], t1;
};

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void load4(void* dst, const CUtensorMap* m, int x, int y, int c, int b, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(s32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(c), "r"(b), "r"(s32(bar))
        : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, int parity) {
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
                     s32(bar)),
                 "r"(parity)
                 : "memory");
}

__global__ void __launch_bounds__(NTHR, MINB) k_probe(const __grid_constant__ Maps mp, int H, int W, float* gl, float* gx) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bars[NST];
    const int tid = threadIdx.x, b = blockIdx.z;
    const int x0 = blockIdx.x * TXB, y0 = blockIdx.y * SEG, y1 = min(y0 + SEG, H);
    const int nsteps = (y1 - y0 + S - 1) / S;
    if (tid == 0) {
        for (int k = 0; k < NST; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bars[k])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int j) {
        float* st = sm + (j % NST) * STAGE;
        uint64_t* bar = &bars[j % NST];
        const int qs = y0 + j * S;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(TX) : "memory");
        load4(st, &mp.lg, x0 - RA, qs, 0, b, bar);
        for (int k = 0; k < 4; ++k) load4(st + LGF + k * IMF, &mp.img[k], x0 - RA, qs, 0, b, bar);
        load4(st + LGF + 4 * IMF, &mp.t1, (x0 >> 1) & ~3, qs >> 1, 0, b, bar);
    };
    if (tid == 0)
        for (int j = 0; j < NST - 1 && j < nsteps; ++j) issue(j);
    const size_t hw = (size_t)H * W;
    for (int i = 0; i < nsteps; ++i) {
        if (tid == 0 && i + NST - 1 < nsteps) issue(i + NST - 1);
        wait(&bars[i % NST], (i / NST) & 1);
        const float* st = sm + (i % NST) * STAGE;
        const int qs = y0 + i * S;
        // writes: 29 + 6 planes x S rows x 60 own columns as float4 (15 quads per row)
        for (int it = tid; it < (NLOG + 6) * S * NQ; it += NTHR) {  // (S rows)
            const int q = it % NQ, r = (it / NQ) % S, pl = it / (NQ * S);
            const int y = qs + r, x = x0 + 4 * q;
            if (y >= y1 || x >= W) continue;
            const float* src = pl < NLOG ? st + (pl * S + r) * RX + RA + 4 * q
                                         : st + LGF + ((pl - NLOG) % 3 + 3 * ((pl - NLOG) / 3)) * S * RX + r * RX + RA + 4 * q;
            const float4 v = *reinterpret_cast<const float4*>(src);
            float* dst = pl < NLOG ? gl + ((size_t)b * NLOG + pl) * hw : gx + ((size_t)b * 6 + (pl - NLOG)) * hw;
            __stcs(reinterpret_cast<float4*>(dst + (size_t)y * W + x), v);
        }
        __syncthreads();  // the stage is free for the issue two steps ahead
    }
}

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8, H = 1080, W = 1920;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (EncodeTiledFn)p;
    const size_t hw = (size_t)H * W;
    float *lg, *img[4], *t1, *gl, *gx;
    cudaMalloc(&lg, B * NLOG * hw * 4);
    for (int k = 0; k < 4; ++k) cudaMalloc(&img[k], B * 3 * hw * 4);
    cudaMalloc(&t1, B * 3 * (hw / 4) * 4);
    cudaMalloc(&gl, B * NLOG * hw * 4);
    cudaMalloc(&gx, B * 6 * hw * 4);
    cudaMemset(lg, 0, B * NLOG * hw * 4);
    auto mk = [&](CUtensorMap* m, void* base, int w, int h, int c, int bx, int by, int bc) {
        cuuint64_t dims[4] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)c, (cuuint64_t)B};
        cuuint64_t str[3] = {(cuuint64_t)w * 4, (cuuint64_t)w * h * 4, (cuuint64_t)w * h * c * 4};
        cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bc, 1}, es[4] = {1, 1, 1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    Maps mp;
    int bad = mk(&mp.lg, lg, W, H, NLOG, RX, S, NLOG);
    for (int k = 0; k < 4; ++k) bad |= mk(&mp.img[k], img[k], W, H, 3, RX, S, 3);
    bad |= mk(&mp.t1, t1, W / 2, H / 2, 3, CB, CT, 3);
    if (bad) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = NST * STAGE * 4;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((W + TXB - 1) / TXB, (H + SEG - 1) / SEG, B);
    for (int w = 0; w < 3; ++w) k_probe<<<grid, NTHR, smem>>>(mp, H, W, gl, gx);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_probe<<<grid, NTHR, smem>>>(mp, H, W, gl, gx);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    // algorithmic bytes of the real kernel's pattern (own pixels): reads 29 + 12 planes + T1/4, writes 29 + 6
    const double px = (double)B * hw, bytes = px * (4.0 * (NLOG + 12) + 3.0 + 4.0 * (NLOG + 6));
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_probe, NTHR, smem);
    printf("pattern probe TXB=%d SEG=%d S=%d stages=%d minb=%d threads=%d (resident %d/SM): %d frames 1080p, smem %d B/CTA, %.3f ms, %.1f B/px -> %.1f GB/s (%s)\n",
           TXB, SEG, PS, NST, MINB, NTHR, nb, B, smem, ms, bytes / px, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
