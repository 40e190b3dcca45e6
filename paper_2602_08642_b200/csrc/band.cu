// Halo transport of the row-band forward over
// peer memory: the producer GPU stores the halo rows straight into the
// neighbour's receive buffer (a CUDA-IPC mapping of the neighbour's device
// memory; NVLink P2P stores), then publishes a generation counter with a
// system-scope release store; the consumer's stream waits on that counter
// with one spinning thread (acquire loads) before the kernel that reads the
// halo.  No NCCL, no host round trip.  The band orchestration is bands.py.
#include <string>

#include "common.cuh"

namespace ssb {
void set_error(const std::string& msg);
int cuda_check(const char* where);

// one contiguous block of `bytes` per plane (the halo rows of that plane),
// V-sized vectors
template <typename V>
__global__ void k_halo_copy(char* __restrict__ dst, long long dst_pitch, const char* __restrict__ src,
                            long long src_pitch, long long bytes) {
    const long long nv = bytes / (long long)sizeof(V);
    const V* s = reinterpret_cast<const V*>(src + blockIdx.y * src_pitch);
    V* d = reinterpret_cast<V*>(dst + blockIdx.y * dst_pitch);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x)
        d[i] = __ldg(s + i);
}

__global__ void k_flag_release(int* flag, int value) {
    // every store of the copy kernel before it on this stream is complete
    // (stream order); make them visible system-wide before the flag
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__global__ void k_flag_wait(const int* flag, int value) {
    int v;
    do {
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= value) break;
        __nanosleep(200);
    } while (true);
    __threadfence_system();
}

}  // namespace ssb

using namespace ssb;

extern "C" {

int ssb_halo_put(void* dst, long long dst_pitch, const void* src, long long src_pitch, int planes, int rows,
                 int row_elems, int esz, int* flag, int value, ssb_stream_t stream) {
    if (!dst || !src || planes < 1 || rows < 0 || row_elems < 1 || (esz != 2 && esz != 4 && esz != 8) ||
        dst_pitch < (long long)rows * row_elems || src_pitch < (long long)rows * row_elems) {
        set_error("ssb_halo_put: bad arguments");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // the rows of one plane are contiguous (row pitch == row_elems): one block
    // of rows * row_elems elements per plane
    const long long bytes = (long long)rows * row_elems * esz;
    const long long dp = dst_pitch * esz, sp = src_pitch * esz;
    if (rows > 0) {
        const bool v16 = ((uintptr_t)dst % 16 == 0) && ((uintptr_t)src % 16 == 0) && dp % 16 == 0 && sp % 16 == 0 &&
                         bytes % 16 == 0;
        const long long n = v16 ? bytes / 16 : bytes / esz;
        const unsigned gx = (unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
        dim3 grid(gx, planes);
        if (v16)
            SSB_LAUNCH(s, k_halo_copy<int4><<<grid, 256, 0, s>>>((char*)dst, dp, (const char*)src, sp, bytes));
        else if (esz == 8)
            SSB_LAUNCH(s, k_halo_copy<long long><<<grid, 256, 0, s>>>((char*)dst, dp, (const char*)src, sp, bytes));
        else if (esz == 4)
            SSB_LAUNCH(s, k_halo_copy<int><<<grid, 256, 0, s>>>((char*)dst, dp, (const char*)src, sp, bytes));
        else
            SSB_LAUNCH(s, k_halo_copy<short><<<grid, 256, 0, s>>>((char*)dst, dp, (const char*)src, sp, bytes));
    }
    if (flag) SSB_LAUNCH(s, k_flag_release<<<1, 1, 0, s>>>(flag, value));
    return cuda_check("ssb_halo_put");
}

int ssb_flag_wait(const int* flag, int value, ssb_stream_t stream) {
    if (!flag) {
        set_error("ssb_flag_wait: null flag");
        return SSB_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    SSB_LAUNCH(s, k_flag_wait<<<1, 1, 0, s>>>(flag, value));
    return cuda_check("ssb_flag_wait");
}

int ssb_enable_peer(int device, int peer) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        set_error("ssb_enable_peer: bad device");
        return SSB_ECUDA;
    }
    int can = 0;
    cudaDeviceCanAccessPeer(&can, device, peer);
    cudaError_t e = can ? cudaDeviceEnablePeerAccess(peer, 0) : cudaErrorPeerAccessUnsupported;
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        e = cudaSuccess;
    }
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        set_error(std::string("ssb_enable_peer: ") + cudaGetErrorString(e));
        return SSB_ECUDA;
    }
    return SSB_OK;
}

}  // extern "C"
