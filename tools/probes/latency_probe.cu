// Probe: host-observed latency floors of the ways a small device frame can move
// from GPU 0 to GPU 1 (one process, peer access enabled), 1 B .. 64 KiB:
//   ce_event   cudaMemcpyAsync peer D2D + cudaEventRecord, host spins on cudaEventQuery
//   k_event    1-CTA copy kernel (peer stores)      + cudaEventRecord, host spins on cudaEventQuery
//   k_flag     copy kernel that, after a system fence, stores a sequence number into
//              pinned host memory (cudaHostAlloc, mapped); host spins on that word
//   launch     empty kernel + event (launch + completion floor)
// Question: which one gives a one-way device-frame latency near 5 us?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o latency_probe latency_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16,
                            const unsigned char* s1, unsigned char* d1, size_t tail,
                            volatile unsigned long long* flag, unsigned long long seq) {
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    for (size_t i = threadIdx.x; i < tail; i += blockDim.x) d1[i] = s1[i];
    if (flag) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            *flag = seq;
        }
    }
}

__global__ void empty_kernel() {}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    const int peer = n > 1 ? 1 : 0;
    CK(cudaSetDevice(0));
    if (peer) CK(cudaDeviceEnablePeerAccess(peer, 0));
    void *src, *dst;
    CK(cudaMalloc(&src, 1 << 20));
    CK(cudaSetDevice(peer));
    CK(cudaMalloc(&dst, 1 << 20));
    CK(cudaSetDevice(0));
    unsigned long long* flag;
    CK(cudaHostAlloc(&flag, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    unsigned long long* dflag;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), flag, 0));
    *flag = 0;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const int iters = 2000;
    printf("peer device %d\n", peer);
    unsigned long long seq = 0;
    for (size_t bytes : {size_t(1), size_t(256), size_t(4096), size_t(65536)}) {
        const size_t n16 = bytes / 16, tail = bytes % 16;
        double best[4] = {1e9, 1e9, 1e9, 1e9}, sum[4] = {0, 0, 0, 0};
        for (int mode = 0; mode < 4; ++mode) {
            for (int it = 0; it < iters + 100; ++it) {
                const double t0 = now_us();
                if (mode == 0) {
                    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
                    CK(cudaEventRecord(ev, s));
                    while (cudaEventQuery(ev) == cudaErrorNotReady) {
                    }
                } else if (mode == 1) {
                    copy_kernel<<<1, 256, 0, s>>>((const uint4*)src, (uint4*)dst, n16, (const unsigned char*)src + n16 * 16,
                                                 (unsigned char*)dst + n16 * 16, tail, nullptr, 0);
                    CK(cudaEventRecord(ev, s));
                    while (cudaEventQuery(ev) == cudaErrorNotReady) {
                    }
                } else if (mode == 2) {
                    ++seq;
                    copy_kernel<<<1, 256, 0, s>>>((const uint4*)src, (uint4*)dst, n16, (const unsigned char*)src + n16 * 16,
                                                 (unsigned char*)dst + n16 * 16, tail, dflag, seq);
                    while (*(volatile unsigned long long*)flag != seq) {
                    }
                } else {
                    empty_kernel<<<1, 32, 0, s>>>();
                    CK(cudaEventRecord(ev, s));
                    while (cudaEventQuery(ev) == cudaErrorNotReady) {
                    }
                }
                const double dt = now_us() - t0;
                if (it >= 100) {
                    sum[mode] += dt;
                    if (dt < best[mode]) best[mode] = dt;
                }
            }
            CK(cudaStreamSynchronize(s));
        }
        printf("%6zu B  ce_event %6.2f us (min %5.2f)  k_event %6.2f (min %5.2f)  k_flag %6.2f (min %5.2f)  launch %6.2f (min %5.2f)\n",
               bytes, sum[0] / iters, best[0], sum[1] / iters, best[1], sum[2] / iters, best[2], sum[3] / iters, best[3]);
    }
    return 0;
}
