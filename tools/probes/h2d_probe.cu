// Probe: pinned host -> device copy bandwidth with the copy split over 1 / 2 / 4
// streams (one cudaMemcpyAsync per stream), 4 GiB, best of 5.  Question: does
// the transpose_sum e2e leg (12.8 GB H2D per step) gain from several copy engines?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o h2d_probe h2d_probe.cu
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

int main() {
    const size_t bytes = size_t(4) << 30;
    void *h = nullptr, *d = nullptr;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&d, bytes));
    memset(h, 1, bytes);
    cudaStream_t s[8];
    for (int i = 0; i < 8; ++i) CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int n : {1, 2, 4, 8}) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0, s[0]));
            for (int i = 1; i < n; ++i) CK(cudaStreamWaitEvent(s[i], e0, 0));
            const size_t part = bytes / n;
            for (int i = 0; i < n; ++i)
                CK(cudaMemcpyAsync(static_cast<char*>(d) + i * part, static_cast<char*>(h) + i * part, part,
                                   cudaMemcpyHostToDevice, s[i]));
            for (int i = 1; i < n; ++i) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, s[i]));
                CK(cudaStreamWaitEvent(s[0], ev, 0));
                CK(cudaEventDestroy(ev));
            }
            CK(cudaEventRecord(e1, s[0]));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        printf("H2D %d stream(s): %.1f GB/s\n", n, bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
