// Raw GPU1 <- GPU0 transfer throughput for back-to-back copies of size n into
// distinct buffers: copy engine pull/push vs SM copy kernels pull/push.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

struct Mode { const char* name; int dev; bool ce; int streams; int grid; };

int main() {
    const int reps = 64;
    Mode modes[] = {{"CE-pull-1s", 1, true, 1, 0},      {"CE-push-1s", 0, true, 1, 0},
                    {"CE-push-4s", 0, true, 4, 0},      {"SM-pull-4s-296", 1, false, 4, 296},
                    {"SM-push-4s-296", 0, false, 4, 296}, {"SM-push-4s-148", 0, false, 4, 148},
                    {"SM-push-1s-592", 0, false, 1, 592}};
    for (size_t n : {(size_t)1 << 20, (size_t)4 << 20, (size_t)16 << 20, (size_t)64 << 20}) {
        char *src, *dst;
        const int nbuf = (int)((((size_t)1 << 30) / n) < 64 ? ((size_t)1 << 30) / n : 64);
        cudaSetDevice(0); cudaMalloc(&src, n * nbuf); cudaDeviceEnablePeerAccess(1, 0);
        cudaSetDevice(1); cudaMalloc(&dst, n * nbuf); cudaDeviceEnablePeerAccess(0, 0);
        for (const Mode& m : modes) {
            cudaSetDevice(m.dev);
            cudaStream_t st[4];
            for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            cudaEvent_t a, b, j[4];
            cudaEventCreate(&a); cudaEventCreate(&b);
            for (auto& e : j) cudaEventCreate(&e);
            float ms = 0;
            for (int warm = 0; warm < 2; ++warm) {
                cudaDeviceSynchronize();
                cudaEventRecord(a, st[0]);
                for (int k = 1; k < 4; ++k) cudaStreamWaitEvent(st[k], a, 0);
                for (int r = 0; r < reps; ++r) {
                    cudaStream_t s = st[r % m.streams];
                    char* sp = src + (size_t)(r % nbuf) * n;
                    char* dp = dst + (size_t)(r % nbuf) * n;
                    if (m.ce) cudaMemcpyAsync(dp, sp, n, cudaMemcpyDefault, s);
                    else copy_kernel<<<m.grid, 512, 0, s>>>((const int4*)sp, (int4*)dp, n / 16);
                }
                for (int k = 1; k < 4; ++k) { cudaEventRecord(j[k], st[k]); cudaStreamWaitEvent(st[0], j[k], 0); }
                cudaEventRecord(b, st[0]);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
            }
            printf("n=%3zu MB %-16s %7.1f GB/s (%.2f us/copy)\n", n >> 20, m.name, (double)n * reps / (ms * 1e-3) / 1e9,
                   ms * 1e3 / reps);
            for (auto& s : st) cudaStreamDestroy(s);
        }
        cudaSetDevice(1); cudaFree(dst); cudaSetDevice(0); cudaFree(src);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
