// Minimal bulk-copy (TMA) probe: one CTA copies rows global->shared with an mbarrier.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2101_08878_b200/csrc/ptx.cuh"

__global__ void probe(const double* src, double* dst, int rows, int mode) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { m4d::ptx::mbar_init(&bar, 1); m4d::ptx::fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) m4d::ptx::mbar_arrive_expect_tx(&bar, rows * 512);
        __syncwarp();
        for (int r = threadIdx.x; r < rows; r += 32) {
            if (mode == 0) m4d::ptx::bulk_g2s(sm + r * 66, src + r * 64, 512, &bar);
        }
    }
    if (mode == 1 && threadIdx.x == 0) {
        for (int r = 0; r < rows; ++r) m4d::ptx::bulk_g2s(sm + r * 66, src + r * 64, 512, &bar);
    }
    m4d::ptx::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < rows * 64; i += blockDim.x) dst[i] = sm[(i / 64) * 66 + i % 64];
}

int main() {
    const int rows = 64;
    double *src, *dst;
    cudaMalloc(&src, rows * 64 * 8);
    cudaMalloc(&dst, rows * 64 * 8);
    double h[rows * 64];
    for (int i = 0; i < rows * 64; ++i) h[i] = i;
    cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dst, 0, sizeof h);
        probe<<<1, 128, rows * 66 * 8>>>(src, dst, rows, mode);
        cudaError_t e = cudaDeviceSynchronize();
        double g[rows * 64];
        cudaMemcpy(g, dst, sizeof g, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < rows * 64; ++i) bad += g[i] != h[i];
        printf("mode %d: %s, mismatches %d\n", mode, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
