// Empirical mbarrier parity semantics on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2101_08878_b200/csrc/ptx.cuh"

__device__ void spin(long long cycles) { long long t0 = clock64(); while (clock64() - t0 < cycles) {} }

__global__ void probe(int* out) {
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int data[2];
    if (threadIdx.x == 0) {
        m4d::ptx::mbar_init(&bar[0], 1);
        m4d::ptx::mbar_init(&bar[1], 1);
        data[0] = data[1] = 0;
        m4d::ptx::fence_mbar_init();
    }
    __syncthreads();
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 1) {
        if (lane == 0) {
            // fresh barrier: parity 1 should pass at once
            long long t0 = clock64();
            m4d::ptx::mbar_wait(&bar[1], 1);
            out[0] = (int)(clock64() - t0);
            spin(2000000);
            data[0] = 42;
            __threadfence_block();
            m4d::ptx::mbar_arrive(&bar[0]);
            spin(2000000);
            data[1] = 43;
            __threadfence_block();
            m4d::ptx::mbar_arrive(&bar[0]);  // second phase
        }
    } else if (warp == 0) {
        long long t0 = clock64();
        m4d::ptx::mbar_wait(&bar[0], 0);
        long long t1 = clock64();
        int d0 = data[0];
        m4d::ptx::mbar_wait(&bar[0], 1);
        long long t2 = clock64();
        int d1 = data[1];
        if (lane == 0) { out[1] = (int)(t1 - t0); out[2] = d0; out[3] = (int)(t2 - t1); out[4] = d1; }
    }
}

int main() {
    int* out; cudaMallocManaged(&out, 64);
    probe<<<1, 64>>>(out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s: fresh parity-1 wait %d cyc; parity-0 wait %d cyc -> data %d; parity-1 wait %d cyc -> data %d\n",
           cudaGetErrorString(e), out[0], out[1], out[2], out[3], out[4]);
    return 0;
}
