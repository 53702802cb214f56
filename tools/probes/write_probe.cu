// NVLink write (push) throughput: every GPU writes into its peer at once (one
// process, all visible GPUs, peer access).  Patterns, each moving `bytes` per GPU:
//   lin    : grid-stride int4 stores, contiguous (512 B per warp instruction)
//   run R  : warps store runs of R 16-byte rows at pseudo-random 16-byte-aligned
//            offsets (the tile scatter's bucket runs; R = 16 is its average)
//   bulk R : the same runs as one TMA bulk store (cp.async.bulk s2g) per run
//   pull   : grid-stride int4 loads from the peer (reference: the read direction)
// Prints per-GPU GB/s for the peer and for the GPU's own memory.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void w_lin(int4* dst, size_t n16) {
    const int4 v = make_int4(threadIdx.x, blockIdx.x, 1, 2);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) dst[i] = v;
}

__global__ void r_lin(const int4* src, int4* sink, size_t n16) {
    int acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) acc ^= src[i].x;
    if (acc == 0x7fffffff) sink[0].x = acc;
}

// one warp per run: lanes store rows lane, lane + 32, ... of a run of R rows
__global__ void w_runs(int4* dst, size_t n16, int R) {
    const size_t runs = n16 / R;
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int4 v = make_int4(lane, 1, 2, 3);
    for (size_t r = warp; r < runs; r += warps) {
        const size_t at = mix(r) % (n16 - R);
        for (int k = lane; k < R; k += 32) dst[at + k] = v;
    }
}

__global__ void w_bulk(int4* dst, size_t n16, int R) {
    __shared__ __align__(128) int4 stage[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) stage[i] = make_int4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const size_t runs = n16 / R;
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x, T = (size_t)gridDim.x * blockDim.x;
    int k = 0;
    for (size_t r = t; r < runs; r += T) {
        const size_t at = mix(r) % (n16 - R);
        const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(stage + ((threadIdx.x * 4) & 1023)));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + at), "r"(s), "r"(R * 16) : "memory");
        if (++k == 8) {
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
            k = 0;
        }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    int G = 0;
    CK(cudaGetDeviceCount(&G));
    if (G < 2) { printf("need 2 GPUs\n"); return 1; }
    G = 2;
    const size_t bytes = size_t(1) << 30, n16 = bytes / 16;
    std::vector<int4*> buf(G), sink(G);
    std::vector<cudaStream_t> st(G);
    std::vector<cudaEvent_t> a(G), b(G);
    for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMalloc(&buf[g], bytes + 4096));
        CK(cudaMalloc(&sink[g], bytes + 4096));
        CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
        CK(cudaEventCreate(&a[g]));
        CK(cudaEventCreate(&b[g]));
        for (int p = 0; p < G; ++p)
            if (p != g) CK(cudaDeviceEnablePeerAccess(p, 0));
    }
    struct Case { const char* name; int kind; int R; };
    const Case cases[] = {{"lin", 0, 0}, {"run 8", 1, 8}, {"run 16", 1, 16}, {"run 64", 1, 64}, {"bulk 16", 2, 16},
                          {"bulk 64", 2, 64}, {"bulk 256", 2, 256}, {"pull", 3, 0}};
    for (int remote = 1; remote >= 0; --remote) {
        for (const Case& c : cases) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                for (int g = 0; g < G; ++g) {
                    CK(cudaSetDevice(g));
                    int4* target = remote ? buf[(g + 1) % G] : buf[g];
                    CK(cudaEventRecord(a[g], st[g]));
                    const int grid = 148 * 4;
                    if (c.kind == 0) w_lin<<<grid, 256, 0, st[g]>>>(target, n16);
                    else if (c.kind == 1) w_runs<<<grid, 256, 0, st[g]>>>(target, n16, c.R);
                    else if (c.kind == 2) w_bulk<<<grid, 256, 0, st[g]>>>(target, n16, c.R);
                    else r_lin<<<grid, 256, 0, st[g]>>>(target, sink[g], n16);
                    CK(cudaEventRecord(b[g], st[g]));
                }
                float worst = 0;
                for (int g = 0; g < G; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaEventSynchronize(b[g]));
                    float ms = 0;
                    CK(cudaEventElapsedTime(&ms, a[g], b[g]));
                    worst = ms > worst ? ms : worst;
                }
                best = worst < best ? worst : best;
            }
            printf("%-6s %-9s %8.1f GB/s per GPU (%.3f ms for %.2f GB)\n", remote ? "peer" : "local", c.name,
                   bytes / best / 1e6, best, bytes / 1e9);
        }
    }
    return 0;
}
