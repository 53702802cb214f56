// NVLink mesh read throughput: every GPU pulls from its peers at once (one
// process, all visible GPUs, peer access), linear int4 streams vs 64x64-fp64
// tiles with a 16000-byte row pitch (the transpose_sum partner-tile pattern).
// Prints per-GPU aggregate GB/s for: all peers, one peer (pairs), and local.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

struct Srcs { const int4* p[8]; int n; };

// linear: grid-stride over `bytes` of each source, split evenly over sources
__global__ void pull_linear(Srcs s, int4* dst, size_t n16) {
    const int src = blockIdx.x % s.n;
    const size_t cta = blockIdx.x / s.n, ctas = gridDim.x / s.n;
    for (size_t i = cta * blockDim.x + threadIdx.x; i < n16; i += ctas * blockDim.x) dst[i] = s.p[src][i];
}

// tiles: one warp-group (256 threads) per 64x64 fp64 tile of a 2000-wide row-major block
__global__ void pull_tiles(Srcs s, double* dst, int tiles_per_src, int pitch) {
    const int src = blockIdx.x % s.n;
    const double* base = reinterpret_cast<const double*>(s.p[src]);
    for (int t = blockIdx.x / s.n; t < tiles_per_src; t += gridDim.x / s.n) {
        const int tr = t / 31, tc = t % 31;  // 31x31 tiles of 64 in a 2000x2000 block (block-local)
        const int blk = t / (31 * 31);
        const double* b = base + (size_t)blk * 2000 * 2000;
        double acc = 0;
        for (int r = threadIdx.x / 16; r < 64; r += blockDim.x / 16) {
            const double2 v = *reinterpret_cast<const double2*>(b + (size_t)(tr % 31 * 64 + r) * pitch + tc * 64 + (threadIdx.x % 16) * 4);
            const double2 w = *reinterpret_cast<const double2*>(b + (size_t)(tr % 31 * 64 + r) * pitch + tc * 64 + (threadIdx.x % 16) * 4 + 2);
            acc += v.x + v.y + w.x + w.y;
        }
        if (acc == 12345.0) dst[0] = acc;  // keep the loads
    }
}

// push: every GPU stores its own buffer into each peer's out buffer (its own region
// there), grid split evenly over destinations -- the write-side mirror of pull_linear
__global__ void push_linear(Srcs d, const int4* src, size_t n16, int self_slot) {
    const int dst = blockIdx.x % d.n;
    const size_t cta = blockIdx.x / d.n, ctas = gridDim.x / d.n;
    int4* out = const_cast<int4*>(d.p[dst]) + (size_t)self_slot * n16;
    for (size_t i = cta * blockDim.x + threadIdx.x; i < n16; i += ctas * blockDim.x) out[i] = src[i];
}

int main() {
    int G = 0;
    CK(cudaGetDeviceCount(&G));
    if (G > 8) G = 8;
    const size_t bytes = (size_t)1 << 30;  // per source buffer
    std::vector<int4*> buf(G), out(G);
    for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaMalloc(&buf[d], bytes));
        CK(cudaMemset(buf[d], 1, bytes));
        CK(cudaMalloc(&out[d], bytes));
        for (int q = 0; q < G; ++q) if (q != d) cudaDeviceEnablePeerAccess(q, 0);
    }
    const int tiles = (int)(bytes / (2000 * 2000 * 8)) * 31 * 31;
    for (int mode = 0; mode < 8; ++mode) {
        const char* names[] = {"linear all-peers", "linear one-peer", "linear local", "tiles all-peers", "tiles one-peer",
                               "tiles local", "push all-peers", "push one-peer"};
        std::vector<cudaEvent_t> a(G), b(G);
        for (int rep = 0; rep < 2; ++rep) {
            for (int d = 0; d < G; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            for (int d = 0; d < G; ++d) {
                CK(cudaSetDevice(d));
                cudaEventCreate(&a[d]); cudaEventCreate(&b[d]);
                Srcs s{}; s.n = 0;
                const int kind = mode >= 6 ? (mode == 6 ? 0 : 1) : mode % 3;
                if (mode >= 6) {  // destinations: the peers' out buffers
                    if (kind == 0) { for (int q = 0; q < G; ++q) if (q != d) s.p[s.n++] = out[q]; }
                    else { s.p[s.n++] = out[d ^ 1]; }
                } else if (kind == 0) { for (int q = 0; q < G; ++q) if (q != d) s.p[s.n++] = buf[q]; }
                else if (kind == 1) { s.p[s.n++] = buf[d ^ 1]; }
                else { s.p[s.n++] = buf[d]; }
                const int grid = 296 / s.n * s.n;
                cudaEventRecord(a[d]);
                for (int k = 0; k < 4; ++k) {
                    if (mode >= 6) push_linear<<<grid, 512>>>(s, buf[d], bytes / 16 / G, d);
                    else if (mode < 3) pull_linear<<<grid, 512>>>(s, out[d], bytes / 16 / s.n);
                    else pull_tiles<<<grid, 256>>>(s, reinterpret_cast<double*>(out[d]), tiles / s.n, 2000);
                }
                cudaEventRecord(b[d]);
            }
            double worst = 1e30, sum = 0;
            for (int d = 0; d < G; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventSynchronize(b[d]));
                float ms; cudaEventElapsedTime(&ms, a[d], b[d]);
                const double moved = mode >= 6 ? 4.0 * (bytes / 16 / G) * 16 * (mode == 6 ? G - 1 : 1)
                                   : mode < 3 ? 4.0 * (bytes / 16 / (mode % 3 == 0 ? G - 1 : 1)) * 16 * (mode % 3 == 0 ? G - 1 : 1)
                                              : 4.0 * (tiles / (mode % 3 == 0 ? G - 1 : 1)) * (mode % 3 == 0 ? G - 1 : 1) * 64.0 * 64 * 8;
                const double gbs = moved / (ms * 1e-3) / 1e9;
                worst = gbs < worst ? gbs : worst; sum += gbs;
            }
            if (rep) printf("G=%d %-18s per-GPU min %7.1f GB/s  mean %7.1f GB/s\n", G, names[mode], worst, sum / G);
        }
    }
    return 0;
}
