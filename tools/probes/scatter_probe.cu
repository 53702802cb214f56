// Probe: single-pass radix scatter of 1e8 (key, payload) rows into F buckets
// (F = 256 .. 8192), SoA input -> bucket-major 16-byte pairs, with per-(bucket,
// CTA) offsets from a histogram.  Variants: tile-staged (1024 threads, 8192-row
// tiles sorted by bucket in shared memory, copied out run by run) and direct
// (one shared cursor per bucket, rows stored straight from registers).
// Question: up to which fan-out does one pass stay near HBM bandwidth?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scatter_probe scatter_probe.cu
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t bucket(int64_t k, int log2b) {
    return static_cast<uint32_t>((mix(static_cast<uint64_t>(k)) & 0xffffffffull) >> (32 - log2b));
}

__global__ void gen(int64_t* k, int64_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        k[i] = (int64_t)(mix(0x4C454654ull + i) % (uint64_t)n);
        v[i] = i;
    }
}

constexpr int kT = 1024, kR = 8, kTile = kT * kR;

// hist[b * ctas + cta]
__global__ void __launch_bounds__(kT) hist(const int64_t* __restrict__ k, int64_t n, int64_t run, int log2b,
                                           uint32_t* __restrict__ h) {
    extern __shared__ uint32_t c[];
    const int F = 1 << log2b;
    for (int b = threadIdx.x; b < F; b += kT) c[b] = 0;
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t base = lo; base < hi; base += kTile) {
        int64_t key[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int64_t i = base + u * kT + threadIdx.x;
            key[u] = i < hi ? __ldcs(k + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kR; ++u)
            if (base + u * kT + threadIdx.x < hi) atomicAdd(&c[bucket(key[u], log2b)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < F; b += kT) h[(int64_t)b * gridDim.x + blockIdx.x] = c[b];
}

// tile-staged scatter: shared layout stage[kTile] longlong2 | bk[kTile] u16 | cnt[F] | tst[F] | cur[F]
__global__ void __launch_bounds__(kT) tile_scatter(const int64_t* __restrict__ k, const int64_t* __restrict__ v,
                                                   int64_t n, int64_t run, int log2b,
                                                   const uint32_t* __restrict__ offs, longlong2* __restrict__ out,
                                                   int bulk) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int F = 1 << log2b;
    longlong2* stage = reinterpret_cast<longlong2*>(sm);
    uint16_t* bk = reinterpret_cast<uint16_t*>(stage + kTile);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(bk + kTile);
    uint32_t* tst = cnt + F;
    uint32_t* cur = tst + F;
    __shared__ uint32_t wsum[32];
    for (int b = threadIdx.x; b < F; b += kT) cur[b] = offs[(int64_t)b * gridDim.x + blockIdx.x];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = F / kT > 0 ? F / kT : 1;  // buckets per thread in the scan (F >= kT), else 1 for first F
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t base = lo; base < hi; base += kTile) {
        for (int b = threadIdx.x; b < F; b += kT) cnt[b] = 0;
        __syncthreads();
        longlong2 row[kR];
        uint32_t b[kR], rk[kR];
        const int rem = (int)(hi - base < kTile ? hi - base : kTile);
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * kT + threadIdx.x;
            if (r < rem) {
                row[u].x = __ldcs(k + base + r);
                row[u].y = __ldcs(v + base + r);
            }
        }
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * kT + threadIdx.x;
            if (r < rem) {
                b[u] = bucket(row[u].x, log2b);
                rk[u] = atomicAdd(&cnt[b[u]], 1u);
            }
        }
        __syncthreads();
        // exclusive scan of cnt -> tst (thread t owns buckets [t*per, t*per+per))
        uint32_t loc = 0;
        if (threadIdx.x * per < F)
            for (int q = 0; q < per; ++q) loc += cnt[threadIdx.x * per + q];
        uint32_t incl = loc;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            uint32_t x = wsum[lane], xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            wsum[lane] = xi - x;
        }
        __syncthreads();
        if (threadIdx.x * per < F) {
            uint32_t run0 = wsum[w] + incl - loc;
            for (int q = 0; q < per; ++q) {
                tst[threadIdx.x * per + q] = run0;
                run0 += cnt[threadIdx.x * per + q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * kT + threadIdx.x;
            if (r < rem) {
                const uint32_t p = tst[b[u]] + rk[u];
                stage[p] = row[u];
                bk[p] = (uint16_t)b[u];
            }
        }
        __syncthreads();
        for (int r = threadIdx.x; r < rem; r += kT) {
            const uint32_t bb = bk[r];
            out[cur[bb] + (r - tst[bb])] = stage[r];
        }
        __syncthreads();
        for (int q = threadIdx.x; q < F; q += kT) cur[q] += cnt[q];
    }
}

__global__ void __launch_bounds__(512) direct_scatter(const int64_t* __restrict__ k, const int64_t* __restrict__ v,
                                                      int64_t n, int64_t run, int log2b,
                                                      const uint32_t* __restrict__ offs, longlong2* __restrict__ out) {
    extern __shared__ uint32_t cur[];
    const int F = 1 << log2b;
    for (int b = threadIdx.x; b < F; b += blockDim.x) cur[b] = offs[(int64_t)b * gridDim.x + blockIdx.x];
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t base = lo; base < hi; base += (int64_t)blockDim.x * kR) {
        longlong2 row[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            if (i < hi) {
                row[u].x = __ldcs(k + i);
                row[u].y = __ldcs(v + i);
            }
        }
#pragma unroll
        for (int u = 0; u < kR; ++u)
            if (base + u * blockDim.x + threadIdx.x < hi) out[atomicAdd(&cur[bucket(row[u].x, log2b)], 1u)] = row[u];
    }
}

__global__ void check(const longlong2* out, int64_t n, const uint32_t* bounds, int log2b, unsigned long long* bad,
                      unsigned long long* vsum) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = bucket(out[i].x, log2b);
        if (i < bounds[b] || (b + 1 < (1u << log2b) && i >= bounds[b + 1])) atomicAdd(bad, 1ull);
        atomicAdd(vsum, (unsigned long long)out[i].y);
    }
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000;
    int64_t *k, *v;
    longlong2* out;
    CK(cudaMalloc(&k, n * 8));
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&out, n * 16));
    gen<<<148 * 8, 256>>>(k, v, n);
    uint32_t *h, *offs, *bounds;
    const int max_ctas = 296;
    CK(cudaMalloc(&h, (size_t)8192 * max_ctas * 4));
    CK(cudaMalloc(&offs, (size_t)8192 * max_ctas * 4));
    CK(cudaMalloc(&bounds, 8192 * 4));
    unsigned long long* dbg;
    CK(cudaMalloc(&dbg, 16));
    void* tmp = nullptr;
    size_t tmpb = 0;
    cub::DeviceScan::ExclusiveSum(tmp, tmpb, h, offs, 8192 * max_ctas);
    CK(cudaMalloc(&tmp, tmpb));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CK(cudaFuncSetAttribute(hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 4));
    CK(cudaFuncSetAttribute(direct_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 4));
    CK(cudaFuncSetAttribute(tile_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    const unsigned long long want = (unsigned long long)(n - 1) * n / 2;
    for (int log2b = 8; log2b <= 13; ++log2b) {
        const int F = 1 << log2b;
        for (int variant = 0; variant < 2; ++variant) {
            const int ctas = variant == 0 ? 148 : 296;
            const int64_t run = (n + ctas - 1) / ctas;
            const int entries = F * ctas;
            float th = 0, ts = 0;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0);
                hist<<<ctas, kT, F * 4>>>(k, n, run, log2b, h);
                cub::DeviceScan::ExclusiveSum(tmp, tmpb, h, offs, entries);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float a;
                cudaEventElapsedTime(&a, e0, e1);
                cudaEventRecord(e0);
                if (variant == 0) {
                    const size_t sm = (size_t)kTile * 18 + (size_t)F * 12;
                    if (sm > 220 * 1024) break;
                    tile_scatter<<<ctas, kT, sm>>>(k, v, n, run, log2b, offs, out, 0);
                } else {
                    direct_scatter<<<ctas, 512, F * 4>>>(k, v, n, run, log2b, offs, out);
                }
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
                float b;
                cudaEventElapsedTime(&b, e0, e1);
                if (rep) {
                    th += a / 3;
                    ts += b / 3;
                }
            }
            // bounds: offs[b * ctas]
            uint32_t* hb = (uint32_t*)malloc(entries * 4);
            CK(cudaMemcpy(hb, offs, entries * 4, cudaMemcpyDeviceToHost));
            uint32_t* bb = (uint32_t*)malloc(F * 4);
            for (int b = 0; b < F; ++b) bb[b] = hb[(int64_t)b * ctas];
            CK(cudaMemcpy(bounds, bb, F * 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(dbg, 0, 16));
            check<<<148 * 8, 256>>>(out, n, bounds, log2b, dbg, dbg + 1);
            unsigned long long r[2];
            CK(cudaMemcpy(r, dbg, 16, cudaMemcpyDeviceToHost));
            printf("F=%5d %-6s ctas=%d  hist+scan %.3f ms (%.0f GB/s keys)  scatter %.3f ms (%.0f GB/s r+w)  %s\n", F,
                   variant == 0 ? "tile" : "direct", ctas, th, n * 8 / th / 1e6, ts, n * 32 / ts / 1e6,
                   (r[0] == 0 && r[1] == want) ? "ok" : "BAD");
            free(hb);
            free(bb);
        }
    }
    return 0;
}
