// Probe: one-pass "tile-local" radix partition + gather join read.
//   pass: every 8192-row tile (one 1024-thread CTA) is counting-sorted by its
//         F-way partition id in shared memory and written back CONTIGUOUSLY to
//         the tile's own region of the output (sequential 128 KB stores), plus
//         the tile's per-partition start offsets (u16) in a [p/16][tile][p%16]
//         layout (one 32-byte sector per (tile, 16 partitions)).
//   gather: one CTA per partition reads its rows out of every tile (runs of
//         ~8192/F rows) -- the read pattern a join over this layout has.
// Question: do both run near HBM bandwidth at F = 4096 / 8192?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tilesort_probe tilesort_probe.cu
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

__device__ __forceinline__ uint32_t part_of(int64_t k, int log2b) {
    return static_cast<uint32_t>((mix(static_cast<uint64_t>(k)) & 0xffffffffull) >> (32 - log2b));
}

__global__ void gen(int64_t* k, int64_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        k[i] = (int64_t)(mix(0x4C454654ull + i) % (uint64_t)n);
        v[i] = i;
    }
}

constexpr int kR = 8;
constexpr int kT = 1024, kTile = kT * kR;  // gather/meta tile (1024-thread variant)

__device__ __forceinline__ int64_t meta_index(int64_t tiles, int p, int64_t t) {
    return ((int64_t)(p >> 4) * tiles + t) * 16 + (p & 15);
}

// persistent: CTA walks tiles blockIdx.x, + gridDim.x, ...  (NT threads, NT*8-row tiles)
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) tile_sort(const int64_t* __restrict__ k, const int64_t* __restrict__ v,
                                                   int64_t n, int log2b, longlong2* __restrict__ out,
                                                   uint16_t* __restrict__ meta, int64_t tiles) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int F = 1 << log2b;
    longlong2* stage = reinterpret_cast<longlong2*>(sm);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(stage + (NT * kR));
    __shared__ uint32_t wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = F / NT;  // F >= NT
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t base = t * (NT * kR);
        const int rem = (int)(n - base < (NT * kR) ? n - base : (NT * kR));
        longlong2 row[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * NT + threadIdx.x;
            if (r < rem) {
                row[u].x = __ldcs(k + base + r);
                row[u].y = __ldcs(v + base + r);
            }
        }
        for (int b = threadIdx.x; b < F; b += NT) cnt[b] = 0;
        __syncthreads();
        uint32_t b[kR], rk[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * NT + threadIdx.x;
            if (r < rem) {
                b[u] = part_of(row[u].x, log2b);
                rk[u] = atomicAdd(&cnt[b[u]], 1u);
            }
        }
        __syncthreads();
        uint32_t c[16], loc = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            c[q] = q < per ? cnt[threadIdx.x * per + q] : 0;
            loc += c[q];
        }
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
        uint32_t run0 = wsum[w] + incl - loc;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if (q < per) {
                const int p = threadIdx.x * per + q;
                cnt[p] = run0;  // now the start
                meta[meta_index(tiles, p, t)] = (uint16_t)run0;
                run0 += c[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const int r = u * NT + threadIdx.x;
            if (r < rem) stage[cnt[b[u]] + rk[u]] = row[u];
        }
        __syncthreads();
        for (int r = threadIdx.x; r < rem; r += NT) __stcs(out + base + r, stage[r]);
        __syncthreads();
    }
}


// Pipelined tile sort: 1024 threads, 4096-row tiles, keys/vals of tile t+1
// TMA-bulk-loaded into the other input buffer while tile t is ranked; rows
// are never staged, only a u16 permutation (sorted position -> tile row).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(b)), "r"(par) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr int kPT = 1024, kPR = 4, kPTile = kPT * kPR;
__global__ void __launch_bounds__(kPT, 1) tile_sort_pipe(const int64_t* __restrict__ k, const int64_t* __restrict__ v,
                                                         int64_t n, int log2b, longlong2* __restrict__ out,
                                                         uint16_t* __restrict__ meta, int64_t tiles) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int F = 1 << log2b;
    int64_t* kin = reinterpret_cast<int64_t*>(sm);           // [2][kPTile]
    int64_t* vin = kin + 2 * kPTile;                          // [2][kPTile]
    uint32_t* cnt = reinterpret_cast<uint32_t*>(vin + 2 * kPTile);  // [F]
    uint16_t* perm = reinterpret_cast<uint16_t*>(cnt + F);   // [kPTile]
    __shared__ uint64_t bar[2];
    __shared__ uint32_t wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = F / kPT;
    for (int b = threadIdx.x; b < F; b += kPT) cnt[b] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t t, int slot) {
        const int64_t base = t * kPTile;
        const int rows = (int)(n - base < kPTile ? n - base : kPTile);
        mbar_expect(&bar[slot], rows * 16);
        bulk_g2s(kin + slot * kPTile, k + base, rows * 8, &bar[slot]);
        bulk_g2s(vin + slot * kPTile, v + base, rows * 8, &bar[slot]);
    };
    int64_t t = blockIdx.x;
    if (threadIdx.x == 0 && t < tiles) issue(t, 0);
    uint32_t phase[2] = {0, 0};
    for (int it = 0; t < tiles; t += gridDim.x, ++it) {
        const int slot = it & 1;
        if (threadIdx.x == 0 && t + gridDim.x < tiles) issue(t + gridDim.x, slot ^ 1);
        const int64_t base = t * kPTile;
        const int rem = (int)(n - base < kPTile ? n - base : kPTile);
        mbar_wait(&bar[slot], phase[slot]);
        phase[slot] ^= 1;
        const int64_t* ks = kin + slot * kPTile;
        const int64_t* vs = vin + slot * kPTile;
        uint32_t b[kPR], rk[kPR];
#pragma unroll
        for (int u = 0; u < kPR; ++u) {
            const int r = u * kPT + threadIdx.x;
            if (r < rem) {
                b[u] = part_of(ks[r], log2b);
                rk[u] = atomicAdd(&cnt[b[u]], 1u);
            }
        }
        __syncthreads();
        uint32_t c[8], loc = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            c[q] = q < per ? cnt[threadIdx.x * per + q] : 0;
            loc += c[q];
        }
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
        uint32_t run0 = wsum[w] + incl - loc;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < per) {
                const int p = threadIdx.x * per + q;
                cnt[p] = run0;
                meta[meta_index(tiles, p, t)] = (uint16_t)run0;
                run0 += c[q];
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPR; ++u) {
            const int r = u * kPT + threadIdx.x;
            if (r < rem) perm[cnt[b[u]] + rk[u]] = (uint16_t)r;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kPR; ++u) {
            const int r = u * kPT + threadIdx.x;
            if (r < rem) {
                const int i = perm[r];
                longlong2 x;
                x.x = ks[i];
                x.y = vs[i];
                __stcs(out + base + r, x);
            }
        }
        for (int q = threadIdx.x; q < F; q += kPT) cnt[q] = 0;
        __syncthreads();
    }
}

// One CTA per partition: lane l of warp w reads the run of tile t (divergent simple gather).
__global__ void __launch_bounds__(1024) gather(const longlong2* __restrict__ in, const uint16_t* __restrict__ meta,
                                               int64_t n, int64_t tiles, int log2b, int kTile,
                                               unsigned long long* __restrict__ acc) {
    const int p = blockIdx.x, F = 1 << log2b;
    unsigned long long s = 0, c = 0;
    for (int64_t t = threadIdx.x; t < tiles; t += blockDim.x) {
        const int64_t base = t * kTile;
        const int rows = (int)(n - base < kTile ? n - base : kTile);
        const int a = meta[meta_index(tiles, p, t)];
        const int z = p + 1 < F ? meta[meta_index(tiles, p + 1, t)] : rows;
        for (int r = a; r < z; ++r) {
            const longlong2 x = __ldcs(in + base + r);
            s += (unsigned long long)x.y;
            ++c;
        }
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, s);
        atomicAdd(acc + 1, c);
    }
}

// Reference read: each CTA streams a contiguous 1/F slice (what a join over a bucket-major layout reads).
__global__ void __launch_bounds__(1024) stream_read(const longlong2* __restrict__ in, int64_t n,
                                                    unsigned long long* __restrict__ acc) {
    unsigned long long s = 0, c = 0;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const longlong2 x = __ldcs(in + i);
        s += (unsigned long long)x.y;
        ++c;
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, s);
        atomicAdd(acc + 1, c);
    }
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000;
    int64_t *k, *v;
    longlong2* out;
    uint16_t* meta;
    CK(cudaMalloc(&k, n * 8));
    CK(cudaMalloc(&v, n * 8));
    CK(cudaMalloc(&out, n * 16));
    CK(cudaMalloc(&meta, (size_t)(n / 4096 + 2) * 8192 * 2));
    unsigned long long* acc;
    CK(cudaMalloc(&acc, 16));
    gen<<<148 * 8, 256>>>(k, v, n);
    CK(cudaFuncSetAttribute(tile_sort<1024, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tile_sort_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tile_sort<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const unsigned long long want = (unsigned long long)(n - 1) * n / 2;
    for (int nt : {4096, 1024, 512})
    for (int log2b = 10; log2b <= 13; ++log2b) {
        const int F = 1 << log2b;
        const int tr = nt == 4096 ? kPTile : nt * kR;
        const int64_t tiles = (n + tr - 1) / tr;
        const size_t smem = nt == 4096 ? (size_t)kPTile * 32 + (size_t)F * 4 + kPTile * 2 : (size_t)tr * 16 + (size_t)F * 4;
        if (F < (nt == 4096 ? 1024 : nt) || smem > (nt == 512 ? 110 : 220) * 1024) continue;
        float tp = 0, tg = 0, tsr = 0;
        unsigned long long r[2] = {0, 0};
        for (int rep = 0; rep < 4; ++rep) {
            float a;
            cudaEventRecord(e0);
            if (nt == 4096)
                tile_sort_pipe<<<148, kPT, smem>>>(k, v, n, log2b, out, meta, tiles);
            else if (nt == 1024)
                tile_sort<1024, 1><<<148, 1024, smem>>>(k, v, n, log2b, out, meta, tiles);
            else
                tile_sort<512, 2><<<296, 512, smem>>>(k, v, n, log2b, out, meta, tiles);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            cudaEventElapsedTime(&a, e0, e1);
            if (rep) tp += a / 3;
            CK(cudaMemset(acc, 0, 16));
            cudaEventRecord(e0);
            gather<<<F, 1024>>>(out, meta, n, tiles, log2b, tr, acc);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            cudaEventElapsedTime(&a, e0, e1);
            if (rep) tg += a / 3;
            CK(cudaMemcpy(r, acc, 16, cudaMemcpyDeviceToHost));
            cudaEventRecord(e0);
            stream_read<<<F, 1024>>>(out, n, acc + 0);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&a, e0, e1);
            if (rep) tsr += a / 3;
        }
        printf("NT=%4d F=%5d  tile_sort %.3f ms (%.0f GB/s r+w)  gather %.3f ms (%.0f GB/s)  stream %.3f ms  %s\n", nt, F, tp,
               n * 32 / tp / 1e6, tg, n * 16 / tg / 1e6, tsr,
               (r[0] == want && r[1] == (unsigned long long)n) ? "ok" : "BAD");
    }
    return 0;
}
