// K5/K7/K8: the key_merge operator:
// generate two int64-key tables, hash-partition them, shuffle partitions to
// their owner rank, and inner-join each partition in shared memory.
//
// Layout: every table is two device columns (SoA, as a cuDF frame): keys
// int64[n] and payload int64[n].  One 64-bit mix h = splitmix64(key) drives
// every placement decision, from disjoint bit ranges:
//   owner rank      = mulhi32(h >> 32, P)                     (mode RANK)
//   local partition = (h & 0xffffffff) >> (32 - log2 parts)   (mode PART)
//   hash-table slot = h & (slots - 1)                          (join)
//
// Partition (K5) is histogram -> exclusive scan -> scatter with per-(bucket,
// CTA) offsets: every CTA owns one contiguous run of rows, so the output is
// bucket-major with one contiguous sub-run per CTA.  With <= 8192 buckets the
// L2 (126 MB) holds the whole write frontier, so the scattered 8-byte stores
// reach DRAM as full sectors.
//
// Join (K7): one CTA per partition builds an open-addressing table (keys +
// build row index, 16384 slots, 192 KB of shared memory) over chunks of at
// most 12288 build rows and streams the partition's probe rows through it;
// matches are emitted with warp-aggregated output reservations and folded into
// an order-independent digest (K8: row count, sum of row hashes, sum of keys,
// all mod 2^64) in the same pass.
#include <cuda_runtime.h>

#include <algorithm>

#include "m4d_internal.h"

namespace {

constexpr int kHistThreads = 512;
constexpr int kMaxBuckets = 16384;
constexpr int kJoinThreads = 1024;
constexpr int kSlots = 16384;
constexpr int kChunk = kSlots * 3 / 4;
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr size_t kJoinSmem = kSlots * (sizeof(int64_t) + sizeof(uint32_t));

__device__ __forceinline__ uint32_t bucket_of(int64_t key, int mode, int buckets, int log2b) {
    const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(key));
    if (mode == M4D_PART_RANK) return __umulhi(static_cast<uint32_t>(h >> 32), static_cast<uint32_t>(buckets));
    return log2b ? static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2b)) : 0u;
}

__device__ __forceinline__ uint64_t row_hash(int64_t k, int64_t l, int64_t r) {
    uint64_t h = m4d_splitmix64(static_cast<uint64_t>(k) ^ 0x6B65795F6D657267ull);
    h = m4d_splitmix64(h ^ static_cast<uint64_t>(l));
    return m4d_splitmix64(h ^ (static_cast<uint64_t>(r) * 0x9E3779B97F4A7C15ull));
}

__global__ void generate_kernel(int64_t* keys, int64_t* vals, int64_t row0, int64_t count, uint64_t total,
                                uint64_t seed, uint64_t band) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = static_cast<uint64_t>(row0 + i);
        keys[i] = static_cast<int64_t>(band + m4d_splitmix64(seed + g) % total);
        vals[i] = static_cast<int64_t>(g);
    }
}

// hist[b * ctas + cta] = rows of this CTA's run that fall in bucket b.
__global__ void __launch_bounds__(kHistThreads) hist_kernel(const int64_t* __restrict__ keys, int64_t n,
                                                            int64_t run, int mode, int buckets, int log2b,
                                                            uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t h[];
    for (int b = threadIdx.x; b < buckets; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
        atomicAdd(&h[bucket_of(__ldcs(keys + i), mode, buckets, log2b)], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < buckets; b += blockDim.x) hist[static_cast<int64_t>(b) * gridDim.x + blockIdx.x] = h[b];
}

// Exclusive scan of hist (bucket-major) in place: three phases over tiles.
constexpr int kScanTile = 4096;

__global__ void scan_reduce_kernel(const uint32_t* __restrict__ v, int64_t n, int64_t* __restrict__ tile_sums) {
    __shared__ int64_t part[32];
    const int64_t lo = blockIdx.x * static_cast<int64_t>(kScanTile);
    int64_t s = 0;
    for (int64_t i = lo + threadIdx.x; i < lo + kScanTile && i < n; i += blockDim.x) s += v[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
        tile_sums[blockIdx.x] = t;
    }
}

__global__ void scan_tiles_kernel(int64_t* tile_sums, int64_t tiles, int64_t* total) {
    // one warp: sequential over tiles in chunks of 32 with a warp scan
    int64_t carry = 0;
    const int lane = threadIdx.x;
    for (int64_t base = 0; base < tiles; base += 32) {
        int64_t x = base + lane < tiles ? tile_sums[base + lane] : 0;
        int64_t incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (base + lane < tiles) tile_sums[base + lane] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) *total = carry;
}

__global__ void scan_apply_kernel(const uint32_t* __restrict__ v, int64_t n, const int64_t* __restrict__ tile_sums,
                                  int64_t* __restrict__ out) {
    // 1024 threads x 4 elements = one tile; block scan with warp shuffles
    __shared__ int64_t warp_tot[32];
    const int64_t lo = blockIdx.x * static_cast<int64_t>(kScanTile);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int64_t x[4];
    int64_t local = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = lo + t * 4 + k;
        x[k] = i < n ? v[i] : 0;
        local += x[k];
    }
    int64_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int64_t w = warp_tot[lane];
        int64_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        warp_tot[lane] = wi - w;
    }
    __syncthreads();
    int64_t run = tile_sums[blockIdx.x] + warp_tot[warp] + incl - local;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = lo + t * 4 + k;
        if (i < n) out[i] = run;
        run += x[k];
    }
}

__global__ void __launch_bounds__(kHistThreads) scatter_kernel(const int64_t* __restrict__ keys,
                                                               const int64_t* __restrict__ vals, int64_t n,
                                                               int64_t run, int mode, int buckets, int log2b,
                                                               const int64_t* __restrict__ offsets,
                                                               int64_t* __restrict__ out_keys,
                                                               int64_t* __restrict__ out_vals) {
    extern __shared__ unsigned long long cursor[];
    for (int b = threadIdx.x; b < buckets; b += blockDim.x)
        cursor[b] = static_cast<unsigned long long>(offsets[static_cast<int64_t>(b) * gridDim.x + blockIdx.x]);
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const int64_t k = __ldcs(keys + i);
        const int64_t v = __ldcs(vals + i);
        const unsigned long long pos = atomicAdd(&cursor[bucket_of(k, mode, buckets, log2b)], 1ull);
        out_keys[pos] = k;
        out_vals[pos] = v;
    }
}

__global__ void bucket_bounds_kernel(const int64_t* __restrict__ offsets, int buckets, int ctas, int64_t total,
                                     int64_t* __restrict__ bounds) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= buckets; b += gridDim.x * blockDim.x)
        bounds[b] = b < buckets ? offsets[static_cast<int64_t>(b) * ctas] : total;
}

__device__ __forceinline__ void warp_emit(bool has, int64_t key, int64_t lval, int64_t rval,
                                          unsigned long long* cursor, int64_t capacity, int64_t* ok,
                                          int64_t* ol, int64_t* orr, int lane) {
    const unsigned mask = __ballot_sync(0xffffffffu, has);
    if (!mask) return;
    unsigned long long base = 0;
    const int leader = __ffs(mask) - 1;
    if (lane == leader) base = atomicAdd(cursor, static_cast<unsigned long long>(__popc(mask)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (has) {
        const unsigned long long pos = base + __popc(mask & ((1u << lane) - 1));
        if (static_cast<int64_t>(pos) < capacity) {
            ok[pos] = key;
            ol[pos] = lval;
            orr[pos] = rval;
        }
    }
}

__global__ void __launch_bounds__(kJoinThreads, 1)
    join_kernel(const int64_t* __restrict__ lk, const int64_t* __restrict__ lv, const int64_t* __restrict__ loff,
                const int64_t* __restrict__ rk, const int64_t* __restrict__ rv, const int64_t* __restrict__ roff,
                int64_t* __restrict__ ok, int64_t* __restrict__ ol, int64_t* __restrict__ orr, int64_t capacity,
                unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ digest) {
    extern __shared__ unsigned char smem[];
    int64_t* tkey = reinterpret_cast<int64_t*>(smem);
    uint32_t* tidx = reinterpret_cast<uint32_t*>(smem + kSlots * sizeof(int64_t));
    const int part = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t b0 = loff[part], b1 = loff[part + 1];
    const int64_t p0 = roff[part], p1 = roff[part + 1];
    unsigned long long cnt = 0, hsum = 0, ksum = 0;
    for (int64_t c0 = b0; c0 < b1; c0 += kChunk) {
        const int64_t c1 = c0 + kChunk < b1 ? c0 + kChunk : b1;
        for (int s = threadIdx.x; s < kSlots; s += blockDim.x) tidx[s] = kEmpty;
        __syncthreads();
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const int64_t k = lk[i];
            uint32_t s = static_cast<uint32_t>(m4d_splitmix64(static_cast<uint64_t>(k))) & (kSlots - 1);
            while (atomicCAS(&tidx[s], kEmpty, static_cast<uint32_t>(i - c0)) != kEmpty) s = (s + 1) & (kSlots - 1);
            tkey[s] = k;
        }
        __syncthreads();
        // probe: the loop trip count is uniform per warp so the emits stay converged
        for (int64_t base = p0; base < p1; base += blockDim.x) {
            const int64_t j = base + threadIdx.x;
            const bool live = j < p1;
            int64_t k = 0, r = 0;
            uint32_t s = 0;
            if (live) {
                k = rk[j];
                r = rv[j];
                s = static_cast<uint32_t>(m4d_splitmix64(static_cast<uint64_t>(k))) & (kSlots - 1);
            }
            bool walking = live;
            while (__any_sync(0xffffffffu, walking)) {
                bool hit = false;
                int64_t l = 0;
                if (walking) {
                    const uint32_t idx = tidx[s];
                    if (idx == kEmpty) {
                        walking = false;
                    } else {
                        if (tkey[s] == k) {
                            hit = true;
                            l = lv[c0 + idx];
                        }
                        s = (s + 1) & (kSlots - 1);
                    }
                }
                if (hit) {
                    ++cnt;
                    hsum += row_hash(k, l, r);
                    ksum += static_cast<unsigned long long>(k);
                }
                warp_emit(hit, k, l, r, cursor, capacity, ok, ol, orr, lane);
            }
        }
        __syncthreads();
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
    }
    if (lane == 0 && cnt) {
        atomicAdd(digest + 0, cnt);
        atomicAdd(digest + 1, hsum);
        atomicAdd(digest + 2, ksum);
    }
}

int log2_exact(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return (1 << l) == v ? l : -1;
}

}  // namespace

using m4d::fail;

extern "C" {

m4d_status m4d_merge_generate(int64_t* keys, int64_t* vals, int64_t row0, int64_t count, uint64_t total,
                              uint64_t seed, uint64_t band, void* stream) {
    if (count < 0 || total == 0) return fail(M4D_ERR_USAGE, "invalid generator range");
    if (!count) return M4D_OK;
    const int64_t grid = std::min<int64_t>((count + 255) / 256, 148 * 16);
    generate_kernel<<<static_cast<unsigned>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        keys, vals, row0, count, total, seed, band);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

static int partition_ctas(int64_t n) {
    const int64_t per = 65536;  // rows per CTA run (>= 64 rows per bucket at 1024 buckets)
    int64_t c = (n + per - 1) / per;
    if (c < 1) c = 1;
    if (c > 148 * 8) c = 148 * 8;
    return static_cast<int>(c);
}

size_t m4d_partition_scratch_bytes(int64_t n, int buckets) {
    const int64_t ctas = partition_ctas(n);
    const int64_t entries = ctas * buckets;
    const int64_t tiles = (entries + kScanTile - 1) / kScanTile;
    return entries * sizeof(uint32_t) + entries * sizeof(int64_t) + (tiles + 1) * sizeof(int64_t) + 256;
}

m4d_status m4d_partition(const int64_t* keys, const int64_t* vals, int64_t n, int mode, int buckets,
                         int64_t* out_keys, int64_t* out_vals, int64_t* bounds, void* scratch,
                         size_t scratch_bytes, void* stream) {
    if (n < 0 || buckets < 1 || buckets > kMaxBuckets) return fail(M4D_ERR_USAGE, "bucket count %d outside [1, %d]", buckets, kMaxBuckets);
    const int log2b = log2_exact(buckets);
    if (mode == M4D_PART_LOCAL && log2b < 0) return fail(M4D_ERR_USAGE, "local partition count must be a power of two");
    if (mode != M4D_PART_LOCAL && mode != M4D_PART_RANK) return fail(M4D_ERR_USAGE, "unknown partition mode %d", mode);
    if (scratch_bytes < m4d_partition_scratch_bytes(n, buckets)) return fail(M4D_ERR_USAGE, "partition scratch too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int ctas = partition_ctas(n);
    const int64_t run = (n + ctas - 1) / ctas;
    const int64_t entries = static_cast<int64_t>(ctas) * buckets;
    const int64_t tiles = (entries + kScanTile - 1) / kScanTile;
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    int64_t* offs = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + ((entries * sizeof(uint32_t) + 255) & ~size_t(255)));
    int64_t* tile_sums = offs + entries;
    int64_t* total = tile_sums + tiles;
    const size_t hist_smem = buckets * sizeof(uint32_t);
    const size_t cur_smem = buckets * sizeof(unsigned long long);
    // (per device; cheap enough to repeat on every call)
    M4D_CUDA_TRY(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 4));
    M4D_CUDA_TRY(cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 8));
    hist_kernel<<<ctas, kHistThreads, hist_smem, s>>>(keys, n, run, mode, buckets, log2b, hist);
    scan_reduce_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums);
    scan_tiles_kernel<<<1, 32, 0, s>>>(tile_sums, tiles, total);
    scan_apply_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, offs);
    scatter_kernel<<<ctas, kHistThreads, cur_smem, s>>>(keys, vals, n, run, mode, buckets, log2b, offs, out_keys, out_vals);
    bucket_bounds_kernel<<<(buckets + 256) / 256, 256, 0, s>>>(offs, buckets, ctas, n, bounds);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

int m4d_partition_launches(void) { return 6; }

m4d_status m4d_hash_join(const int64_t* lkeys, const int64_t* lvals, const int64_t* lbounds, const int64_t* rkeys,
                         const int64_t* rvals, const int64_t* rbounds, int parts, int64_t* out_keys,
                         int64_t* out_lvals, int64_t* out_rvals, int64_t capacity, unsigned long long* result,
                         void* stream) {
    if (parts < 0) return fail(M4D_ERR_USAGE, "negative partition count");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    M4D_CUDA_TRY(cudaFuncSetAttribute(join_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kJoinSmem)));
    // result = {cursor, count, hash_sum, key_sum}
    M4D_CUDA_TRY(cudaMemsetAsync(result, 0, 4 * sizeof(unsigned long long), s));
    if (parts)
        join_kernel<<<parts, kJoinThreads, kJoinSmem, s>>>(lkeys, lvals, lbounds, rkeys, rvals, rbounds, out_keys,
                                                           out_lvals, out_rvals, capacity, result, result + 1);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

}  // extern "C"
