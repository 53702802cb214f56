// K5/K7/K8: the key_merge operator:
// generate two int64-key tables, hash-partition them, shuffle partitions to
// their owner rank, and inner-join each partition in shared memory.
//
// Layout: every table is two device columns (SoA, as a cuDF frame): keys
// int64[n] and payload int64[n].  One 64-bit mix h = splitmix64(key) drives
// every placement decision, from disjoint bit ranges:
//   owner rank      = mulhi32(h >> 32, P)                     (mode RANK)
//   local partition = (h & 0xffffffff) >> (32 - log2 parts)   (mode PART)
//   hash-table slot = 13-bit multiplicative hash of the folded key (join)
//
// Partition (K5) is histogram -> exclusive scan -> scatter with per-(bucket,
// CTA) offsets: every CTA owns one contiguous run of rows, so the output is
// bucket-major with one contiguous sub-run per CTA.  Partitioned rows are
// written as 16-byte (key, payload) pairs, one store per row: with at most
// 2 x 148 resident CTAs the write frontier (CTAs x buckets x one 32-byte
// sector) stays inside the 126 MB L2 even at 16384 buckets, so the scattered
// stores leave L2 as full sectors instead of DRAM read-modify-writes.
//
// Join (K7): one CTA per partition builds an open-addressing table (keys +
// build row index, 16384 slots, 192 KB of shared memory) over chunks of at
// most 12288 build rows and streams the partition's probe rows through it
// twice: a counting walk (block scan -> one output reservation per CTA), then
// an emitting walk that writes (key, lval, rval) rows and folds them into an
// order-independent digest (K8: row count, sum of row hashes, sum of keys,
// all mod 2^64, reduced per CTA before one atomic each).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "m4d_internal.h"
#include "ptx.cuh"

namespace {

constexpr int kHistThreads = 512;
constexpr int kRowsPerThread = 8;        // rows each thread loads before using any (memory-level parallelism)
constexpr int kMaxBuckets = 16384;       // single-pass partition limit (shared-memory counters)
constexpr int kMaxParts = 1 << 16;       // two-pass LOCAL partition limit (128 KB of 16-bit counters)
constexpr int kSinglePassMax = 256;      // LOCAL above this: two passes (L2 write frontier)
constexpr int kMaxGroups = 8;            // pass-2 CTA groups per segment (per-group histograms)
constexpr int kPass2Groups = 8;  // measured: pass 2 0.88 -> 0.81 ms at 1e8 rows (tools/km_pass2_groups.sh)
constexpr int kJoinThreads = 1024;
constexpr int kSlotBits = 14;                 // 16384 chain heads
constexpr int kSlots = 1 << kSlotBits;
constexpr int kChunk = 13000;                 // build rows per table (keys + links in shared memory)
constexpr int kIdxBits = 14;                  // build row index within a chunk
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr uint16_t kNil = 0xffffu;
constexpr int kStage = 256;  // staged matches per warp per emit round
constexpr int kJoinPer = 3;   // probe / build rows per thread per batch (3072; join 1.506 ms vs 1.524 at 4, 1.576 at 2)
constexpr size_t kJoinSmem = kSlots * sizeof(uint32_t) + kChunk * (sizeof(int64_t) + sizeof(uint16_t)) +
                             (kJoinThreads / 32) * kStage * sizeof(uint32_t);
static_assert(kChunk < (1 << kIdxBits) && kIdxBits + 12 <= 32 && kJoinThreads * kJoinPer <= (1 << 12),
              "stage entry packing");
static_assert(kJoinSmem <= 227 * 1024, "join shared memory");
// Join variant "small" (M4D_JOIN=small): two 512-thread CTAs per SM, each with
// half the table (8192 heads, 6500-row chunks), for ~6K-row partitions.  Twice
// the resident warps make the join itself faster (1.74 -> 1.61 ms at 1e8
// rows/side) but the 16384 partitions it needs slow pass 2 more (partition
// 3.69 -> 3.95 ms): merge step 5.48 -> 5.60 ms, so "big" stays the default.
constexpr int kSmallThreads = 512;
constexpr int kSmallSlotBits = 13;
constexpr int kSmallChunk = 6500;
constexpr int kSmallStage = 128;
constexpr size_t kSmallSmem = (1 << kSmallSlotBits) * sizeof(uint32_t) + kSmallChunk * (sizeof(int64_t) + sizeof(uint16_t)) +
                              (kSmallThreads / 32) * kSmallStage * sizeof(uint32_t);
static_assert(2 * (kSmallSmem + 1024) <= 228 * 1024, "two small join CTAs per SM");

// mode LOCAL: log2b bits of the low word; RANK: owner of `buckets` ranks;
// OWNER_COARSE: owner of buckets >> log2b ranks, then log2b low-word bits.
__device__ __forceinline__ uint32_t bucket_of(int64_t key, int mode, int buckets, int log2b) {
    const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(key));
    const uint32_t low = log2b ? static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2b)) : 0u;
    if (mode == M4D_PART_RANK) return __umulhi(static_cast<uint32_t>(h >> 32), static_cast<uint32_t>(buckets));
    if (mode == M4D_PART_OWNER_COARSE)
        return __umulhi(static_cast<uint32_t>(h >> 32), static_cast<uint32_t>(buckets >> log2b)) << log2b | low;
    return low;
}

// Shared-table slot: a 32-bit multiplicative hash of the folded key (cheap;
// independent of the partition bits, which come from splitmix64).
template <int kBits = kSlotBits>
__device__ __forceinline__ uint32_t slot_of(int64_t k) {
    const uint32_t x = static_cast<uint32_t>(k) ^ static_cast<uint32_t>(static_cast<uint64_t>(k) >> 32);
    return (x * 0x9E3779B1u) >> (32 - kBits);
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

// L2 bulk prefetch of elements [a, min(a + count, end)) of an array (16-byte
// aligned pieces only; a no-op on anything else).
template <typename T>
__device__ __forceinline__ void l2_prefetch(const T* p, int64_t a, int64_t count, int64_t end) {
    const int64_t z = a + count < end ? a + count : end;
    if (z <= a) return;
    const uint32_t b = static_cast<uint32_t>((static_cast<uint64_t>(z - a) * sizeof(T)) & ~uint64_t(15));
    if (b && (reinterpret_cast<uintptr_t>(p + a) & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + a), "r"(b) : "memory");
}

// Key of row i: SoA input (vals != null) or 16-byte (key, payload) pairs.
__device__ __forceinline__ int64_t key_at(const int64_t* keys, const int64_t* vals, int64_t i) {
    return vals ? __ldcs(keys + i) : __ldcs(keys + 2 * i);
}

// Calls fn(key) for every row of [lo, hi), spread over the CTA, kRowsPerThread
// loads in flight per thread.  A 16-byte aligned SoA key column is read two keys
// per load (an odd first / last row on its own); pf: thread 0 prefetches the next
// chunk into L2.  For the counting passes, which need only the keys.
template <typename Fn>
__device__ __forceinline__ void for_each_key(const int64_t* __restrict__ keys, const int64_t* __restrict__ vals,
                                             int64_t lo, int64_t hi, bool pf, Fn fn) {
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kRowsPerThread;
    if (vals && (reinterpret_cast<uintptr_t>(keys) & 15) == 0) {
        int64_t a = lo, z = hi;
        if (a < z && (a & 1)) {
            if (threadIdx.x == 0) fn(__ldcs(keys + a));
            ++a;
        }
        if (a < z && ((z - a) & 1)) {
            if (threadIdx.x == 0) fn(__ldcs(keys + z - 1));
            --z;
        }
        const longlong2* kp = reinterpret_cast<const longlong2*>(keys + a);
        const int64_t np = (z - a) / 2;
        if (pf && threadIdx.x == 0) l2_prefetch(keys, a, 2 * chunk, z);
        for (int64_t pb = 0; pb < np; pb += chunk) {
            if (pf && threadIdx.x == 0) l2_prefetch(keys, a + 2 * (pb + chunk), 2 * chunk, z);
            longlong2 v[kRowsPerThread];
#pragma unroll
            for (int u = 0; u < kRowsPerThread; ++u) {
                const int64_t i = pb + u * blockDim.x + threadIdx.x;
                v[u] = i < np ? __ldcs(kp + i) : make_longlong2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < kRowsPerThread; ++u)
                if (pb + u * blockDim.x + threadIdx.x < np) {
                    fn(v[u].x);
                    fn(v[u].y);
                }
        }
        return;
    }
    auto prefetch = [&](int64_t a) {  // keys only: a SoA key column, or the pairs
        if (vals) l2_prefetch(keys, a, chunk, hi);
        else l2_prefetch(reinterpret_cast<const longlong2*>(keys), a, chunk, hi);
    };
    if (pf && threadIdx.x == 0) prefetch(lo);
    for (int64_t base = lo; base < hi; base += chunk) {
        if (pf && threadIdx.x == 0) prefetch(base + chunk);
        int64_t k[kRowsPerThread];
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            k[u] = i < hi ? key_at(keys, vals, i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u)
            if (base + u * blockDim.x + threadIdx.x < hi) fn(k[u]);
    }
}

// hist[b * ctas + cta] = rows of scatter CTA cta's run that fall in bucket b.
// `split` histogram CTAs share one scatter run (grid = ctas * split, so a
// grid sized for 1024-thread scatter CTAs still fills every SM); with
// split > 1 they add into a zeroed hist.
__global__ void __launch_bounds__(kHistThreads) hist_kernel(const int64_t* __restrict__ keys,
                                                            const int64_t* __restrict__ vals, int64_t n,
                                                            int64_t run, int mode, int buckets, int log2b,
                                                            int split, uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t h[];
    for (int b = threadIdx.x; b < buckets; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const int cta = blockIdx.x / split, part = blockIdx.x % split, ctas = gridDim.x / split;
    const int64_t r0 = cta * run, r1 = r0 + run < n ? r0 + run : n;
    const int64_t len = r1 > r0 ? r1 - r0 : 0;
    const int64_t lo = r0 + len * part / split, hi = r0 + len * (part + 1) / split;
    for_each_key(keys, vals, lo, hi, false,
                 [&](int64_t key) { atomicAdd(&h[bucket_of(key, mode, buckets, log2b)], 1u); });
    __syncthreads();
    for (int b = threadIdx.x; b < buckets; b += blockDim.x) {
        uint32_t* dst = hist + static_cast<int64_t>(b) * ctas + cta;
        if (split == 1)
            *dst = h[b];
        else if (h[b])
            atomicAdd(dst, h[b]);
    }
}

// Exclusive scan of hist (bucket-major) in place: three phases over tiles.
constexpr int kScanTile = 4096;

// gate (all three): a scan launched for the exact fallback of a speculative pass 1
// returns at once unless *gate is set.
__global__ void scan_reduce_kernel(const uint32_t* __restrict__ v, int64_t n, int64_t* __restrict__ tile_sums,
                                   const int* __restrict__ gate) {
    if (gate && !*gate) return;
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

__global__ void scan_tiles_kernel(int64_t* tile_sums, int64_t tiles, int64_t* total, const int* __restrict__ gate) {
    if (gate && !*gate) return;
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
                                  int64_t* __restrict__ out, const int* __restrict__ gate) {
    if (gate && !*gate) return;
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
                                                               longlong2* __restrict__ out) {
    extern __shared__ uint32_t cursor[];  // row positions fit 32 bits (n < 2^32, checked by the host)
    for (int b = threadIdx.x; b < buckets; b += blockDim.x)
        cursor[b] = static_cast<uint32_t>(offsets[static_cast<int64_t>(b) * gridDim.x + blockIdx.x]);
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    for (int64_t base = lo; base < hi; base += static_cast<int64_t>(blockDim.x) * kRowsPerThread) {
        longlong2 row[kRowsPerThread];
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            if (i < hi) {
                if (vals) {
                    row[u].x = __ldcs(keys + i);
                    row[u].y = __ldcs(vals + i);
                } else {
                    row[u] = __ldcs(reinterpret_cast<const longlong2*>(keys) + i);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u)
            if (base + u * blockDim.x + threadIdx.x < hi)
                out[atomicAdd(&cursor[bucket_of(row[u].x, mode, buckets, log2b)], 1u)] = row[u];
    }
}

// Tile-sorted scatter for <= 256 buckets.  Each CTA stages a tile of
// kT x 8 rows in shared memory ordered by bucket (each warp ranks its rows
// per bucket: shared atomics on the warp's own counters by default, or a
// ballot multisplit that keeps input order), then copies each bucket's run of
// the tile to its global position, so every global store belongs to a
// contiguous run and DRAM sees full sectors.
constexpr int kTileBuckets = 256;
template <int kT>
constexpr size_t tile_smem() { return kT * kRowsPerThread * (sizeof(longlong2) + 1) + (kT / 32) * kTileBuckets * 2; }

// Tile scatter, steps 1-2 for one warp: load its rows of the tile and rank each
// row among the warp's rows of the same bucket (peers found with one ballot per
// bucket bit, cheaper than MATCH.ANY's serialised match); the leader of each
// peer group advances the warp's bucket counter wb[b].  kFull: all rows of the
// tile exist; kBits: compile-time bucket bits (0 = nbits at run time).
template <bool kFull, int kBits>
__device__ __forceinline__ void load_and_rank(const int64_t* __restrict__ keys, const int64_t* __restrict__ vals,
                                              int64_t tile, int rem, int w, int lane, int mode, int buckets, int log2b,
                                              int nbits, uint16_t* wb, longlong2 (&row)[kRowsPerThread],
                                              uint32_t (&bk)[kRowsPerThread], uint16_t (&off)[kRowsPerThread]) {
    const unsigned lower = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
        const int r = w * 256 + u * 32 + lane;
        if (kFull || r < rem) {
            const int64_t i = tile + r;
            if (vals) {
                row[u].x = __ldcs(keys + i);
                row[u].y = __ldcs(vals + i);
            } else {
                row[u] = __ldcs(reinterpret_cast<const longlong2*>(keys) + i);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
        const bool live = kFull || w * 256 + u * 32 + lane < rem;
        bk[u] = live ? bucket_of(row[u].x, mode, buckets, log2b) : 0xffffffffu;
        unsigned peers = 0xffffffffu;
        if (!kFull) {
            peers = __ballot_sync(0xffffffffu, live);
            peers = live ? peers : ~peers;
        }
#pragma unroll
        for (int bit = 0; bit < 8; ++bit) {  // buckets <= 256
            if (kBits ? bit < kBits : bit < nbits) {
                const unsigned v = __ballot_sync(0xffffffffu, (bk[u] >> bit) & 1u);
                peers &= (bk[u] >> bit) & 1u ? v : ~v;
            }
        }
        const int leader = __ffs(peers) - 1;
        uint32_t start = 0;
        if (live && lane == leader) {
            start = wb[bk[u]];
            wb[bk[u]] = static_cast<uint16_t>(start + __popc(peers));
        }
        start = __shfl_sync(0xffffffffu, start, leader);
        off[u] = static_cast<uint16_t>(start + __popc(peers & lower));
        __syncwarp();
    }
}

// Atomic variant of load_and_rank: each row takes its rank with one shared-memory
// atomicAdd on the warp's own counter wb[b] (conflicts only among the warp's
// lanes), instead of 8 ballots + leader election.  Rows of one warp that share a
// bucket are ordered by the hardware's atomic serialisation, so the order inside
// a partition is not tied to input order (the join's result is a multiset).
// Full-id counts of the speculative pass 1 (kSpec): 16-bit shared counters, two per
// word; the increment that takes one to 0x8000 moves 0x8000 to the global count.
struct FullCounts {
    uint32_t* smem;                 // ids / 2 words
    unsigned long long* global;     // this CTA's group row of the per-group full-id histogram, or
    uint32_t* global32;             // (push) the sender's per-(owner, local partition) counts
    int shift;                      // 32 - log2 of the local partition count
};

__device__ __forceinline__ void count_id(const FullCounts& fc, uint32_t id) {
    const uint32_t sh = (id & 1u) * 16u;
    const uint32_t old = atomicAdd(&fc.smem[id >> 1], 1u << sh);
    if (((old >> sh) & 0xffffu) == 0x7fffu) {
        atomicSub(&fc.smem[id >> 1], 0x8000u << sh);
        if (fc.global32) atomicAdd(fc.global32 + id, 0x8000u);
        else atomicAdd(fc.global + id, 0x8000ull);
    }
}

__device__ __forceinline__ void count_full(const FullCounts& fc, uint32_t low) { count_id(fc, low >> fc.shift); }

template <bool kFull, bool kSpec = false, bool kFine = false>
__device__ __forceinline__ void load_and_rank_atomic(const int64_t* __restrict__ keys, const int64_t* __restrict__ vals,
                                                     int64_t tile, int rem, int w, int lane, int mode, int buckets,
                                                     int log2b, uint16_t* wb, longlong2 (&row)[kRowsPerThread],
                                                     uint32_t (&bk)[kRowsPerThread], uint16_t (&off)[kRowsPerThread],
                                                     const FullCounts& fc = FullCounts{}) {
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
        const int r = w * 256 + u * 32 + lane;
        if (kFull || r < rem) {
            const int64_t i = tile + r;
            if (vals) {
                row[u].x = __ldcs(keys + i);
                row[u].y = __ldcs(vals + i);
            } else {
                row[u] = __ldcs(reinterpret_cast<const longlong2*>(keys) + i);
            }
        }
    }
    uint32_t* wb32 = reinterpret_cast<uint32_t*>(wb);  // 16-bit counters, two per word
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u) {
        const bool live = kFull || w * 256 + u * 32 + lane < rem;
        if (kSpec) {  // mode LOCAL: the top log2b bits of the hash's low word, and the full id
            const uint32_t low = live ? static_cast<uint32_t>(m4d_splitmix64(static_cast<uint64_t>(row[u].x))) : 0u;
            bk[u] = live ? low >> (32 - log2b) : 0xffffffffu;
            if (live) count_full(fc, low);
        } else if (kFine) {  // mode OWNER_COARSE (bucket_of), and the (owner, local partition) id
            const uint64_t h = live ? m4d_splitmix64(static_cast<uint64_t>(row[u].x)) : 0ull;
            const uint32_t low = static_cast<uint32_t>(h);
            const uint32_t owner = __umulhi(static_cast<uint32_t>(h >> 32), static_cast<uint32_t>(buckets >> log2b));
            bk[u] = live ? owner << log2b | (log2b ? low >> (32 - log2b) : 0u) : 0xffffffffu;
            if (live) count_id(fc, owner << (32 - fc.shift) | low >> fc.shift);
        } else {
            bk[u] = live ? bucket_of(row[u].x, mode, buckets, log2b) : 0xffffffffu;
        }
        if (live) {
            const uint32_t sh = (bk[u] & 1u) * 16u;
            off[u] = static_cast<uint16_t>(atomicAdd(&wb32[bk[u] >> 1], 1u << sh) >> sh);
        }
    }
    __syncwarp();
}

// Push targets of the fused owner scatter + shuffle: owner d's rows go to
// seg[d] (its receive buffer, a CUDA-IPC mapping when d is a peer B200),
// bucket (d, c) at the same offset it has inside d's segment of the local
// bucket-major order.
constexpr int kMaxPushOwners = 64;
struct PushTargets {
    longlong2* seg[kMaxPushOwners];
};

// L2 bulk prefetch of rows [r0, min(r0 + rows, hi)) of SoA columns (or 16-byte pairs).
__device__ __forceinline__ void l2_prefetch_rows(const int64_t* keys, const int64_t* vals, int64_t r0, int64_t hi,
                                                 int rows) {
    const int64_t r1 = r0 + rows < hi ? r0 + rows : hi;
    if (r1 <= r0) return;
    auto pf = [](const void* p, uint64_t bytes) {
        const uint32_t b = static_cast<uint32_t>(bytes & ~uint64_t(15));
        if (b && (reinterpret_cast<uintptr_t>(p) & 15) == 0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(b) : "memory");
    };
    if (vals) {
        pf(keys + r0, static_cast<uint64_t>(r1 - r0) * 8);
        pf(vals + r0, static_cast<uint64_t>(r1 - r0) * 8);
    } else {
        pf(keys + 2 * r0, static_cast<uint64_t>(r1 - r0) * 16);
    }
}

// Speculative pass 1 of the two-pass LOCAL partition (kSpec), and the gate of
// its exact fallback.  kSpec: no histogram pass ran before; CTA c writes bucket
// b's rows into its own region of `cap` rows at (b * ctas + c) * cap, counts
// every row by its full partition id (per-group histogram for pass 2), writes
// its exact per-bucket counts to counts[b * ctas + c] (the layout the
// histogram pass produces), and raises *overflow if any region would take more
// than cap rows (rows past cap are not stored).  gate: a kernel launched as the
// exact fallback returns at once unless *gate is set.
struct SpecArgs {
    int64_t cap = 0;
    int log2full = 0;
    int groups = 1;
    unsigned long long* hist_grp = nullptr;  // [groups][1 << log2full]
    uint32_t* counts = nullptr;              // [buckets][ctas]
    int* overflow = nullptr;
    const int* gate = nullptr;
    uint32_t* fine_out = nullptr;  // kFine (push): [world][1 << log2full] counts of this sender's rows, + a
                                   // completion counter word
    int fine_ids = 0;              // world << log2full
    uint32_t* fine_dst[kMaxPushOwners] = {};  // kFine: where owner d takes this sender's row of counts (or null)
};

template <int kT, bool kPush, bool kBulk, bool kSpec = false, bool kFine = false>
__global__ void __launch_bounds__(kT, (kT >= 1024 ? 1 : kT >= 512 ? 2 : 4)) tile_scatter_kernel(const int64_t* __restrict__ keys,
                                                                       const int64_t* __restrict__ vals, int64_t n,
                                                                       int64_t run, int mode, int buckets, int log2b,
                                                                       const int64_t* __restrict__ offsets,
                                                                       longlong2* __restrict__ out,
                                                                       const __grid_constant__ PushTargets push,
                                                                       bool atomic_rank, int tile_prefetch,
                                                                       const SpecArgs spec) {
    if (spec.gate && !*spec.gate) return;  // exact fallback of a speculative pass 1 that did not overflow
    constexpr int kTileRows = kT * kRowsPerThread;
    extern __shared__ __align__(16) unsigned char tsm[];
    longlong2* stage = reinterpret_cast<longlong2*>(tsm);
    uint8_t* sbucket = tsm + kTileRows * sizeof(longlong2);
    uint16_t* wbase = reinterpret_cast<uint16_t*>(sbucket + kTileRows);  // [warps][256]
    __shared__ uint32_t gcur[kTileBuckets];
    __shared__ uint32_t tstart[kTileBuckets + 1];
    __shared__ uint32_t dbase[kTileBuckets];  // global row of a tile row r in bucket b: dbase[b] + r
    __shared__ uint32_t scan_tmp[kTileBuckets / 32];
    __shared__ uint32_t lim[kSpec ? kTileBuckets : 1];  // kSpec: end of bucket b's region
    constexpr int kW = kT / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int nbits = 0;
    while ((1 << nbits) < buckets) ++nbits;
    FullCounts fc{};
    if (kSpec) {
        fc.smem = reinterpret_cast<uint32_t*>(wbase + kW * kTileBuckets);
        fc.global = spec.hist_grp + (static_cast<int64_t>(blockIdx.x) * spec.groups / gridDim.x << spec.log2full);
        fc.shift = 32 - spec.log2full;
        for (int i = threadIdx.x; i < (1 << spec.log2full) / 2; i += blockDim.x) fc.smem[i] = 0;
    }
    if (kFine) {  // the push also counts its rows per (owner, local partition): the owners' split needs no histogram
        fc.smem = reinterpret_cast<uint32_t*>(wbase + kW * kTileBuckets);
        fc.global32 = spec.fine_out;
        fc.shift = 32 - spec.log2full;
        for (int i = threadIdx.x; i < spec.fine_ids / 2; i += blockDim.x) fc.smem[i] = 0;
    }
    for (int b = threadIdx.x; b < kTileBuckets; b += blockDim.x) {
        if (kSpec) {
            const uint32_t r0 = static_cast<uint32_t>((static_cast<int64_t>(b) * gridDim.x + blockIdx.x) * spec.cap);
            gcur[b] = b < buckets ? r0 : 0u;
            lim[b] = b < buckets ? r0 + static_cast<uint32_t>(spec.cap) : 0u;
        } else {
            gcur[b] = b < buckets ? static_cast<uint32_t>(offsets[static_cast<int64_t>(b) * gridDim.x + blockIdx.x]) : 0u;
        }
    }
    if (kSpec || kFine) __syncthreads();  // full-id counters zeroed before any rank
    // kPush: bucket b = (owner d, coarse c) writes row j of the local order to
    // seg[d] + (j - start of d's segment), so each owner's rows land contiguous
    // in its receive buffer, C coarse runs in order.  (Shared only when used.)
    __shared__ longlong2* bptr[kPush ? kTileBuckets : 1];
    if (kPush) {
        for (int b = threadIdx.x; b < buckets; b += blockDim.x) {
            const int d = b >> log2b;
            const int64_t seg0 = offsets[static_cast<int64_t>(d << log2b) * gridDim.x];
            bptr[b] = reinterpret_cast<longlong2*>(reinterpret_cast<uintptr_t>(push.seg[d]) -
                                                   static_cast<uintptr_t>(seg0) * sizeof(longlong2));
        }
    }
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    const int pf = tile_prefetch;  // tiles prefetched ahead
    if (pf && threadIdx.x == 0) l2_prefetch_rows(keys, vals, lo, hi, pf * kTileRows);
    for (int64_t tile = lo; tile < hi; tile += kTileRows) {
        // the next tile(s) stream into L2 while this one is ranked, staged and copied out
        if (pf && threadIdx.x == 0 && tile + pf * kTileRows < hi)
            l2_prefetch_rows(keys, vals, tile + pf * kTileRows, hi, kTileRows);
        // 1-2. load (warp w owns rows [tile + 256 w, tile + 256 w + 256)) and rank each
        // row among the warp's rows of its bucket.  Full tiles and 256 buckets (the
        // common case) run without per-row bounds or bit-count checks.
        longlong2 row[kRowsPerThread];
        uint32_t bk[kRowsPerThread];
        uint16_t off[kRowsPerThread];
        uint16_t* wb = wbase + w * kTileBuckets;
        for (int b = lane; b < kTileBuckets; b += 32) wb[b] = 0;
        __syncwarp();
        const int rem = hi - tile < kTileRows ? static_cast<int>(hi - tile) : kTileRows;
        if (kFine) {  // (atomic ranking only)
            if (rem == kTileRows)
                load_and_rank_atomic<true, false, true>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off, fc);
            else
                load_and_rank_atomic<false, false, true>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off, fc);
        } else if (kSpec) {  // (atomic ranking only)
            if (rem == kTileRows)
                load_and_rank_atomic<true, true>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off, fc);
            else
                load_and_rank_atomic<false, true>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off, fc);
        } else if (atomic_rank) {
            if (rem == kTileRows)
                load_and_rank_atomic<true>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off);
            else
                load_and_rank_atomic<false>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, wb, row, bk, off);
        } else if (rem == kTileRows && nbits == 8)
            load_and_rank<true, 8>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, nbits, wb, row, bk, off);
        else
            load_and_rank<false, 0>(keys, vals, tile, rem, w, lane, mode, buckets, log2b, nbits, wb, row, bk, off);
        __syncthreads();
        // 3. per-bucket tile totals, exclusive over buckets; warp bases within each bucket.
        // Thread b also owns bucket b's cursor: it records where the tile's run goes
        // (dbase) and advances gcur itself, so no barrier follows the copy-out (the
        // next tile's first barrier already orders it before anything it reads).
        uint32_t total = 0, tst = 0, gstart = 0;
        if (kBulk && threadIdx.x < kTileBuckets) m4d::ptx::bulk_wait_read_all();  // last tile's runs left the stage
        if (threadIdx.x < kTileBuckets) {
            const int b = threadIdx.x;
            for (int ww = 0; ww < kW; ++ww) {
                const uint32_t c = wbase[ww * kTileBuckets + b];
                wbase[ww * kTileBuckets + b] = static_cast<uint16_t>(total);
                total += c;
            }
            uint32_t incl = total;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) scan_tmp[w] = incl;
        }
        __syncthreads();
        if (threadIdx.x < kTileBuckets) {
            const int b = threadIdx.x;
            uint32_t before = 0;
            for (int ww = 0; ww < w; ++ww) before += scan_tmp[ww];
            uint32_t incl = total;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            tst = before + incl - total;
            tstart[b] = tst;
            if (b == kTileBuckets - 1) tstart[kTileBuckets] = before + incl;
            gstart = gcur[b];
            dbase[b] = gstart - tst;  // (mod 2^32: dbase[b] + r with r >= tst is the row)
            gcur[b] = gstart + total;
            for (int ww = 0; ww < kW; ++ww)
                wbase[ww * kTileBuckets + b] = static_cast<uint16_t>(wbase[ww * kTileBuckets + b] + tst);
        }
        __syncthreads();
        // 4. stage rows in bucket order
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            if (bk[u] == 0xffffffffu) continue;
            const uint32_t pos = wbase[w * kTileBuckets + bk[u]] + off[u];
            stage[pos] = row[u];
            sbucket[pos] = static_cast<uint8_t>(bk[u]);
        }
        if (kBulk) m4d::ptx::fence_proxy_async_smem();  // stage writes before the TMA engine reads them
        __syncthreads();
        // 5. copy each bucket's run to its global place: kBulk, one TMA bulk store
        // per run (thread b issues bucket b's; the stage is reused only after the
        // copies have read it, step 3 of the next tile); else row by row.
        if (kBulk) {
            if (threadIdx.x < kTileBuckets) {
                const int b = threadIdx.x;
                uint32_t keep = total;
                if (kSpec) keep = gstart >= lim[b] ? 0u : (lim[b] - gstart < total ? lim[b] - gstart : total);
                if (keep) {
                    longlong2* dst = (kPush ? bptr[b] : out) + gstart;
                    m4d::ptx::bulk_s2g(dst, stage + tst, keep * static_cast<uint32_t>(sizeof(longlong2)));
                }
                m4d::ptx::bulk_commit();
            }
        } else {
            const uint32_t valid = tstart[kTileBuckets];
            for (uint32_t r = threadIdx.x; r < valid; r += blockDim.x) {
                const uint32_t b = sbucket[r];
                if (kPush)
                    bptr[b][dbase[b] + r] = stage[r];
                else if (!kSpec || dbase[b] + r < lim[b])
                    out[dbase[b] + r] = stage[r];
            }
        }
    }
    if (kBulk && threadIdx.x < kTileBuckets) m4d::ptx::bulk_wait_all();
    if (kSpec) {
        // exact per-bucket counts (what the histogram pass would have produced), the
        // overflow flag, and this CTA's full-id counts into its group's histogram
        if (threadIdx.x < buckets) {
            const int b = threadIdx.x;
            const uint32_t r0 = lim[b] - static_cast<uint32_t>(spec.cap);
            spec.counts[static_cast<int64_t>(b) * gridDim.x + blockIdx.x] = gcur[b] - r0;
            if (gcur[b] > lim[b]) atomicExch(spec.overflow, 1);
        }
        __syncthreads();  // every rank's count_full is done
        for (int i = threadIdx.x; i < (1 << spec.log2full); i += blockDim.x) {
            const uint32_t c = (fc.smem[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
            if (c) atomicAdd(fc.global + i, static_cast<unsigned long long>(c));
        }
    }
    if (kFine) {
        __syncthreads();  // every rank's count_id is done
        for (int i = threadIdx.x; i < spec.fine_ids; i += blockDim.x) {
            const uint32_t c = (fc.smem[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
            if (c) atomicAdd(fc.global32 + i, c);
        }
        // the last CTA to finish hands every owner its row of counts (peer stores into the
        // owner's buffer), so no copy follows the kernel
        __threadfence();
        __syncthreads();
        __shared__ int last_cta;
        if (threadIdx.x == 0) last_cta = atomicAdd(spec.fine_out + spec.fine_ids, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last_cta) {
            __threadfence();
            const int parts = 1 << spec.log2full;
            for (int i = threadIdx.x; i < spec.fine_ids; i += blockDim.x) {
                uint32_t* dst = spec.fine_dst[i >> spec.log2full];
                if (dst) dst[i & (parts - 1)] = __ldcg(spec.fine_out + i);
            }
        }
    }
}

// ---- two-pass LOCAL partition (buckets > kSinglePassMax) -------------------------------
// Pass 1 groups rows by the top b1 bits of the partition id into a scratch
// pair array; pass 2 (one CTA per pass-1 segment) splits every segment by
// the low b2 bits straight into its final place.  One histogram of the full
// id (per CTA: counts by top bits for pass 1; summed globally: the final
// bounds) serves both passes, so no second histogram read is needed.  Both
// passes keep their write frontier (CTAs x fan-out x 32 B) inside L2.

// Full-id histogram in shared memory: 32-bit counters up to 32768 partitions;
// for 65536, 16-bit counters packed two per word (128 KB, what a CTA can
// hold).  A packed counter that would pass 65535 (one key repeated that often
// inside one CTA's rows) flags the CTA, which then recounts its rows with
// global atomics: exact under any skew.
template <bool kPacked>
__global__ void __launch_bounds__(1024) hist2_kernel(const int64_t* __restrict__ keys,
                                                     const int64_t* __restrict__ vals, int64_t n, int64_t run,
                                                     int log2b, int b1, int groups, uint32_t* __restrict__ hist_top,
                                                     unsigned long long* __restrict__ hist_grp, bool pf) {
    extern __shared__ uint32_t h2[];  // 2^log2b 16-bit counters
    __shared__ uint32_t top[256];
    __shared__ int overflow;
    const int buckets = 1 << log2b;
    unsigned long long* hist_all = hist_grp + static_cast<int64_t>(blockIdx.x * groups / gridDim.x) * buckets;
    const int words = kPacked ? (buckets + 1) / 2 : buckets;
    const int shift = log2b - b1;
    for (int w = threadIdx.x; w < words; w += blockDim.x) h2[w] = 0;
    if (threadIdx.x == 0) overflow = 0;
    __syncthreads();
    const int64_t lo = blockIdx.x * run, hi = lo + run < n ? lo + run : n;
    auto count_key = [&](int64_t key) {
        const uint32_t b = bucket_of(key, M4D_PART_LOCAL, buckets, log2b);
        if (kPacked) {
            const uint32_t half = (b & 1u) << 4;
            const uint32_t old = atomicAdd(&h2[b >> 1], 1u << half);
            if (((old >> half) & 0xffffu) == 0xffffu) overflow = 1;
        } else {
            atomicAdd(&h2[b], 1u);
        }
    };
    for_each_key(keys, vals, lo, hi, pf, count_key);
    __syncthreads();
    if (!overflow) {
        auto count = [&](int b) -> uint32_t { return kPacked ? (h2[b >> 1] >> ((b & 1) << 4)) & 0xffffu : h2[b]; };
        for (int b = threadIdx.x; b < buckets; b += blockDim.x) {
            const uint32_t c = count(b);
            if (c) atomicAdd(hist_all + b, static_cast<unsigned long long>(c));
        }
        for (int t = threadIdx.x; t < (1 << b1); t += blockDim.x) {
            uint32_t c = 0;
            for (int q = 0; q < (1 << shift); ++q) c += count(t << shift | q);
            hist_top[static_cast<int64_t>(t) * gridDim.x + blockIdx.x] = c;
        }
        return;
    }
    // rare skew path: exact recount with global atomics
    for (int t = threadIdx.x; t < 256; t += blockDim.x) top[t] = 0;
    __syncthreads();
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const uint32_t b = bucket_of(key_at(keys, vals, i), M4D_PART_LOCAL, buckets, log2b);
        atomicAdd(hist_all + b, 1ull);
        atomicAdd(&top[b >> shift], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < (1 << b1); t += blockDim.x)
        hist_top[static_cast<int64_t>(t) * gridDim.x + blockIdx.x] = top[t];
}

// hist_grp[g][b] -> counts of the groups before g (exclusive over g); hist_all[b] = total.
__global__ void group_prefix_kernel(unsigned long long* __restrict__ hist_grp, int groups, int buckets,
                                    unsigned long long* __restrict__ hist_all) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < buckets; b += gridDim.x * blockDim.x) {
        unsigned long long run = 0;
        for (int g = 0; g < groups; ++g) {
            const unsigned long long c = hist_grp[static_cast<int64_t>(g) * buckets + b];
            hist_grp[static_cast<int64_t>(g) * buckets + b] = run;
            run += c;
        }
        hist_all[b] = run;
    }
}

__global__ void exclusive_scan_u64_kernel(const unsigned long long* __restrict__ v, int n, int64_t* __restrict__ out,
                                          int64_t total) {
    // one CTA of 1024 threads; n <= 65536
    __shared__ int64_t warp_tot[32];
    const int per = (n + 1023) / 1024;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int64_t local = 0;
    for (int k = 0; k < per; ++k) {
        const int i = t * per + k;
        if (i < n) local += static_cast<int64_t>(v[i]);
    }
    int64_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int64_t w = warp_tot[lane], wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        warp_tot[lane] = wi - w;
    }
    __syncthreads();
    int64_t run = warp_tot[warp] + incl - local;
    for (int k = 0; k < per; ++k) {
        const int i = t * per + k;
        if (i < n) {
            out[i] = run;
            run += static_cast<int64_t>(v[i]);
        }
    }
    if (t == 0) out[n] = total;
}

// Second-level scatter of rows [lo, hi) of `in` by the low bits of their local
// partition id, through per-partition cursors in shared memory.  pf: thread 0
// prefetches the next chunk into L2 while the CTA scatters this one.
__device__ __forceinline__ void scatter_by_low_bits(const longlong2* __restrict__ in, int64_t lo, int64_t hi,
                                                    uint32_t* cursor, int log2b, uint32_t mask,
                                                    longlong2* __restrict__ out, bool pf) {
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kRowsPerThread;
    if (pf && threadIdx.x == 0) l2_prefetch(in, lo, chunk, hi);
    for (int64_t base = lo; base < hi; base += chunk) {
        if (pf && threadIdx.x == 0) l2_prefetch(in, base + chunk, chunk, hi);
        longlong2 row[kRowsPerThread];
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            if (i < hi) row[u] = __ldcs(in + i);
        }
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            if (base + u * blockDim.x + threadIdx.x >= hi) continue;
            const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(row[u].x));
            const uint32_t b2 = static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2b)) & mask;
            out[atomicAdd(&cursor[b2], 1u)] = row[u];
        }
    }
}

// Pass 2: one CTA per (segment, group of pass-1 CTAs).  Within a segment the
// rows of one group are contiguous, and the group's cursors start at the
// partition bounds plus the counts of the earlier groups (from the per-group
// histograms), so groups scatter independently and rows keep their order.
// fan x groups CTAs instead of fan (256 CTAs of 1024 threads ran in 1.7
// waves on 148 SMs).
__global__ void __launch_bounds__(1024)
    scatter_pass2_kernel(const longlong2* __restrict__ in, const int64_t* __restrict__ offs, int ctas, int64_t n,
                         const unsigned long long* __restrict__ grp_before, int groups,
                         const int64_t* __restrict__ bounds, int log2b, int b1, longlong2* __restrict__ out,
                         bool pf) {
    extern __shared__ uint32_t cursor[];  // 2^(log2b - b1)
    const int sub = 1 << (log2b - b1);
    const int seg = blockIdx.x / groups, g = blockIdx.x % groups;
    const int buckets = 1 << log2b;
    for (int k = threadIdx.x; k < sub; k += blockDim.x) {
        const int b = seg * sub + k;
        cursor[k] = static_cast<uint32_t>(bounds[b] + static_cast<int64_t>(grp_before[static_cast<int64_t>(g) * buckets + b]));
    }
    __syncthreads();
    const int k0 = (g * ctas + groups - 1) / groups, k1 = ((g + 1) * ctas + groups - 1) / groups;
    const int64_t entries = static_cast<int64_t>(ctas) << b1;
    const int64_t i0 = static_cast<int64_t>(seg) * ctas + k0, i1 = static_cast<int64_t>(seg) * ctas + k1;
    const int64_t lo = i0 < entries ? offs[i0] : n, hi = i1 < entries ? offs[i1] : n;
    scatter_by_low_bits(in, lo, hi, cursor, log2b, static_cast<uint32_t>(sub - 1), out, pf);
}

// Pass 2 after a speculative pass 1: one CTA per (segment, group of pass-1
// CTAs) as above, but the group's rows sit in one region per pass-1 CTA --
// (seg * ctas + c) * cap when pass 1 fit its regions, offs[seg * ctas + c] when
// *overflow sent it through the exact fallback -- holding counts[seg * ctas + c]
// rows each.  The CTA walks the regions as one virtual row range.
constexpr int kMaxRegions = 1024;

__global__ void __launch_bounds__(1024)
    spec_pass2_kernel(const longlong2* __restrict__ in, const uint32_t* __restrict__ counts,
                      const int64_t* __restrict__ offs, const int* __restrict__ overflow, int64_t cap, int ctas,
                      const unsigned long long* __restrict__ grp_before, int groups,
                      const int64_t* __restrict__ bounds, int log2b, int b1, longlong2* __restrict__ out, bool pf) {
    extern __shared__ uint32_t cursor[];  // 2^(log2b - b1)
    __shared__ int64_t rstart[kMaxRegions];
    __shared__ uint32_t rpre[kMaxRegions + 1];
    const int sub = 1 << (log2b - b1);
    const int seg = blockIdx.x / groups, g = blockIdx.x % groups;
    const int buckets = 1 << log2b;
    for (int k = threadIdx.x; k < sub; k += blockDim.x) {
        const int b = seg * sub + k;
        cursor[k] = static_cast<uint32_t>(bounds[b] + static_cast<int64_t>(grp_before[static_cast<int64_t>(g) * buckets + b]));
    }
    const int k0 = (g * ctas + groups - 1) / groups, k1 = ((g + 1) * ctas + groups - 1) / groups;
    const int nreg = k1 - k0;
    const bool exact = *overflow != 0;
    const int64_t idx0 = static_cast<int64_t>(seg) * ctas + k0;
    for (int k = threadIdx.x; k < nreg; k += blockDim.x) rstart[k] = exact ? offs[idx0 + k] : (idx0 + k) * cap;
    if (threadIdx.x < 32) {  // exclusive prefix of the region counts
        const int lane = threadIdx.x;
        uint32_t carry = 0;
        for (int base = 0; base < nreg; base += 32) {
            const uint32_t c = base + lane < nreg ? counts[idx0 + base + lane] : 0u;
            uint32_t incl = c;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (base + lane < nreg) rpre[base + lane] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) rpre[nreg] = carry;
    }
    __syncthreads();
    const int64_t total = rpre[nreg];
    const uint32_t mask = static_cast<uint32_t>(sub - 1);
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kRowsPerThread;
    // region of virtual row i: the last r with rpre[r] <= i
    auto region = [&](int64_t i) {
        int lo = 0, hi = nreg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rpre[mid] <= i) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    auto prefetch = [&](int64_t v0) {  // the pieces of virtual rows [v0, v0 + chunk)
        if (v0 >= total) return;
        const int64_t v1 = v0 + chunk < total ? v0 + chunk : total;
        for (int r = region(v0); r < nreg && rpre[r] < v1; ++r) {
            const int64_t a = v0 > rpre[r] ? v0 : rpre[r], z = v1 < rpre[r + 1] ? v1 : rpre[r + 1];
            if (z > a) l2_prefetch(in, rstart[r] + (a - rpre[r]), z - a, rstart[r] + (z - rpre[r]));
        }
    };
    if (pf && threadIdx.x == 0) prefetch(0);
    for (int64_t base = 0; base < total; base += chunk) {
        if (pf && threadIdx.x == 0) prefetch(base + chunk);
        longlong2 row[kRowsPerThread];
        int r = base + threadIdx.x < total ? region(base + threadIdx.x) : 0;
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            if (i < total) {
                while (r + 1 < nreg && rpre[r + 1] <= i) ++r;
                row[u] = __ldcs(in + rstart[r] + (i - rpre[r]));
            }
        }
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            if (base + u * blockDim.x + threadIdx.x >= total) continue;
            const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(row[u].x));
            const uint32_t b2 = static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2b)) & mask;
            out[atomicAdd(&cursor[b2], 1u)] = row[u];
        }
    }
}

// Receiver side of the owner+coarse exchange (M4D_PART_OWNER_COARSE): S
// source segments, each holding C coarse runs in bucket order, are split into
// the final 2^log2b partitions.  Every (coarse run, source) piece is cut into
// G row ranges; one CTA per (run, source, range) counts its rows per
// sub-partition (the low log2b - cbits bits), the counts become cursors
// (partition bounds plus the rows of earlier (source, range) pairs, so rows
// stay source-ordered), and a CTA per (run, source, range) scatters its rows.
// C x S x G CTAs per pass: enough to fill 148 SMs (C x S alone can be 128).
__device__ __forceinline__ void piece_range(const int64_t* __restrict__ runs, int piece, int g, int groups,
                                            int64_t* a, int64_t* z) {
    const int64_t lo = runs[2 * piece], hi = runs[2 * piece + 1], len = hi - lo;
    *a = lo + len * g / groups;
    *z = lo + len * (g + 1) / groups;
}

__global__ void __launch_bounds__(1024) runs_hist_kernel(const longlong2* __restrict__ in, const int64_t* __restrict__ runs,
                                                         int sources, int groups, int log2b, int cbits,
                                                         unsigned long long* __restrict__ hist_grp, bool pf) {
    extern __shared__ uint32_t h[];  // 2^(log2b - cbits)
    const int sub = 1 << (log2b - cbits), buckets = 1 << log2b;
    const int g = blockIdx.x % groups, piece = blockIdx.x / groups;  // piece = c * sources + src
    const int c = piece / sources, src = piece % sources;
    for (int k = threadIdx.x; k < sub; k += blockDim.x) h[k] = 0;
    __syncthreads();
    int64_t a, z;
    piece_range(runs, piece, g, groups, &a, &z);
    const int64_t chunk = static_cast<int64_t>(blockDim.x) * kRowsPerThread;
    if (pf && threadIdx.x == 0) l2_prefetch(in, a, chunk, z);
    for (int64_t base = a; base < z; base += chunk) {
        if (pf && threadIdx.x == 0) l2_prefetch(in, base + chunk, chunk, z);
        int64_t k[kRowsPerThread];
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            k[u] = i < z ? __ldcs(&in[i].x) : 0;
        }
#pragma unroll
        for (int u = 0; u < kRowsPerThread; ++u)
            if (base + u * blockDim.x + threadIdx.x < z)
                atomicAdd(&h[bucket_of(k[u], M4D_PART_LOCAL, buckets, log2b) & (sub - 1)], 1u);
    }
    __syncthreads();
    unsigned long long* out = hist_grp + static_cast<int64_t>(src * groups + g) * buckets + c * sub;
    for (int k = threadIdx.x; k < sub; k += blockDim.x) out[k] = h[k];
}

__global__ void __launch_bounds__(1024)
    runs_pass2_kernel(const longlong2* __restrict__ in, const int64_t* __restrict__ runs, int sources, int groups,
                      const unsigned long long* __restrict__ grp_before, const int64_t* __restrict__ bounds,
                      int log2b, int cbits, longlong2* __restrict__ out, bool pf) {
    extern __shared__ uint32_t cursor[];  // 2^(log2b - cbits)
    const int sub = 1 << (log2b - cbits), buckets = 1 << log2b;
    const int g = blockIdx.x % groups, piece = blockIdx.x / groups;
    const int c = piece / sources, src = piece % sources;
    const unsigned long long* before = grp_before + static_cast<int64_t>(src * groups + g) * buckets + c * sub;
    for (int k = threadIdx.x; k < sub; k += blockDim.x)
        cursor[k] = static_cast<uint32_t>(bounds[c * sub + k] + static_cast<int64_t>(before[k]));
    __syncthreads();
    int64_t a, z;
    piece_range(runs, piece, g, groups, &a, &z);
    scatter_by_low_bits(in, a, z, cursor, log2b, static_cast<uint32_t>(sub - 1), out, pf);
}

__global__ void bucket_bounds_kernel(const int64_t* __restrict__ offsets, int buckets, int ctas, int64_t total,
                                     int64_t* __restrict__ bounds) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= buckets; b += gridDim.x * blockDim.x)
        bounds[b] = b < buckets ? offsets[static_cast<int64_t>(b) * ctas] : total;
}

// One CTA per partition: a chained hash table of the left rows in shared
// memory (chunks of kChunk rows): 16384 chain heads, the chunk's keys and one
// 16-bit link per row.  Inserting is one atomicExch per row (no probing
// loops); a probe walks only the rows that share its head, Poisson(rows /
// 16384) long, so lanes of a warp finish together (linear probing at the same
// load ran ~6 divergent steps per warp for ~1.2 per row).  The right rows
// stream through in batches of kJoinThreads * kJoinPer, warp-independently:
// (1) each thread walks its rows' chains once, keeping per row the first
// matching build row and the match count; (2) a warp scan plus one global
// atomic per warp reserves the warp's output range; (3) each thread writes its
// matches as packed (probe row, build row) entries into the warp's stage
// (re-walking only rows with several matches); (4) the warp emits the stage
// with all 32 lanes: coalesced output stores, full-width row hashes.
// Indices are 32-bit offsets from the partition start.
template <int kJoinThreads, int kSlotBits, int kChunk, int kStage, int kMinBlocks, int kKeep>
__global__ void __launch_bounds__(kJoinThreads, kMinBlocks)
    join_kernel(const longlong2* __restrict__ build, const int64_t* __restrict__ loff,
                const longlong2* __restrict__ probe, const int64_t* __restrict__ roff, int64_t* __restrict__ ok,
                int64_t* __restrict__ ol, int64_t* __restrict__ orr, int64_t capacity,
                unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ digest, int parts, int pf,
                int ahead) {
    constexpr int kSlots = 1 << kSlotBits;
    extern __shared__ __align__(16) unsigned char smem[];
    int64_t* bkey = reinterpret_cast<int64_t*>(smem);                                   // [kChunk]
    uint32_t* head = reinterpret_cast<uint32_t*>(smem + kChunk * sizeof(int64_t));      // [kSlots]
    uint16_t* link = reinterpret_cast<uint16_t*>(head + kSlots);                        // [kChunk]
    uint32_t* stage_all = reinterpret_cast<uint32_t*>(link + kChunk);
    __shared__ unsigned long long red[kJoinThreads / 32][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int T = kJoinThreads;
    constexpr int kPer = kJoinPer;
    uint32_t* stage = stage_all + warp * kStage;
    unsigned long long cnt = 0, hsum = 0, ksum = 0;
    // grid = parts: one partition per CTA; a smaller (persistent) grid walks partitions
    // blockIdx.x, + gridDim.x, ... and prefetches the next one's rows into L2 meanwhile.
    for (int part = blockIdx.x; part < parts; part += gridDim.x) {
    if (part != static_cast<int>(blockIdx.x)) __syncthreads();  // the previous partition's table is done
    if (threadIdx.x == 0 && part + static_cast<int>(gridDim.x) < parts) {
        const int nx = part + gridDim.x;
        const int64_t ln = loff[nx + 1] - loff[nx], rn = roff[nx + 1] - roff[nx];
        const uint32_t lb = static_cast<uint32_t>((ln < (1 << 20) ? ln : (1 << 20)) * 16);
        const uint32_t rb = static_cast<uint32_t>((rn < (1 << 20) ? rn : (1 << 20)) * 16);
        if (lb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(build + loff[nx]), "r"(lb) : "memory");
        if (rb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(probe + roff[nx]), "r"(rb) : "memory");
    }
    const longlong2* brow = build + loff[part];
    const longlong2* prow = probe + roff[part];
    // L2 bulk prefetches (M4D_JOIN_PF bits): 1 = this partition's probe rows
    // (stream in while the table is built), 2 = its build rows, 4 = both sides
    // of partition part + ahead (about one wave of CTAs later, any SM).
    if (pf && threadIdx.x == 0) {
        auto l2 = [](const longlong2* p, int64_t rows) {
            const uint32_t b = static_cast<uint32_t>((rows < (1 << 20) ? rows : (1 << 20)) * 16);
            if (b) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(b) : "memory");
        };
        if (pf & 1) l2(prow, roff[part + 1] - roff[part]);
        if (pf & 2) l2(brow, loff[part + 1] - loff[part]);
        if ((pf & 4) && part + ahead < parts) {
            const int nx = part + ahead;
            l2(build + loff[nx], loff[nx + 1] - loff[nx]);
            l2(probe + roff[nx], roff[nx + 1] - roff[nx]);
        }
    }
    if (loff[part + 1] - loff[part] > INT32_MAX || roff[part + 1] - roff[part] > INT32_MAX)
        __trap();  // partitions are < 2^31 rows (32-bit offsets); fail loudly rather than mis-join
    const int bn = static_cast<int>(loff[part + 1] - loff[part]);
    const int pn = static_cast<int>(roff[part + 1] - roff[part]);
    for (int c0 = 0; c0 < bn; c0 += kChunk) {
        const int cn = bn - c0 < kChunk ? bn - c0 : kChunk;
        const longlong2* crow = brow + c0;
        if (c0) __syncthreads();  // every warp is done probing the previous chunk's table
        for (int s = threadIdx.x; s < kSlots; s += T) head[s] = kEmpty;
        __syncthreads();
        for (int base = 0; base < cn; base += T * kPer) {
            int64_t k[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = base + u * T + threadIdx.x;
                k[u] = i < cn ? crow[i].x : 0;
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int i = base + u * T + threadIdx.x;
                if (i >= cn) break;  // rows ascend with u
                bkey[i] = k[u];
                const uint32_t old = atomicExch(&head[slot_of<kSlotBits>(k[u])], static_cast<uint32_t>(i));
                link[i] = old == kEmpty ? kNil : static_cast<uint16_t>(old);
            }
        }
        __syncthreads();
        for (int base = 0; base < pn; base += T * kPer) {
            int64_t r[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int j = base + u * T + threadIdx.x;
                r[u] = j < pn ? prow[j].x : 0;
            }
            // first matching build row | min(matches, 0xffff) << 16, and the second and
            // third matches (16 bits each): with duplicate keys (Poisson(1) copies per key
            // here) 42 % of the matched rows have two or more, and keeping two more
            // indices leaves a re-walk below to the 3 % with four or more
            uint32_t info[kPer], second[kPer];
            uint32_t mine = 0;
#pragma unroll
            for (int u = 0; u < kPer; ++u) {  // (1) count
                info[u] = 0;
                second[u] = 0;
                if (base + u * T + static_cast<int>(threadIdx.x) >= pn) continue;
                uint32_t c = 0, first = 0, sec = 0;
                const uint32_t h0 = head[slot_of<kSlotBits>(r[u])];
                for (uint32_t i = h0 == kEmpty ? kNil : h0; i != kNil; i = link[i])
                    if (bkey[i] == r[u]) {
                        if (kKeep > 1) sec = c == 1 ? i : (kKeep > 2 && c == 2) ? sec | i << 16 : sec;
                        first = c ? first : i;
                        ++c;
                    }
                info[u] = first | (c < 0xffffu ? c : 0xffffu) << 16;
                second[u] = sec;
                mine += c;
            }
            uint32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t warp_total = __shfl_sync(0xffffffffu, incl, 31);
            if (!warp_total) continue;  // warp-uniform
            unsigned long long wbase = 0;  // (2) reserve
            if (lane == 31) wbase = atomicAdd(cursor, static_cast<unsigned long long>(warp_total));
            wbase = __shfl_sync(0xffffffffu, wbase, 31);
            const uint32_t my0 = incl - mine;
            for (uint32_t win = 0; win < warp_total; win += kStage) {  // warp-uniform rounds
                if (mine && my0 < win + kStage && my0 + mine > win) {  // (3) stage
                    uint32_t e = my0;
#pragma unroll
                    for (int u = 0; u < kPer; ++u) {
                        const uint32_t c = info[u] >> 16;
                        if (!c) continue;
                        const uint32_t loc = static_cast<uint32_t>(u * T + threadIdx.x) << kIdxBits;
                        const uint32_t first = info[u] & 0xffffu;
                        if (c <= static_cast<uint32_t>(kKeep)) {
                            if (e >= win && e < win + kStage) stage[e - win] = loc | first;
                            ++e;
                            if (kKeep > 1 && c >= 2) {
                                if (e >= win && e < win + kStage) stage[e - win] = loc | (second[u] & 0xffffu);
                                ++e;
                            }
                            if (kKeep > 2 && c == 3) {
                                if (e >= win && e < win + kStage) stage[e - win] = loc | (second[u] >> 16);
                                ++e;
                            }
                            continue;
                        }
                        for (uint32_t i = first; i != kNil; i = link[i]) {
                            if (bkey[i] != r[u]) continue;
                            if (e >= win && e < win + kStage) stage[e - win] = loc | i;
                            ++e;
                        }
                    }
                }
                __syncwarp();
                const uint32_t n = warp_total - win < kStage ? warp_total - win : kStage;
                for (uint32_t q = lane; q < n; q += 32) {  // (4) emit, all lanes
                    const uint32_t ent = stage[q];
                    const uint32_t i = ent & ((1u << kIdxBits) - 1);
                    const int64_t key = bkey[i];
                    const int64_t l = crow[i].y;
                    const int64_t rv = prow[base + static_cast<int>(ent >> kIdxBits)].y;
                    const unsigned long long pos = wbase + win + q;
                    if (static_cast<int64_t>(pos) < capacity) {
                        ok[pos] = key;
                        ol[pos] = l;
                        orr[pos] = rv;
                    }
                    ++cnt;
                    hsum += row_hash(key, l, rv);
                    ksum += static_cast<unsigned long long>(key);
                }
                __syncwarp();
            }
        }
    }
    }  // partitions
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
    }
    if (lane == 0) {
        red[warp][0] = cnt;
        red[warp][1] = hsum;
        red[warp][2] = ksum;
    }
    __syncthreads();
    if (warp == 0) {
        static_assert(kJoinThreads / 32 <= 32, "one warp folds the per-warp sums");
        cnt = lane < kJoinThreads / 32 ? red[lane][0] : 0;
        hsum = lane < kJoinThreads / 32 ? red[lane][1] : 0;
        ksum = lane < kJoinThreads / 32 ? red[lane][2] : 0;
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
}

// Sender side of the counted receiver split: rows per (owner, local partition)
// of this rank's table -- what every owner's split would otherwise count from
// the received rows.  16-bit shared-memory counters, two per word, for all
// owners x partitions (8 x 8192 in 128 KB); the increment that takes a counter
// to 0x8000 moves 0x8000 to the global count, so a half never carries into its
// neighbour and any skew stays exact.
__global__ void __launch_bounds__(1024) fine_count_kernel(const int64_t* __restrict__ keys,
                                                          const int64_t* __restrict__ vals, int64_t n, int world,
                                                          int log2b, uint32_t* __restrict__ out, int pf) {
    extern __shared__ uint32_t fc[];  // (world << log2b) / 2 words
    const int total = world << log2b;
    for (int i = threadIdx.x; i < total / 2; i += blockDim.x) fc[i] = 0;
    __syncthreads();
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
    for_each_key(keys, vals, lo, hi, pf != 0, [&](int64_t key) {
        const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(key));
        const uint32_t owner = __umulhi(static_cast<uint32_t>(h >> 32), static_cast<uint32_t>(world));
        const uint32_t p = static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2b));
        const uint32_t idx = owner << log2b | p, sh = (idx & 1u) * 16u;
        const uint32_t old = atomicAdd(&fc[idx >> 1], 1u << sh);
        if (((old >> sh) & 0xffffu) == 0x7fffu) {  // this increment reached 0x8000: spill it
            atomicSub(&fc[idx >> 1], 0x8000u << sh);
            atomicAdd(out + idx, 0x8000u);
        }
    });
    __syncthreads();
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const uint32_t c = (fc[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
        if (c) atomicAdd(out + i, c);
    }
}

// Receiver side: per-source counts (fine[src][b]) -> rows of earlier sources per
// partition (grp_before[src][b]) and per-partition totals.
__global__ void fine_prefix_kernel(const uint32_t* __restrict__ fine, int sources, int buckets,
                                   unsigned long long* __restrict__ grp_before, unsigned long long* __restrict__ hist_all) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < buckets; b += gridDim.x * blockDim.x) {
        unsigned long long run = 0;
        for (int src = 0; src < sources; ++src) {
            grp_before[static_cast<int64_t>(src) * buckets + b] = run;
            run += fine[static_cast<int64_t>(src) * buckets + b];
        }
        hist_all[b] = run;
    }
}

int log2_exact(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return (1 << l) == v ? l : -1;
}

}  // namespace

using m4d::fail;

// Threads per tile-scatter CTA (M4D_TILE_THREADS = 256 | 512 | 1024, default 512): sets the
// resident CTAs per SM (2048 / threads, at most 4) and so the partition grid.  Measured
// (1e8 rows/side, both sides' partitions): ballot ranking 1.02 / 1.12 / 1.35 ms per tile
// scatter at 256 / 512 / 1024; atomic ranking 3.47 / 3.27 / 3.66 ms for all partitions.
static int tile_threads() {
    static const int t = [] {
        const char* v = getenv("M4D_TILE_THREADS");
        const int x = v ? atoi(v) : 512;
        return x == 256 || x == 1024 ? x : 512;
    }();
    return t;
}

static int partition_ctas(int64_t n, int threads = tile_threads(), int per_sm_cap = 4) {
    // One wave of the tile scatter (its L2 write frontier must fit, see top).
    int per_sm = threads >= 1024 ? 1 : threads >= 512 ? 2 : 4;
    if (per_sm > per_sm_cap) per_sm = per_sm_cap;
    const int64_t per = 65536 * 2 / per_sm;
    int64_t c = (n + per - 1) / per;
    if (c < 1) c = 1;
    if (c > 148 * per_sm) c = 148 * per_sm;
    return static_cast<int>(c);
}

// Tile-scatter stores (M4D_TILE_STORE = bulk | rows): one TMA bulk store per
// bucket run of a tile, or the row-by-row copy.  Default: bulk for the push
// scatter (runs cross NVLink), rows for local partitions (measured 5.46 vs
// 5.56 ms per local merge step; push N=2 8.63 vs 8.76 ms).
static bool tile_bulk(bool push) {
    static const int mode = [] {
        const char* v = getenv("M4D_TILE_STORE");
        return !v ? -1 : strcmp(v, "rows") == 0 ? 0 : 1;
    }();
    return mode < 0 ? push : mode == 1;
}

// The speculative pass 1 (see SpecArgs) stores runs with TMA bulk copies unless
// M4D_TILE_STORE=rows: N=1 merge step 4.21 vs 4.32 ms (profiles/r2_spec_align.txt).
static bool tile_bulk_spec() {
    const char* v = getenv("M4D_TILE_STORE");
    return !(v && strcmp(v, "rows") == 0);
}

// Threads per push-scatter CTA (M4D_PUSH_TILE_THREADS, default 1024): longer
// runs per bucket per tile make NVLink stores efficient (N=2 / N=4 at 128
// push buckets: 8.08 / 9.99 ms with 256 threads, 7.72 / 9.39 ms with 1024).
static int push_tile_threads() {
    static const int t = [] {
        const char* v = getenv("M4D_PUSH_TILE_THREADS");
        const int x = v ? atoi(v) : 1024;
        return x == 256 || x == 512 ? x : 1024;
    }();
    return t;
}

// Push-scatter CTAs per SM (M4D_PUSH_CTAS_PER_SM, default 4 = as many as fit):
// fewer leave SM room for the receiver split running beside the push.
static int push_ctas_per_sm() {
    static const int c = [] {
        const char* v = getenv("M4D_PUSH_CTAS_PER_SM");
        const int x = v ? atoi(v) : 4;
        return x < 1 ? 1 : x > 4 ? 4 : x;
    }();
    return c;
}

// SMs the push scatter's grid may occupy (M4D_PUSH_SMS, default 96): the rest
// stay free for the receiver split of the side pushed before (split stream),
// which otherwise waits for push CTAs to retire (they hold the register file).
// Sweep (tools/r2_push_sms.sh, N=2 / N=4 step ms): 148 -> 7.06 / 8.68,
// 112 -> 6.84 / 8.19, 96 -> 6.84 / 8.04, 80 -> 6.90 / 8.40, 64 -> 6.89 / 8.51.
static int push_sms() {
    static const int c = [] {
        const char* v = getenv("M4D_PUSH_SMS");
        const int x = v ? atoi(v) : 96;
        return x < 1 ? 1 : x > 148 ? 148 : x;
    }();
    return c;
}

// Threads per receiver-split CTA (M4D_RUNS_THREADS = 512 | 1024, default 1024).
static int runs_threads() {
    static const int t = [] {
        const char* v = getenv("M4D_RUNS_THREADS");
        return v && atoi(v) == 512 ? 512 : 1024;
    }();
    return t;
}

// Tile-scatter ranking (M4D_TILE_RANK = atomic | ballot, default atomic): see
// load_and_rank_atomic / load_and_rank.  Measured at 1e8 rows/side: 496M -> 289M
// instructions per tile-scatter launch, merge step 5.53 -> 5.29 ms (N=1), 7.43 ->
// 7.29 ms (N=2).
static bool tile_rank_atomic() {
    static const bool a = [] {
        const char* v = getenv("M4D_TILE_RANK");
        return !(v && strcmp(v, "ballot") == 0);
    }();
    return a;
}

// L2 bulk prefetch of the next chunk in every streaming partition pass (tile
// scatter, histograms, pass 2, the receiver split), M4D_L2_PF (default 1; 0
// off): the loads of a chunk then hit L2 instead of waiting on HBM.  Measured at
// 1e8 rows/side (tools/sweeps/r2_stream_pf*.sh): merge step 4.81 -> 4.62 ms
// (N=1); the tile scatter alone gives 0.16 ms of it.  Prefetching the tile
// scatter 2 or 3 tiles ahead is slower (4.78 / 4.93 ms: the lines are evicted
// before use), so the distance stays one chunk.
static int l2_pf() {
    static const int a = [] {
        const char* v = getenv("M4D_L2_PF");
        return v && atoi(v) <= 0 ? 0 : 1;
    }();
    return a;
}

template <int kT, bool kPush, bool kBulk, bool kSpec = false, bool kFine = false>
static cudaError_t launch_tile_scatter_t(int ctas, cudaStream_t s, const int64_t* keys, const int64_t* vals, int64_t n,
                                         int64_t run, int mode, int buckets, int log2b, const int64_t* offs,
                                         longlong2* out, const PushTargets& push, const SpecArgs& spec) {
    const size_t smem = tile_smem<kT>() + (kSpec ? (size_t(1) << spec.log2full) / 2 * sizeof(uint32_t) : 0) +
                        (kFine ? static_cast<size_t>(spec.fine_ids) / 2 * sizeof(uint32_t) : 0);
    const cudaError_t e = cudaFuncSetAttribute(tile_scatter_kernel<kT, kPush, kBulk, kSpec, kFine>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    tile_scatter_kernel<kT, kPush, kBulk, kSpec, kFine><<<ctas, kT, smem, s>>>(keys, vals, n, run, mode, buckets, log2b, offs,
                                                                        out, push, tile_rank_atomic(), l2_pf(), spec);
    return cudaGetLastError();
}

template <int kT>
static cudaError_t launch_tile_scatter_k(int ctas, cudaStream_t s, const int64_t* keys, const int64_t* vals, int64_t n,
                                         int64_t run, int mode, int buckets, int log2b, const int64_t* offs,
                                         longlong2* out, const PushTargets* push, const SpecArgs& spec, bool speculative) {
    static const PushTargets none{};
    if (push && spec.fine_out)  // the push with fused (owner, local partition) counts (bulk run stores)
        return launch_tile_scatter_t<kT, true, true, false, true>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, *push, spec);
    if (speculative)  // TMA bulk run stores unless M4D_TILE_STORE=rows (4.21 vs 4.32 ms per merge step)
        return tile_bulk_spec() ? launch_tile_scatter_t<kT, false, true, true>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, none, spec)
                                : launch_tile_scatter_t<kT, false, false, true>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, none, spec);
    if (tile_bulk(push != nullptr))
        return push ? launch_tile_scatter_t<kT, true, true>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, *push, spec)
                    : launch_tile_scatter_t<kT, false, true>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, none, spec);
    return push ? launch_tile_scatter_t<kT, true, false>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, *push, spec)
                : launch_tile_scatter_t<kT, false, false>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, none, spec);
}

// spec / speculative: see SpecArgs (the speculative pass 1, or the gate of its exact fallback).
static cudaError_t launch_tile_scatter(int ctas, cudaStream_t s, const int64_t* keys, const int64_t* vals, int64_t n,
                                       int64_t run, int mode, int buckets, int log2b, const int64_t* offs,
                                       longlong2* out, const PushTargets* push = nullptr,
                                       const SpecArgs& spec = SpecArgs{}, bool speculative = false) {
    switch (push ? push_tile_threads() : tile_threads()) {
        case 256: return launch_tile_scatter_k<256>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, push, spec, speculative);
        case 1024: return launch_tile_scatter_k<1024>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, push, spec, speculative);
        default: return launch_tile_scatter_k<512>(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs, out, push, spec, speculative);
    }
}

static int pass1_bits(int log2b) { return log2b > 8 ? 8 : log2b; }

// Speculative pass 1 (M4D_PASS1 = spec | hist, default spec): the two-pass LOCAL
// partition skips the histogram pass; pass 1 writes into fixed regions of
// spec_cap rows per (bucket, CTA) -- the mean plus six standard deviations plus
// 32 rows, at most the CTA's rows -- and an exact fallback (scan + the usual
// pass 1, gated on the overflow flag, so skew costs one more pass but never a
// wrong result) runs only when a region overflowed.  Up to 8192 partitions
// (16 KB of full-id counters keeps two 512-thread CTAs per SM).
static bool pass1_spec() {
    static const bool on = [] {
        const char* v = getenv("M4D_PASS1");
        return !(v && strcmp(v, "hist") == 0);
    }();
    return on;
}

static int64_t spec_cap(int64_t n, int ctas, int fan) {
    const int64_t run = (n + ctas - 1) / ctas;
    const double mean = static_cast<double>(run) / fan;
    int64_t cap = static_cast<int64_t>(std::ceil(mean + 6.0 * std::sqrt(mean) + 32.0));
    return cap > run ? (run > 0 ? run : 1) : cap;
}

static bool spec_applies(int64_t n, int ctas, int fan, int log2b) {
    if (!pass1_spec() || !tile_rank_atomic() || log2b > 13 || fan > kTileBuckets) return false;
    if ((ctas + kPass2Groups - 1) / kPass2Groups > kMaxRegions) return false;
    const int64_t run = (n + ctas - 1) / ctas;
    return static_cast<int64_t>(fan) * ctas * spec_cap(n, ctas, fan) + run < (int64_t(1) << 32);
}

// Single-pass partition (hist -> scan -> scatter) into `buckets` buckets; the
// bucket function gets (mode, buckets, log2b) as bucket_of documents.  The
// plan (histogram, per-(bucket, CTA) offsets in scratch, bounds) and the
// scatter can run as separate calls (kPlan / kScatter) on the same scratch:
// the fused owner push needs every owner's counts before it can write.
enum { kPlan = 1, kScatter = 2, kPlanAndScatter = 3 };

static m4d_status partition_single(const int64_t* keys, const int64_t* vals, int64_t n, int mode, int buckets,
                                   int log2b, int64_t* out_pairs, int64_t* bounds, void* scratch,
                                   size_t scratch_bytes, cudaStream_t s, int phases = kPlanAndScatter,
                                   const PushTargets* push = nullptr, bool push_layout = false,
                                   const SpecArgs& fine = SpecArgs{}) {
    if (scratch_bytes < m4d_partition_scratch_bytes(n, buckets)) return fail(M4D_ERR_USAGE, "partition scratch too small");
    // (the push scatter's plan and scatter calls both size the grid for its CTAs)
    int ctas = push_layout ? partition_ctas(n, push_tile_threads(), push_ctas_per_sm())
                           : partition_ctas(n, tile_threads());
    if (push_layout) {
        const int per_sm = push_tile_threads() >= 1024 ? 1 : push_tile_threads() >= 512 ? 2 : 4;
        const int cap = push_sms() * (per_sm < push_ctas_per_sm() ? per_sm : push_ctas_per_sm());
        if (ctas > cap) ctas = cap;
    }
    const int64_t run = (n + ctas - 1) / ctas;
    if (buckets > kMaxBuckets) return fail(M4D_ERR_USAGE, "bucket count %d above the single-pass limit", buckets);
    if (push && buckets > kTileBuckets) return fail(M4D_ERR_USAGE, "push scatter limited to %d buckets", kTileBuckets);
    const int64_t entries = static_cast<int64_t>(ctas) * buckets;
    const int64_t tiles = (entries + kScanTile - 1) / kScanTile;
    uint32_t* hist = static_cast<uint32_t*>(scratch);
    int64_t* offs = reinterpret_cast<int64_t*>(static_cast<char*>(scratch) + ((entries * sizeof(uint32_t) + 255) & ~size_t(255)));
    int64_t* tile_sums = offs + entries;
    int64_t* total = tile_sums + tiles;
    const size_t hist_smem = buckets * sizeof(uint32_t);
    const size_t cur_smem = buckets * sizeof(uint32_t);
    if (phases & kPlan) {
        // (per device; cheap enough to repeat on every call)
        M4D_CUDA_TRY(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 4));
        // a histogram grid of at least 4 x 148 CTAs (kHistThreads each) however few scatter CTAs
        const int split = (4 * 148 + ctas - 1) / ctas;
        if (split > 1) M4D_CUDA_TRY(cudaMemsetAsync(hist, 0, entries * sizeof(uint32_t), s));
        hist_kernel<<<ctas * split, kHistThreads, hist_smem, s>>>(keys, vals, n, run, mode, buckets, log2b, split, hist);
        scan_reduce_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, nullptr);
        scan_tiles_kernel<<<1, 32, 0, s>>>(tile_sums, tiles, total, nullptr);
        scan_apply_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, offs, nullptr);
        bucket_bounds_kernel<<<(buckets + 256) / 256, 256, 0, s>>>(offs, buckets, ctas, n, bounds);
    }
    if (phases & kScatter) {
        if (buckets <= kTileBuckets) {
            if (fine.fine_out)  // counts + the completion counter
                M4D_CUDA_TRY(cudaMemsetAsync(fine.fine_out, 0, static_cast<size_t>(fine.fine_ids + 1) * sizeof(uint32_t), s));
            M4D_CUDA_TRY(launch_tile_scatter(ctas, s, keys, vals, n, run, mode, buckets, log2b, offs,
                                             reinterpret_cast<longlong2*>(out_pairs), push, fine));
        } else {
            M4D_CUDA_TRY(cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 4));
            scatter_kernel<<<ctas, kHistThreads, cur_smem, s>>>(keys, vals, n, run, mode, buckets, log2b, offs,
                                                                reinterpret_cast<longlong2*>(out_pairs));
        }
    }
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

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

int m4d_owner_coarse_count(int world) {
    int c = 1;
    while (world > 0 && world * c * 2 <= 256) c *= 2;
    return c;
}

size_t m4d_partition_scratch_bytes(int64_t n, int buckets) {
    const int64_t ctas = partition_ctas(n);
    const int64_t fan = buckets > kSinglePassMax ? (int64_t(1) << pass1_bits(log2_exact(buckets) < 0 ? 14 : log2_exact(buckets))) : buckets;
    const int64_t entries = ctas * fan;
    const int64_t tiles = (entries + kScanTile - 1) / kScanTile;
    size_t bytes = entries * sizeof(uint32_t) + entries * sizeof(int64_t) + (tiles + 1) * sizeof(int64_t) + 512;
    if (buckets > kSinglePassMax) {  // per-group + global histograms, overflow flag, pass-1 pairs
        int64_t rows = n;
        const int lb = log2_exact(buckets);
        if (lb > 0 && spec_applies(n, static_cast<int>(ctas), static_cast<int>(fan), lb))
            rows = std::max<int64_t>(n, fan * ctas * spec_cap(n, static_cast<int>(ctas), static_cast<int>(fan)));
        bytes += (kMaxGroups + 1) * (buckets * sizeof(unsigned long long) + 256) + 256 + static_cast<size_t>(rows) * 16 + 256;
    }
    return bytes;
}

m4d_status m4d_partition(const int64_t* keys, const int64_t* vals, int64_t n, int mode, int buckets,
                         int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes, void* stream) {
    if (n < 0 || n >= (int64_t(1) << 32)) return fail(M4D_ERR_USAGE, "partition of %lld rows outside [0, 2^32)", (long long)n);
    if (mode == M4D_PART_OWNER_COARSE) return fail(M4D_ERR_USAGE, "owner+coarse partitions go through m4d_partition_owner_coarse");
    const int log2b = log2_exact(buckets);
    const bool two_pass = mode == M4D_PART_LOCAL && buckets > kSinglePassMax;
    if (n < 0 || buckets < 1 || buckets > (mode == M4D_PART_LOCAL ? kMaxParts : kMaxBuckets))
        return fail(M4D_ERR_USAGE, "bucket count %d outside the supported range", buckets);
    if (mode == M4D_PART_LOCAL && log2b < 0) return fail(M4D_ERR_USAGE, "local partition count must be a power of two");
    if (mode != M4D_PART_LOCAL && mode != M4D_PART_RANK) return fail(M4D_ERR_USAGE, "unknown partition mode %d", mode);
    if (scratch_bytes < m4d_partition_scratch_bytes(n, buckets)) return fail(M4D_ERR_USAGE, "partition scratch too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int ctas = partition_ctas(n);
    const int64_t run = (n + ctas - 1) / ctas;
    if (two_pass) {
        const int b1 = pass1_bits(log2b);
        const int fan = 1 << b1;
        const int64_t entries = static_cast<int64_t>(ctas) * fan;
        const int64_t tiles = (entries + kScanTile - 1) / kScanTile;
        char* base = static_cast<char*>(scratch);
        uint32_t* hist = reinterpret_cast<uint32_t*>(base);
        base += (entries * sizeof(uint32_t) + 255) & ~size_t(255);
        int64_t* offs = reinterpret_cast<int64_t*>(base);
        int64_t* tile_sums = offs + entries;
        int64_t* total = tile_sums + tiles;
        base += ((entries + tiles + 1) * sizeof(int64_t) + 255) & ~size_t(255);
        unsigned long long* hist_all = reinterpret_cast<unsigned long long*>(base);
        base += (buckets * sizeof(unsigned long long) + 255) & ~size_t(255);
        unsigned long long* hist_grp = reinterpret_cast<unsigned long long*>(base);
        base += (kMaxGroups * buckets * sizeof(unsigned long long) + 255) & ~size_t(255);
        int* overflow = reinterpret_cast<int*>(base);
        base += 256;
        longlong2* tmp = reinterpret_cast<longlong2*>(base);
        static const int groups = [] {
            const char* v = getenv("M4D_PASS2_GROUPS");
            const int g = v ? atoi(v) : kPass2Groups;
            return g < 1 ? 1 : g > kMaxGroups ? kMaxGroups : g;
        }();
        if (spec_applies(n, ctas, fan, log2b)) {
            // speculative pass 1 (no histogram pass), its gated exact fallback, pass 2 over the regions
            SpecArgs sa;
            sa.cap = spec_cap(n, ctas, fan);
            sa.log2full = log2b;
            sa.groups = groups;
            sa.hist_grp = hist_grp;
            sa.counts = hist;
            sa.overflow = overflow;
            M4D_CUDA_TRY(cudaMemsetAsync(hist_grp, 0, groups * buckets * sizeof(unsigned long long), s));
            M4D_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int), s));
            M4D_CUDA_TRY(launch_tile_scatter(ctas, s, keys, vals, n, run, M4D_PART_LOCAL, fan, b1, nullptr, tmp, nullptr,
                                             sa, true));
            scan_reduce_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, overflow);
            scan_tiles_kernel<<<1, 32, 0, s>>>(tile_sums, tiles, total, overflow);
            scan_apply_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, offs, overflow);
            SpecArgs gate;
            gate.gate = overflow;
            M4D_CUDA_TRY(launch_tile_scatter(ctas, s, keys, vals, n, run, M4D_PART_LOCAL, fan, b1, offs, tmp, nullptr, gate));
            group_prefix_kernel<<<(buckets + 255) / 256, 256, 0, s>>>(hist_grp, groups, buckets, hist_all);
            exclusive_scan_u64_kernel<<<1, 1024, 0, s>>>(hist_all, buckets, bounds, n);
            spec_pass2_kernel<<<fan * groups, 1024, (buckets >> b1) * sizeof(uint32_t), s>>>(
                tmp, hist, offs, overflow, sa.cap, ctas, hist_grp, groups, bounds, log2b, b1,
                reinterpret_cast<longlong2*>(out_pairs), l2_pf());
            M4D_CUDA_TRY(cudaGetLastError());
            return M4D_OK;
        }
        const bool packed = buckets > (1 << 15);
        const size_t hist_smem = packed ? (buckets + 1) / 2 * sizeof(uint32_t) : buckets * sizeof(uint32_t);
        M4D_CUDA_TRY(cudaFuncSetAttribute(hist2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxParts * 2));
        M4D_CUDA_TRY(cudaFuncSetAttribute(hist2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxParts * 2));
        M4D_CUDA_TRY(cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxBuckets * 4));
        M4D_CUDA_TRY(cudaMemsetAsync(hist_grp, 0, groups * buckets * sizeof(unsigned long long), s));
        (packed ? hist2_kernel<true> : hist2_kernel<false>)<<<ctas, 1024, hist_smem, s>>>(keys, vals, n, run, log2b, b1,
                                                                                        groups, hist, hist_grp, l2_pf());
        scan_reduce_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, nullptr);
        scan_tiles_kernel<<<1, 32, 0, s>>>(tile_sums, tiles, total, nullptr);
        scan_apply_kernel<<<static_cast<unsigned>(tiles), 1024, 0, s>>>(hist, entries, tile_sums, offs, nullptr);
        // pass 1: by the top b1 bits of the partition id (mode LOCAL with 2^b1 buckets == those bits)
        M4D_CUDA_TRY(launch_tile_scatter(ctas, s, keys, vals, n, run, M4D_PART_LOCAL, fan, b1, offs, tmp));
        group_prefix_kernel<<<(buckets + 255) / 256, 256, 0, s>>>(hist_grp, groups, buckets, hist_all);
        exclusive_scan_u64_kernel<<<1, 1024, 0, s>>>(hist_all, buckets, bounds, n);
        scatter_pass2_kernel<<<fan * groups, 1024, (buckets >> b1) * sizeof(uint32_t), s>>>(
            tmp, offs, ctas, n, hist_grp, groups, bounds, log2b, b1, reinterpret_cast<longlong2*>(out_pairs),
            l2_pf());
        M4D_CUDA_TRY(cudaGetLastError());
        return M4D_OK;
    }
    return partition_single(keys, vals, n, mode, buckets, log2b, out_pairs, bounds, scratch, scratch_bytes, s);
}

m4d_status m4d_partition_owner_coarse(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                      int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes,
                                      void* stream) {
    if (n < 0 || n >= (int64_t(1) << 32)) return fail(M4D_ERR_USAGE, "partition of %lld rows outside [0, 2^32)", (long long)n);
    if (world < 1 || world > 256) return fail(M4D_ERR_USAGE, "owner count %d outside [1, 256]", world);
    const int cbits = log2_exact(coarse);
    if (cbits < 0 || world * coarse > 256) return fail(M4D_ERR_USAGE, "coarse count %d invalid for %d owners", coarse, world);
    return partition_single(keys, vals, n, M4D_PART_OWNER_COARSE, world * coarse, cbits, out_pairs, bounds, scratch,
                            scratch_bytes, static_cast<cudaStream_t>(stream));
}

static m4d_status owner_coarse_check(int64_t n, int world, int coarse, int* cbits) {
    if (n < 0 || n >= (int64_t(1) << 32)) return fail(M4D_ERR_USAGE, "partition of %lld rows outside [0, 2^32)", (long long)n);
    if (world < 1 || world > 256) return fail(M4D_ERR_USAGE, "owner count %d outside [1, 256]", world);
    *cbits = log2_exact(coarse);
    if (*cbits < 0 || world * coarse > 256) return fail(M4D_ERR_USAGE, "coarse count %d invalid for %d owners", coarse, world);
    return M4D_OK;
}

m4d_status m4d_partition_owner_plan(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                    int64_t* bounds, void* scratch, size_t scratch_bytes, void* stream) {
    int cbits = 0;
    const m4d_status st = owner_coarse_check(n, world, coarse, &cbits);
    if (st != M4D_OK) return st;
    return partition_single(keys, vals, n, M4D_PART_OWNER_COARSE, world * coarse, cbits, nullptr, bounds, scratch,
                            scratch_bytes, static_cast<cudaStream_t>(stream), kPlan, nullptr, true);
}

m4d_status m4d_partition_owner_push(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                    const uint64_t* seg_dest, void* scratch, size_t scratch_bytes, void* stream) {
    int cbits = 0;
    const m4d_status st = owner_coarse_check(n, world, coarse, &cbits);
    if (st != M4D_OK) return st;
    if (world > kMaxPushOwners) return fail(M4D_ERR_USAGE, "push scatter limited to %d owners", kMaxPushOwners);
    if (!seg_dest) return fail(M4D_ERR_USAGE, "null push destinations");
    PushTargets push{};
    for (int d = 0; d < world; ++d) push.seg[d] = reinterpret_cast<longlong2*>(seg_dest[d]);
    return partition_single(keys, vals, n, M4D_PART_OWNER_COARSE, world * coarse, cbits, nullptr, nullptr, scratch,
                            scratch_bytes, static_cast<cudaStream_t>(stream), kScatter, &push, true);
}

size_t m4d_push_fine_smem_limit(void) {
    // shared memory the push scatter CTA (M4D_PUSH_TILE_THREADS) leaves for 16-bit fine counters
    const size_t tile = push_tile_threads() == 256 ? tile_smem<256>() : push_tile_threads() == 512 ? tile_smem<512>()
                                                                                                   : tile_smem<1024>();
    const size_t cap = 227 * 1024 - 8192;  // (static shared memory of the kernel: cursors, push pointers)
    return cap > tile ? cap - tile : 0;
}

m4d_status m4d_partition_owner_push_fine(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                         const uint64_t* seg_dest, int parts, uint32_t* fine_out,
                                         const uint64_t* count_dest, void* scratch, size_t scratch_bytes,
                                         void* stream) {
    int cbits = 0;
    const m4d_status st = owner_coarse_check(n, world, coarse, &cbits);
    if (st != M4D_OK) return st;
    const int pbits = log2_exact(parts);
    if (world > kMaxPushOwners) return fail(M4D_ERR_USAGE, "push scatter limited to %d owners", kMaxPushOwners);
    if (!seg_dest || !fine_out) return fail(M4D_ERR_USAGE, "null push destinations or counts");
    if (pbits < 1 || static_cast<size_t>(world) * parts * 2 > m4d_push_fine_smem_limit())
        return fail(M4D_ERR_USAGE, "%d owners x %d partitions of 16-bit counters do not fit the push CTA", world, parts);
    if (!tile_rank_atomic()) return fail(M4D_ERR_USAGE, "fused fine counts need atomic tile ranking");
    PushTargets push{};
    for (int d = 0; d < world; ++d) push.seg[d] = reinterpret_cast<longlong2*>(seg_dest[d]);
    SpecArgs fine;
    fine.fine_out = fine_out;
    fine.fine_ids = world * parts;
    fine.log2full = pbits;
    for (int d = 0; d < world && count_dest; ++d) fine.fine_dst[d] = reinterpret_cast<uint32_t*>(count_dest[d]);
    return partition_single(keys, vals, n, M4D_PART_OWNER_COARSE, world * coarse, cbits, nullptr, nullptr, scratch,
                            scratch_bytes, static_cast<cudaStream_t>(stream), kScatter, &push, true, fine);
}

// Join variant (M4D_JOIN = big | small, default big): see kSmallThreads.
static bool join_small() {
    static const bool b = [] {
        const char* v = getenv("M4D_JOIN");
        return v && strcmp(v, "small") == 0;
    }();
    return b;
}

// Join grid: one CTA per partition, or (M4D_JOIN_PERSIST=1) one wave of
// persistent CTAs that walk the partitions and prefetch the next one into L2.
static int join_pf() {
    static const int v = [] {
        // default 3: 1.75 -> 1.58 ms per join at 1e8 rows/side (tools/km_join_pf_sweep.sh;
        // the look-ahead bit 4 made it slower: 1.8-2.1 ms)
        const char* e = getenv("M4D_JOIN_PF");
        return e ? atoi(e) & 7 : 3;
    }();
    return v;
}

static int join_pf_ahead() {
    static const int v = [] {
        const char* e = getenv("M4D_JOIN_PF_AHEAD");
        return e && atoi(e) > 0 ? atoi(e) : 148;
    }();
    return v;
}

// Matches per probe row the count walk keeps, so staging them needs no second walk
// of the chain (M4D_JOIN_KEEP = 1..3, default 2).  Same box, 1e8 rows/side
// (tools/sweeps/r2_join_second.sh): f = 0.3 join 1.58 / 1.52 / 1.54 ms, f = 1.0
// 2.50 / 2.47 / 2.38 ms for 1 / 2 / 3.
static int join_keep() {
    static const int v = [] {
        const char* e = getenv("M4D_JOIN_KEEP");
        const int x = e ? atoi(e) : 2;
        return x < 1 ? 1 : x > 3 ? 3 : x;
    }();
    return v;
}

static int join_grid(int parts, int per_sm) {
    static const bool persist = [] {
        const char* v = getenv("M4D_JOIN_PERSIST");
        return v && atoi(v) == 1;
    }();
    return persist && parts > 148 * per_sm ? 148 * per_sm : parts;
}

// Row ranges per (coarse run, source) piece of the receiver split: about 8 CTAs
// of 1024 threads per SM in total, at most kMaxRunGroups.
constexpr int kMaxRunGroups = 64;
static int runs_groups(int coarse, int sources) {
    const int pieces = coarse * sources;
    static const int per_sm = [] {
        const char* v = getenv("M4D_RUNS_CTAS_PER_SM");
        const int x = v ? atoi(v) : 8;
        return x < 1 ? 1 : x > 64 ? 64 : x;
    }();
    int g = (148 * per_sm + pieces - 1) / pieces;
    return g < 1 ? 1 : g > kMaxRunGroups ? kMaxRunGroups : g;
}

size_t m4d_partition_runs_scratch_bytes(int sources, int buckets, int coarse) {
    if (sources < 1 || buckets < 1 || coarse < 1) return 0;
    return (static_cast<size_t>(sources) * kMaxRunGroups + 1) * buckets * sizeof(unsigned long long) +
           2 * static_cast<size_t>(coarse) * sources * sizeof(int64_t) + 1024;
}

m4d_status m4d_partition_runs(const int64_t* in_pairs, int64_t n, const int64_t* runs_host, int coarse, int sources,
                              int buckets, int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes,
                              void* stream) {
    const int log2b = log2_exact(buckets), cbits = log2_exact(coarse);
    if (n < 0 || n >= (int64_t(1) << 32)) return fail(M4D_ERR_USAGE, "partition of %lld rows outside [0, 2^32)", (long long)n);
    if (log2b < 0 || buckets > (1 << 15)) return fail(M4D_ERR_USAGE, "partition count %d must be a power of two <= 32768", buckets);
    if (cbits < 0 || coarse > buckets || coarse > 256) return fail(M4D_ERR_USAGE, "coarse run count %d invalid", coarse);
    if (sources < 1 || sources > 256) return fail(M4D_ERR_USAGE, "source count %d outside [1, 256]", sources);
    if (scratch_bytes < m4d_partition_runs_scratch_bytes(sources, buckets, coarse))
        return fail(M4D_ERR_USAGE, "partition scratch too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int groups = runs_groups(coarse, sources);
    char* base = static_cast<char*>(scratch);
    unsigned long long* hist_grp = reinterpret_cast<unsigned long long*>(base);               // [sources][groups][buckets]
    unsigned long long* hist_all = hist_grp + static_cast<int64_t>(sources) * groups * buckets;  // [buckets]
    int64_t* runs = reinterpret_cast<int64_t*>(hist_grp + (static_cast<int64_t>(sources) * kMaxRunGroups + 1) * buckets);
    const size_t run_bytes = 2 * static_cast<size_t>(coarse) * sources * sizeof(int64_t);
    M4D_CUDA_TRY(cudaMemcpyAsync(runs, runs_host, run_bytes, cudaMemcpyHostToDevice, s));
    const int ctas = coarse * sources * groups;
    const size_t sub_smem = static_cast<size_t>(buckets >> cbits) * sizeof(uint32_t);
    runs_hist_kernel<<<ctas, runs_threads(), sub_smem, s>>>(reinterpret_cast<const longlong2*>(in_pairs), runs, sources, groups,
                                                  log2b, cbits, hist_grp, l2_pf());
    group_prefix_kernel<<<(buckets + 255) / 256, 256, 0, s>>>(hist_grp, sources * groups, buckets, hist_all);
    exclusive_scan_u64_kernel<<<1, 1024, 0, s>>>(hist_all, buckets, bounds, n);
    runs_pass2_kernel<<<ctas, runs_threads(), sub_smem, s>>>(reinterpret_cast<const longlong2*>(in_pairs), runs, sources, groups,
                                                   hist_grp, bounds, log2b, cbits,
                                                   reinterpret_cast<longlong2*>(out_pairs), l2_pf());
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

m4d_status m4d_partition_fine_counts(const int64_t* keys, const int64_t* vals, int64_t n, int world, int buckets,
                                     uint32_t* out_counts, void* stream) {
    const int log2b = log2_exact(buckets);
    if (n < 0 || world < 1 || log2b < 1) return fail(M4D_ERR_USAGE, "invalid fine-count request");
    const size_t smem = static_cast<size_t>(world) * buckets * sizeof(uint16_t);
    if (smem > m4d_fine_count_smem_limit()) return fail(M4D_ERR_USAGE, "%d owners x %d partitions exceed the counters a CTA holds", world, buckets);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    M4D_CUDA_TRY(cudaMemsetAsync(out_counts, 0, static_cast<size_t>(world) * buckets * sizeof(uint32_t), s));
    if (!n) return M4D_OK;
    M4D_CUDA_TRY(cudaFuncSetAttribute(fine_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int dev = 0, sms = 148;
    M4D_CUDA_TRY(cudaGetDevice(&dev));
    M4D_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    fine_count_kernel<<<sms, 1024, smem, s>>>(keys, vals, n, world, log2b, out_counts, l2_pf());
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

size_t m4d_fine_count_smem_limit(void) { return 200 * 1024; }

m4d_status m4d_partition_runs_counted(const int64_t* in_pairs, int64_t n, const int64_t* runs_host, int coarse,
                                      int sources, int buckets, const uint32_t* fine_in, int64_t* out_pairs,
                                      int64_t* bounds, void* scratch, size_t scratch_bytes, void* stream) {
    const int log2b = log2_exact(buckets), cbits = log2_exact(coarse);
    if (n < 0 || n >= (int64_t(1) << 32)) return fail(M4D_ERR_USAGE, "partition of %lld rows outside [0, 2^32)", (long long)n);
    if (log2b < 0 || buckets > (1 << 15)) return fail(M4D_ERR_USAGE, "partition count %d must be a power of two <= 32768", buckets);
    if (cbits < 0 || coarse > buckets || coarse > 256) return fail(M4D_ERR_USAGE, "coarse run count %d invalid", coarse);
    if (sources < 1 || sources > 256) return fail(M4D_ERR_USAGE, "source count %d outside [1, 256]", sources);
    if (scratch_bytes < m4d_partition_runs_scratch_bytes(sources, buckets, coarse))
        return fail(M4D_ERR_USAGE, "partition scratch too small");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* base = static_cast<char*>(scratch);
    unsigned long long* grp_before = reinterpret_cast<unsigned long long*>(base);                // [sources][buckets]
    unsigned long long* hist_all = grp_before + static_cast<int64_t>(sources) * buckets;        // [buckets]
    int64_t* runs = reinterpret_cast<int64_t*>(grp_before + (static_cast<int64_t>(sources) * kMaxRunGroups + 1) * buckets);
    const size_t run_bytes = 2 * static_cast<size_t>(coarse) * sources * sizeof(int64_t);
    M4D_CUDA_TRY(cudaMemcpyAsync(runs, runs_host, run_bytes, cudaMemcpyHostToDevice, s));
    fine_prefix_kernel<<<(buckets + 255) / 256, 256, 0, s>>>(fine_in, sources, buckets, grp_before, hist_all);
    exclusive_scan_u64_kernel<<<1, 1024, 0, s>>>(hist_all, buckets, bounds, n);
    const size_t sub_smem = static_cast<size_t>(buckets >> cbits) * sizeof(uint32_t);
    runs_pass2_kernel<<<coarse * sources, runs_threads(), sub_smem, s>>>(reinterpret_cast<const longlong2*>(in_pairs), runs,
                                                                       sources, 1, grp_before, bounds, log2b, cbits,
                                                                       reinterpret_cast<longlong2*>(out_pairs), l2_pf());
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}


int m4d_join_partition_rows(void) {
    // M4D_JOIN_PART_ROWS overrides the target rows per partition (the small join
    // then builds a 12K-row partition in two chunks, re-reading probe rows from L2).
    static const int rows = [] {
        const char* v = getenv("M4D_JOIN_PART_ROWS");
        return v && atoi(v) > 0 ? atoi(v) : 0;
    }();
    return rows ? rows : join_small() ? 6200 : 12400;
}

int m4d_partition_launches(int buckets) { return buckets > kSinglePassMax ? 9 : 6; }

m4d_status m4d_hash_join(const int64_t* lpairs, const int64_t* lbounds, const int64_t* rpairs,
                         const int64_t* rbounds, int parts, int64_t* out_keys, int64_t* out_lvals,
                         int64_t* out_rvals, int64_t capacity, unsigned long long* result, void* stream) {
    if (parts < 0) return fail(M4D_ERR_USAGE, "negative partition count");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // result = {cursor, count, hash_sum, key_sum}
    M4D_CUDA_TRY(cudaMemsetAsync(result, 0, 4 * sizeof(unsigned long long), s));
    if (parts) {
        const longlong2* lp = reinterpret_cast<const longlong2*>(lpairs);
        const longlong2* rp = reinterpret_cast<const longlong2*>(rpairs);
        if (join_small()) {
            auto k = join_kernel<kSmallThreads, kSmallSlotBits, kSmallChunk, kSmallStage, 2, 3>;
            M4D_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmallSmem)));
            k<<<join_grid(parts, 2), kSmallThreads, kSmallSmem, s>>>(lp, lbounds, rp, rbounds, out_keys, out_lvals,
                                                                     out_rvals, capacity, result, result + 1, parts, join_pf(),
                                                                     join_pf_ahead());
        } else {
            auto k = join_keep() == 1 ? join_kernel<kJoinThreads, kSlotBits, kChunk, kStage, 1, 1>
                     : join_keep() == 2 ? join_kernel<kJoinThreads, kSlotBits, kChunk, kStage, 1, 2>
                                        : join_kernel<kJoinThreads, kSlotBits, kChunk, kStage, 1, 3>;
            M4D_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kJoinSmem)));
            k<<<join_grid(parts, 1), kJoinThreads, kJoinSmem, s>>>(lp, lbounds, rp, rbounds, out_keys, out_lvals,
                                                                   out_rvals, capacity, result, result + 1, parts, join_pf(),
                                                                   join_pf_ahead());
        }
    }
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

}  // extern "C"
