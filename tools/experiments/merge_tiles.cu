// key_merge, tile-local layout (K5' partition + K7' join; SPEC.md:422-430,
// PAPER.md:387-389).
//
// Partition (m4d_tile_partition): the input rows are cut into tiles of
// kTileRows rows (a tile never crosses an input segment).  Each tile is
// counting-sorted by its LOCAL partition id in shared memory and written back
// to the SAME rows of the output, so the pass reads and writes HBM strictly
// sequentially (no global histogram, no scan kernels, no write frontier in
// L2).  Per tile and partition it records the run's start row (u16) -- first
// as [p / 16][tile][p % 16] (full 32-byte sectors per tile), then transposed
// to meta[p][tile] so one join CTA reads its partition's starts contiguously.
// The next tile's keys/payloads stream into the second of two shared-memory
// buffers (TMA bulk copies, mbarrier completion) while the current tile is
// ranked; rows are never staged: a u16 permutation maps sorted positions to
// tile rows for the copy-out.
//
// Join (m4d_tile_join): one CTA per partition gathers its build rows (runs of
// ~1 row per tile) into a chained hash table in shared memory -- per row a
// 32-bit fingerprint, its global row position and a 16-bit link, 16384 chain
// heads; partitions above kChunk build rows are joined in balanced chunks --
// then streams its probe rows through it in rounds of up to 4096 rows.  A
// fingerprint match is a candidate; the emit step loads the build row, keeps
// the exact key matches (ballot), reserves output rows with one atomic per
// warp round and writes (key, lval, rval) plus the order-independent digest
// (K8: count, sum of row hashes, sum of keys, mod 2^64).
#include <cuda_runtime.h>

#include <cstring>

#include "m4d_internal.h"
#include "ptx.cuh"

namespace {

constexpr int kTileRows = 4096;          // rows per tile (u16 starts)
constexpr int kSortThreads = 1024;
constexpr int kSortPer = kTileRows / kSortThreads;
constexpr int kMaxTileParts = 8192;
constexpr int kMaxSegs = 64;

struct Segs {
    int n;
    int64_t off[kMaxSegs];     // first row of segment s
    int64_t rows[kMaxSegs];    // rows of segment s
    int64_t tile0[kMaxSegs + 1];  // first tile of segment s (tile0[n] = tiles)
};

__device__ __forceinline__ uint32_t part_of(int64_t key, int log2p) {
    const uint64_t h = m4d_splitmix64(static_cast<uint64_t>(key));
    return log2p ? static_cast<uint32_t>((h & 0xffffffffull) >> (32 - log2p)) : 0u;
}

// Tile t -> (first row, rows).
__device__ __forceinline__ void tile_geom(const Segs& sg, int64_t t, int64_t* base, int* rows) {
    int s = 0;
    while (s + 1 < sg.n && sg.tile0[s + 1] <= t) ++s;
    const int64_t first = (t - sg.tile0[s]) * kTileRows;
    const int64_t left = sg.rows[s] - first;
    *base = sg.off[s] + first;
    *rows = static_cast<int>(left < kTileRows ? left : kTileRows);
}

// TMA bulk copies need 16-byte aligned sources and sizes: SoA tiles at an odd
// row or with an odd row count are copied by the threads instead.
template <bool kPairs>
__device__ __forceinline__ bool tile_tma_ok(int64_t base, int rows) {
    return kPairs || ((base | rows) & 1) == 0;
}

__device__ __forceinline__ int64_t staged_meta_index(int64_t tiles, int p, int64_t t) {
    return ((static_cast<int64_t>(p >> 4) * tiles + t) << 4) + (p & 15);
}

// Persistent tile sort: CTA b sorts tiles b, b + grid, ...  kPairs: input rows
// are 16-byte (key, payload) pairs at `keys`; else SoA columns keys / vals.
template <bool kPairs>
__global__ void __launch_bounds__(kSortThreads, 1)
    tile_sort_kernel(const int64_t* __restrict__ keys, const int64_t* __restrict__ vals, const __grid_constant__ Segs sg,
                     int64_t tiles, int log2p, longlong2* __restrict__ out, uint16_t* __restrict__ staged) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int P = 1 << log2p;
    // two input buffers: SoA [2][keys kTileRows | vals kTileRows] or pairs [2][kTileRows]
    int64_t* in = reinterpret_cast<int64_t*>(sm);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(in + 4 * kTileRows);  // [P]
    uint16_t* perm = reinterpret_cast<uint16_t*>(cnt + (P > kSortThreads ? P : kSortThreads));  // [kTileRows]
    __shared__ uint64_t bar[2];
    __shared__ uint32_t wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = P >= kSortThreads ? P / kSortThreads : 1;  // partitions per scan thread
    const bool scan_lane = threadIdx.x * per < P;
    for (int b = threadIdx.x; b < P; b += kSortThreads) cnt[b] = 0;
    if (threadIdx.x == 0) {
        m4d::ptx::mbar_init(&bar[0], 1);
        m4d::ptx::mbar_init(&bar[1], 1);
        m4d::ptx::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t, int slot) {
        int64_t base;
        int rows;
        tile_geom(sg, t, &base, &rows);
        if (!tile_tma_ok<kPairs>(base, rows)) return;
        int64_t* dst = in + slot * 2 * kTileRows;
        m4d::ptx::mbar_arrive_expect_tx(&bar[slot], static_cast<uint32_t>(rows) * 16u);
        if (kPairs) {
            m4d::ptx::bulk_g2s(dst, keys + 2 * base, rows * 16u, &bar[slot]);
        } else {
            m4d::ptx::bulk_g2s(dst, keys + base, rows * 8u, &bar[slot]);
            m4d::ptx::bulk_g2s(dst + kTileRows, vals + base, rows * 8u, &bar[slot]);
        }
    };
    int64_t t = blockIdx.x;
    if (threadIdx.x == 0 && t < tiles) issue(t, 0);
    uint32_t phase = 0;  // bit s: parity of buffer s
    for (int it = 0; t < tiles; t += gridDim.x, ++it) {
        const int slot = it & 1;
        // the other buffer was released by the previous iteration's last barrier
        if (threadIdx.x == 0 && t + gridDim.x < tiles) issue(t + gridDim.x, slot ^ 1);
        int64_t base;
        int rem;
        tile_geom(sg, t, &base, &rem);
        int64_t* buf = in + slot * 2 * kTileRows;
        if (tile_tma_ok<kPairs>(base, rem)) {
            m4d::ptx::mbar_wait(&bar[slot], (phase >> slot) & 1u);
            phase ^= 1u << slot;
        } else {
            for (int r = threadIdx.x; r < rem; r += kSortThreads) {
                buf[r] = keys[base + r];
                buf[kTileRows + r] = vals[base + r];
            }
            __syncthreads();
        }
        uint32_t b[kSortPer], rk[kSortPer];
#pragma unroll
        for (int u = 0; u < kSortPer; ++u) {
            const int r = u * kSortThreads + threadIdx.x;
            if (r < rem) {
                const int64_t key = kPairs ? buf[2 * r] : buf[r];
                b[u] = part_of(key, log2p);
                rk[u] = atomicAdd(&cnt[b[u]], 1u);
            }
        }
        __syncthreads();
        // exclusive scan of the counts: thread i owns partitions [i * per, i * per + per)
        uint32_t c[kMaxTileParts / kSortThreads], loc = 0;
#pragma unroll
        for (int q = 0; q < kMaxTileParts / kSortThreads; ++q) {
            c[q] = (q < per && scan_lane) ? cnt[threadIdx.x * per + q] : 0u;
            loc += c[q];
        }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            const uint32_t x = wsum[lane];
            uint32_t xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            wsum[lane] = xi - x;
        }
        __syncthreads();
        if (scan_lane) {
            uint32_t run = wsum[w] + incl - loc;
#pragma unroll
            for (int q = 0; q < kMaxTileParts / kSortThreads; ++q) {
                if (q < per) {
                    const int p = threadIdx.x * per + q;
                    cnt[p] = run;  // now the run start
                    staged[staged_meta_index(tiles, p, t)] = static_cast<uint16_t>(run);
                    run += c[q];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kSortPer; ++u) {
            const int r = u * kSortThreads + threadIdx.x;
            if (r < rem) perm[cnt[b[u]] + rk[u]] = static_cast<uint16_t>(r);
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kSortPer; ++u) {
            const int r = u * kSortThreads + threadIdx.x;
            if (r < rem) {
                const int i = perm[r];
                longlong2 x;
                if (kPairs) {
                    x = reinterpret_cast<const longlong2*>(buf)[i];
                } else {
                    x.x = buf[i];
                    x.y = buf[kTileRows + i];
                }
                __stcs(out + base + r, x);
            }
        }
        for (int q = threadIdx.x; q < P; q += kSortThreads) cnt[q] = 0;
        __syncthreads();  // buffer `slot` and the counts are free again
    }
}

// staged[p / 16][tile][p % 16] -> meta[p][tile]: one CTA per (group of 16
// partitions, 1024 tiles).
constexpr int kTrTiles = 1024;
__global__ void __launch_bounds__(512) meta_transpose_kernel(const uint16_t* __restrict__ staged, int64_t tiles, int parts,
                                                             uint16_t* __restrict__ meta) {
    __shared__ uint16_t s[16][kTrTiles + 2];
    const int g = blockIdx.y;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTrTiles;
    const int nt = static_cast<int>(tiles - t0 < kTrTiles ? tiles - t0 : kTrTiles);
    const uint16_t* src = staged + (static_cast<int64_t>(g) * tiles + t0) * 16;
    for (int i = threadIdx.x; i < nt * 16; i += blockDim.x) s[i & 15][i >> 4] = src[i];
    __syncthreads();
    const int pn = parts - g * 16 < 16 ? parts - g * 16 : 16;
    for (int q = 0; q < pn; ++q) {
        uint16_t* dst = meta + static_cast<int64_t>(g * 16 + q) * tiles + t0;
        for (int i = threadIdx.x; i < nt; i += blockDim.x) dst[i] = s[q][i];
    }
}

// ---- join ----------------------------------------------------------------------------

constexpr int kJoinThreads = 1024;
constexpr int kHeadBits = 14;
constexpr int kHeads = 1 << kHeadBits;
constexpr int kChunk = 13000;        // build rows per table
constexpr int kRound = 4096;         // probe rows per round (ppos buffer)
constexpr int kStage = 128;          // staged candidates per warp per emit round
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr uint16_t kNil = 0xffffu;
constexpr int kIdxBits = 14;
constexpr size_t kJoinSmem = kHeads * 4 + static_cast<size_t>(kChunk) * (4 + 4 + 2) + kRound * 4 +
                             (kJoinThreads / 32) * kStage * 4;
static_assert(kChunk < (1 << kIdxBits) && kIdxBits + 12 <= 32, "candidate packing");
static_assert(kJoinSmem <= 227 * 1024 - 2048, "join shared memory");

__device__ __forceinline__ uint64_t row_hash(int64_t k, int64_t l, int64_t r) {
    uint64_t h = m4d_splitmix64(static_cast<uint64_t>(k) ^ 0x6B65795F6D657267ull);
    h = m4d_splitmix64(h ^ static_cast<uint64_t>(l));
    return m4d_splitmix64(h ^ (static_cast<uint64_t>(r) * 0x9E3779B97F4A7C15ull));
}

// Table slot and fingerprint from one multiplicative hash (disjoint bit
// ranges; independent of the splitmix64 partition bits).  Equal keys always
// agree; a fingerprint match is confirmed on the full key at emit time.
__device__ __forceinline__ void slot_fp(int64_t key, uint32_t* slot, uint32_t* fp) {
    const uint64_t x = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull;
    *slot = static_cast<uint32_t>(x >> (64 - kHeadBits));
    *fp = static_cast<uint32_t>(x >> 18);
}

struct JoinSide {
    const longlong2* rows;
    const uint16_t* meta;  // [parts][tiles]
    int64_t tiles;
    Segs sg;
};

// Block-wide exclusive scan of v (1024 threads); returns the exclusive prefix, *total the sum.
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* wsum, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = wsum[lane];
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        wsum[lane] = xi - x;
        if (lane == 31) wsum[32] = xi;
    }
    __syncthreads();
    const uint32_t r = wsum[w] + incl - v;
    *total = wsum[32];
    __syncthreads();  // wsum reusable
    return r;
}

// Run of partition p in tile t of one side: [*a, *z) rows relative to *base.
__device__ __forceinline__ void run_of(const JoinSide& sd, int p, int parts, int64_t t, int64_t* base, int* a, int* z) {
    int rows;
    tile_geom(sd.sg, t, base, &rows);
    *a = sd.meta[static_cast<int64_t>(p) * sd.tiles + t];
    *z = p + 1 < parts ? sd.meta[static_cast<int64_t>(p + 1) * sd.tiles + t] : rows;
}

constexpr int kWalkTiles = 4;  // tiles per thread per walk round

__global__ void __launch_bounds__(kJoinThreads, 1)
    tile_join_kernel(const __grid_constant__ JoinSide L, const __grid_constant__ JoinSide R, int parts,
                     int64_t* __restrict__ ok, int64_t* __restrict__ ol, int64_t* __restrict__ orr, int64_t capacity,
                     unsigned long long* __restrict__ result) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* head = reinterpret_cast<uint32_t*>(smem);          // [kHeads]
    uint32_t* bfp = head + kHeads;                                // [kChunk]
    uint32_t* bpos = bfp + kChunk;                                // [kChunk] global row of the build row
    uint32_t* ppos = bpos + kChunk;                               // [kRound]
    uint32_t* stage_all = ppos + kRound;                          // [warps][kStage]
    uint16_t* link = reinterpret_cast<uint16_t*>(stage_all + (kJoinThreads / 32) * kStage);  // [kChunk]
    __shared__ uint32_t wsum[33];
    __shared__ unsigned long long red[kJoinThreads / 32][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* stage = stage_all + warp * kStage;
    unsigned long long cnt = 0, hsum = 0, ksum = 0;
    unsigned long long* cursor = result;
    const int p = blockIdx.x;

    // build rows of this partition (sum of the runs over every build tile)
    uint32_t mine = 0;
    for (int64_t t = threadIdx.x; t < L.tiles; t += kJoinThreads) {
        int64_t base;
        int a, z;
        run_of(L, p, parts, t, &base, &a, &z);
        mine += static_cast<uint32_t>(z - a);
    }
    uint32_t bn = 0;
    block_scan(mine, wsum, &bn);
    const uint32_t nch = (bn + kChunk - 1) / kChunk;
    const uint32_t csz = nch ? (bn + nch - 1) / nch : 0;

    for (uint32_t ch = 0; ch < nch; ++ch) {
        const uint32_t c0 = ch * csz, cn = bn - c0 < csz ? bn - c0 : csz;
        for (int s = threadIdx.x; s < kHeads; s += kJoinThreads) head[s] = kEmpty;
        // (a) positions of this chunk's build rows, in (tile, row) order
        uint32_t dense0 = 0;
        for (int64_t t0 = 0; t0 < L.tiles; t0 += static_cast<int64_t>(kJoinThreads) * kWalkTiles) {
            int64_t base[kWalkTiles];
            int a[kWalkTiles], z[kWalkTiles];
            uint32_t len = 0;
#pragma unroll
            for (int u = 0; u < kWalkTiles; ++u) {
                const int64_t t = t0 + static_cast<int64_t>(threadIdx.x) * kWalkTiles + u;
                a[u] = z[u] = 0;
                base[u] = 0;
                if (t < L.tiles) run_of(L, p, parts, t, &base[u], &a[u], &z[u]);
                len += static_cast<uint32_t>(z[u] - a[u]);
            }
            uint32_t total;
            uint32_t d = dense0 + block_scan(len, wsum, &total);
            if (d < c0 + cn && d + len > c0) {
#pragma unroll
                for (int u = 0; u < kWalkTiles; ++u)
                    for (int r = a[u]; r < z[u]; ++r, ++d)
                        if (d >= c0 && d < c0 + cn) bpos[d - c0] = static_cast<uint32_t>(base[u] + r);
            }
            dense0 += total;
            if (dense0 >= c0 + cn) break;  // block-uniform
        }
        __syncthreads();
        // (b) load the rows, insert: one atomicExch per row on its chain head
        for (uint32_t i0 = 0; i0 < cn; i0 += kJoinThreads * 4) {
            int64_t k[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * kJoinThreads + threadIdx.x;
                k[u] = i < cn ? L.rows[bpos[i]].x : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * kJoinThreads + threadIdx.x;
                if (i >= cn) break;
                uint32_t slot, fp;
                slot_fp(k[u], &slot, &fp);
                bfp[i] = fp;
                const uint32_t old = atomicExch(&head[slot], i);
                link[i] = old == kEmpty ? kNil : static_cast<uint16_t>(old);
            }
        }
        __syncthreads();
        // (c) probe rounds: up to kWalkTiles * 1024 probe tiles, cut into sub-rounds of kRound rows
        for (int64_t t0 = 0; t0 < R.tiles; t0 += static_cast<int64_t>(kJoinThreads) * kWalkTiles) {
            int64_t base[kWalkTiles];
            int a[kWalkTiles], z[kWalkTiles];
            uint32_t len = 0;
#pragma unroll
            for (int u = 0; u < kWalkTiles; ++u) {
                const int64_t t = t0 + static_cast<int64_t>(threadIdx.x) * kWalkTiles + u;
                a[u] = z[u] = 0;
                base[u] = 0;
                if (t < R.tiles) run_of(R, p, parts, t, &base[u], &a[u], &z[u]);
                len += static_cast<uint32_t>(z[u] - a[u]);
            }
            uint32_t total;
            const uint32_t my0 = block_scan(len, wsum, &total);
            for (uint32_t s0 = 0; s0 < total; s0 += kRound) {
                const uint32_t sn = total - s0 < kRound ? total - s0 : kRound;
                if (my0 < s0 + sn && my0 + len > s0) {
                    uint32_t d = my0;
#pragma unroll
                    for (int u = 0; u < kWalkTiles; ++u)
                        for (int r = a[u]; r < z[u]; ++r, ++d)
                            if (d >= s0 && d < s0 + sn) ppos[d - s0] = static_cast<uint32_t>(base[u] + r);
                }
                __syncthreads();
                // probe the sub-round: thread owns rows threadIdx.x + u * 1024
                int64_t rk[4];
                uint32_t info[4];  // first candidate | min(candidates, 0xffff) << 16
                uint32_t fpv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t j = u * kJoinThreads + threadIdx.x;
                    rk[u] = j < sn ? R.rows[ppos[j]].x : 0;
                }
                uint32_t cand = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    info[u] = 0;
                    const uint32_t j = u * kJoinThreads + threadIdx.x;
                    if (j >= sn) continue;
                    uint32_t slot;
                    slot_fp(rk[u], &slot, &fpv[u]);
                    uint32_t c = 0, first = 0;
                    const uint32_t h0 = head[slot];
                    for (uint32_t i = h0 == kEmpty ? kNil : h0; i != kNil; i = link[i])
                        if (bfp[i] == fpv[u]) {
                            first = c ? first : i;
                            ++c;
                        }
                    info[u] = first | (c < 0xffffu ? c : 0xffffu) << 16;
                    cand += c;
                }
                uint32_t incl = cand;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t warp_total = __shfl_sync(0xffffffffu, incl, 31);
                const uint32_t e0 = incl - cand;
                for (uint32_t win = 0; win < warp_total; win += kStage) {  // warp-uniform rounds
                    if (cand && e0 < win + kStage && e0 + cand > win) {
                        uint32_t e = e0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint32_t c = info[u] >> 16;
                            if (!c) continue;
                            const uint32_t loc = static_cast<uint32_t>(u * kJoinThreads + threadIdx.x) << kIdxBits;
                            const uint32_t first = info[u] & 0xffffu;
                            if (c == 1) {
                                if (e >= win && e < win + kStage) stage[e - win] = loc | first;
                                ++e;
                                continue;
                            }
                            for (uint32_t i = first; i != kNil; i = link[i]) {
                                if (bfp[i] != fpv[u]) continue;
                                if (e >= win && e < win + kStage) stage[e - win] = loc | i;
                                ++e;
                            }
                        }
                    }
                    __syncwarp();
                    const uint32_t n = warp_total - win < kStage ? warp_total - win : kStage;
                    for (uint32_t q0 = 0; q0 < n; q0 += 32) {  // emit: verify, compact, reserve, store
                        const uint32_t q = q0 + lane;
                        int64_t key = 0, lv = 0, rv = 0;
                        bool ok_row = false;
                        if (q < n) {
                            const uint32_t ent = stage[q];
                            const longlong2 brow = L.rows[bpos[ent & ((1u << kIdxBits) - 1)]];
                            const longlong2 prow = R.rows[ppos[ent >> kIdxBits]];
                            ok_row = brow.x == prow.x;
                            key = brow.x;
                            lv = brow.y;
                            rv = prow.y;
                        }
                        const unsigned m = __ballot_sync(0xffffffffu, ok_row);
                        if (!m) continue;
                        unsigned long long at = 0;
                        if (lane == 0) at = atomicAdd(cursor, static_cast<unsigned long long>(__popc(m)));
                        at = __shfl_sync(0xffffffffu, at, 0);
                        if (ok_row) {
                            const unsigned long long pos = at + __popc(m & ((1u << lane) - 1u));
                            if (static_cast<int64_t>(pos) < capacity) {
                                ok[pos] = key;
                                ol[pos] = lv;
                                orr[pos] = rv;
                            }
                            ++cnt;
                            hsum += row_hash(key, lv, rv);
                            ksum += static_cast<unsigned long long>(key);
                        }
                    }
                    __syncwarp();
                }
                __syncthreads();  // ppos is rewritten by the next sub-round
            }
        }
        __syncthreads();  // the table is rebuilt for the next chunk
    }
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
        cnt = red[lane][0];
        hsum = red[lane][1];
        ksum = red[lane][2];
        for (int o = 16; o; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
            ksum += __shfl_xor_sync(0xffffffffu, ksum, o);
        }
        if (lane == 0 && cnt) {
            atomicAdd(result + 1, cnt);
            atomicAdd(result + 2, hsum);
            atomicAdd(result + 3, ksum);
        }
    }
}

int log2_exact(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return (1 << l) == v ? l : -1;
}

m4d_status make_segs(const int64_t* seg_off, const int64_t* seg_rows, int nseg, Segs* sg, int64_t* tiles) {
    if (nseg < 1 || nseg > kMaxSegs) return m4d::fail(M4D_ERR_USAGE, "segment count %d outside [1, %d]", nseg, kMaxSegs);
    if (!seg_off || !seg_rows) return m4d::fail(M4D_ERR_USAGE, "null segment arrays");
    std::memset(sg, 0, sizeof(*sg));
    sg->n = nseg;
    int64_t t = 0;
    for (int s = 0; s < nseg; ++s) {
        if (seg_rows[s] < 0 || seg_off[s] < 0 || seg_off[s] + seg_rows[s] > (int64_t(1) << 32))
            return m4d::fail(M4D_ERR_USAGE, "segment %d outside [0, 2^32) rows", s);
        sg->off[s] = seg_off[s];
        sg->rows[s] = seg_rows[s];
        sg->tile0[s] = t;
        t += (seg_rows[s] + kTileRows - 1) / kTileRows;
    }
    sg->tile0[nseg] = t;
    *tiles = t;
    return M4D_OK;
}

}  // namespace

extern "C" {

int m4d_tile_rows(void) { return kTileRows; }

int64_t m4d_tile_count(const int64_t* seg_rows, int nseg) {
    int64_t t = 0;
    for (int s = 0; s < nseg; ++s) t += (seg_rows[s] + kTileRows - 1) / kTileRows;
    return t;
}

size_t m4d_tile_meta_bytes(int64_t tiles, int parts) {
    return static_cast<size_t>((parts + 15) / 16 * 16) * static_cast<size_t>(tiles) * sizeof(uint16_t) + 256;
}

m4d_status m4d_tile_partition(const int64_t* keys, const int64_t* vals, const int64_t* seg_off, const int64_t* seg_rows,
                              int nseg, int parts, int64_t* out_pairs, uint16_t* meta, void* scratch,
                              size_t scratch_bytes, void* stream) {
    const int log2p = log2_exact(parts);
    if (log2p < 0 || parts > kMaxTileParts) return m4d::fail(M4D_ERR_USAGE, "partition count %d not a power of two <= %d", parts, kMaxTileParts);
    Segs sg;
    int64_t tiles = 0;
    m4d_status st = make_segs(seg_off, seg_rows, nseg, &sg, &tiles);
    if (st != M4D_OK) return st;
    if (scratch_bytes < m4d_tile_meta_bytes(tiles, parts)) return m4d::fail(M4D_ERR_USAGE, "tile scratch too small");
    if (!tiles) return M4D_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint16_t* staged = static_cast<uint16_t*>(scratch);
    const size_t smem = 4 * kTileRows * sizeof(int64_t) +
                        static_cast<size_t>(parts > kSortThreads ? parts : kSortThreads) * sizeof(uint32_t) +
                        kTileRows * sizeof(uint16_t);
    int dev = 0, sms = 148;
    M4D_CUDA_TRY(cudaGetDevice(&dev));
    M4D_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const unsigned grid = static_cast<unsigned>(tiles < sms ? tiles : sms);
    if (vals) {
        M4D_CUDA_TRY(cudaFuncSetAttribute(tile_sort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        tile_sort_kernel<false><<<grid, kSortThreads, smem, s>>>(keys, vals, sg, tiles, log2p,
                                                                 reinterpret_cast<longlong2*>(out_pairs), staged);
    } else {
        M4D_CUDA_TRY(cudaFuncSetAttribute(tile_sort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        tile_sort_kernel<true><<<grid, kSortThreads, smem, s>>>(keys, nullptr, sg, tiles, log2p,
                                                                reinterpret_cast<longlong2*>(out_pairs), staged);
    }
    dim3 tg(static_cast<unsigned>((tiles + kTrTiles - 1) / kTrTiles), static_cast<unsigned>((parts + 15) / 16));
    meta_transpose_kernel<<<tg, 512, 0, s>>>(staged, tiles, parts, meta);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

m4d_status m4d_tile_join(const int64_t* lpairs, const uint16_t* lmeta, const int64_t* lseg_off, const int64_t* lseg_rows,
                         int lnseg, const int64_t* rpairs, const uint16_t* rmeta, const int64_t* rseg_off,
                         const int64_t* rseg_rows, int rnseg, int parts, int64_t* out_keys, int64_t* out_lvals,
                         int64_t* out_rvals, int64_t capacity, unsigned long long* result, void* stream) {
    if (log2_exact(parts) < 0 || parts > kMaxTileParts) return m4d::fail(M4D_ERR_USAGE, "partition count %d not a power of two <= %d", parts, kMaxTileParts);
    JoinSide l{}, r{};
    m4d_status st = make_segs(lseg_off, lseg_rows, lnseg, &l.sg, &l.tiles);
    if (st != M4D_OK) return st;
    st = make_segs(rseg_off, rseg_rows, rnseg, &r.sg, &r.tiles);
    if (st != M4D_OK) return st;
    l.rows = reinterpret_cast<const longlong2*>(lpairs);
    r.rows = reinterpret_cast<const longlong2*>(rpairs);
    l.meta = lmeta;
    r.meta = rmeta;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    M4D_CUDA_TRY(cudaMemsetAsync(result, 0, 4 * sizeof(unsigned long long), s));
    if (!l.tiles || !r.tiles) return M4D_OK;
    M4D_CUDA_TRY(cudaFuncSetAttribute(tile_join_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kJoinSmem)));
    tile_join_kernel<<<parts, kJoinThreads, kJoinSmem, s>>>(l, r, parts, out_keys, out_lvals, out_rvals, capacity, result);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

int m4d_tile_join_partition_rows(void) { return 2 * kChunk - 1000; }

}  // extern "C"
