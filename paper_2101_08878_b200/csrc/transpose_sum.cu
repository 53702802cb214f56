// K3/K4: fused transpose-add-reduce for sum(x + x.T) over a chunked fp64
// array, plus the deterministic input
// generator of BASELINE.md §3.
//
// Work decomposition.  Every output block y(i,j) = x(i,j) + x(j,i)^T is cut
// into 64x64 fp64 tiles; one *item* is one tile position:
//   * paired item  : y(i,j) tile (tr,tc) AND y(j,i) tile (tc,tr).  Both x tiles
//                    are staged once in shared memory, so x is read exactly
//                    once for both outputs (16 B of HBM per output element).
//   * single item  : y(i,j) tile only; the x(j,i) tile may live on a peer B200
//                    and is read straight over NVLink through its IPC mapping.
//   * diagonal     : y(i,i) tiles (tr,tc) and (tc,tr) of the same block.
//
// Main kernel (ts_kernel_tma): persistent, one CTA per SM, warp-specialised.
// A producer warp takes items blockIdx.x, blockIdx.x + grid, ... and streams both x tiles
// into a 3-stage shared-memory ring with tiled TMA loads (2-D tensor maps over
// each block pool, 128-byte swizzle, 4 boxes of 64x16 fp64 per tile, mbarrier
// complete_tx); 8 consumer warps transpose-add, store y with coalesced 256 B
// row segments and reduce per warp; an epilogue warp folds the warp partials
// into per-tile sums off the critical path.  Items come from a global cursor
// (dynamic) so the in-flight window stays compact in the array, which keeps
// DRAM pages hot (round-robin static assignment measured 5.15 vs 3.93 ms).  Two tile
// pairs are in flight while a third is consumed.  The swizzle keeps the transposed shared-memory read at <= 2-way
// bank conflicts without padding.
//
// Fallback (ts_kernel_ldg): one CTA per item, LDG-staged, padded shared
// tiles; used when the block edge is odd or the pointers cannot be described
// by tensor maps.
//
// Reduction.  Each tile's sum is accumulated in a fixed thread/element order
// that does not depend on whether the tile was computed paired or single, so
// per-block sums are bit-identical for any worker count and either kernel.
// The CTA that completes a block folds its tile sums in fixed order
// (threadfence-reduction pattern), and the one completing the last block folds
// the block sums.  On the TMA path that bookkeeping is a second, tiny launch
// (ts_fold_kernel, one CTA per block): measured 3.93 ms vs 4.86 ms with the
// per-item completion atomics inline (40000^2 / 2000, one B200).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "m4d_internal.h"
#include "ptx.cuh"

namespace {

constexpr int kTile = 64;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerWarp = kTile / kWarps;  // 8

// LDG path: padded pitch 65 -> conflict-free 64-bit column reads.
constexpr int kPitchLdg = kTile + 1;
constexpr size_t kSmemLdg = 2ull * kTile * kPitchLdg * sizeof(double);

// TMA path: a tile is 4 swizzled boxes of 64 rows x 16 fp64 (128 B rows).
constexpr int kBoxCols = 16;
constexpr int kBoxes = kTile / kBoxCols;
constexpr uint32_t kBoxBytes = kTile * kBoxCols * sizeof(double);  // 8 KB
constexpr uint32_t kTileBytes = kBoxes * kBoxBytes;                // 32 KB
constexpr int kStages = 3;
constexpr int kTmaThreads = kThreads + 64;  // 8 consumer warps + producer warp + epilogue warp
constexpr int kSmemOffsets = 1024;  // item offsets kept in shared memory up to this many tasks + 1
constexpr size_t kSmemTma = kStages * 2ull * kTileBytes + kSmemOffsets * sizeof(int64_t) + 1024;  // + alignment slack
constexpr int kMaxMaps = 16;
constexpr int kMaxStreams = 16;  // item streams of the dynamic scheduler: <= 15 peer groups + local

struct TsMaps {
    CUtensorMap m[kMaxMaps];
};

struct TsParams {
    const m4d_ts_task* tasks;
    const int4* refs;         // per task: (map of a, slot of a, map of bt, slot of bt)
    const int64_t* item_off;  // ntasks + 1 prefix offsets of tile items
    int ntasks;
    int T;                    // tiles per block edge
    int64_t b;                // block edge (elements)
    int64_t items;            // total tile items
    int64_t items_remote;     // items [0, items_remote) read a peer tile (tasks sorted remote-first)
    int64_t stream_off[kMaxStreams + 1];  // item range of each stream: peer groups, then local
    int nstreams;             // peer streams + 1 (local is the last one)
    int remote_ctas;          // CTAs that start on a peer stream (dynamic TMA path)
    int remote_cap;           // CTAs [remote_cap, grid) never take remote items
    int nslots;
    double* tile_sums;        // [nslots][T*T]
    unsigned* block_done;     // [nslots]
    unsigned* all_done;       // [1]
    unsigned long long* work; // [2] dynamic item cursors: remote stream, local stream (TMA path)
    unsigned* exits;          // [1] CTAs done (TMA path)
    double* block_sums;       // [nslots]
    double* total;            // [1] or null
    int dynamic;              // TMA path: 1 = items from the global cursor, 0 = blockIdx.x + k * grid
    int fold_inline;          // TMA path: 1 = block completion via atomics in-kernel, 0 = ts_fold_kernel
};

struct Item {
    int task;
    int tr, tc;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Fixed-order reduction of n values by one warp (lane-strided partials, then
// a butterfly); identical result whichever CTA runs it.
__device__ __forceinline__ double warp_fold(const double* v, int n, int lane) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += __ldcg(v + i);
    return warp_sum(s);
}

__device__ __forceinline__ Item decode_item(const TsParams& p, int64_t item) {
    int lo = 0, hi = p.ntasks - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (p.item_off[mid] <= item) lo = mid; else hi = mid - 1;
    }
    Item it;
    it.task = lo;
    int64_t local = item - p.item_off[lo];
    const int T = p.T;
    if (p.tasks[lo].diag) {  // upper triangle of the tile grid, row by row
        int tr = 0;
        while (local >= T - tr) { local -= T - tr; ++tr; }
        it.tr = tr;
        it.tc = tr + static_cast<int>(local);
    } else {
        it.tr = static_cast<int>(local / T);
        it.tc = static_cast<int>(local % T);
    }
    return it;
}

// Shared-tile addressing.  Padded: row-major with pitch 65.  Swizzled: the
// TMA 128-byte swizzle of 4 boxes (16-byte chunk index XOR row % 8).
struct PaddedTile {
    const double* base;
    __device__ __forceinline__ double operator()(int r, int c) const { return base[r * kPitchLdg + c]; }
};

struct SwizzledTile {
    const unsigned char* base;
    __device__ __forceinline__ double operator()(int r, int c) const {
        const int box = c >> 4, cc = c & 15;
        const uint32_t off = box * kBoxBytes + r * 128 + ((((cc >> 1) ^ (r & 7))) << 4) + ((cc & 1) << 3);
        return *reinterpret_cast<const double*>(base + off);
    }
};

// y(i,j)[R0+r][C0+c] = A(r,c) + B(c,r);  y(j,i)[C0+r][R0+c] = B(r,c) + A(c,r),
// where A is the x(i,j) tile and B the x(j,i) tile (rows C0.., cols R0..).
// Thread (warp w, lane l) owns rows w*8..w*8+7, columns l and l+32 of both
// output tiles and accumulates them in that fixed order (the determinism
// contract: identical per-tile sums for paired and single computation).
template <typename Tile>
__device__ __forceinline__ void transpose_add_tile(const Tile& A, const Tile& B, double* y, double* y2,
                                                   bool second, int64_t b, int64_t R0, int64_t C0, int warp,
                                                   int lane, double& s1, double& s2) {
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            if (R0 + r < b && C0 + c < b) {
                const double v = A(r, c) + B(c, r);
                __stcs(y + (R0 + r) * b + (C0 + c), v);
                s1 += v;
            }
            if (second && C0 + r < b && R0 + c < b) {
                const double w = B(r, c) + A(c, r);
                __stcs(y2 + (C0 + r) * b + (R0 + c), w);
                s2 += w;
            }
        }
    }
}

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* addr, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v) : "memory");
    return old;
}

// Records one item's tile sums; the CTA that completes an output block folds
// its tile sums, and the one completing the last block folds the block sums.
// Ordering uses acquire-release atomics on the completion counters (the
// tile-sum stores happen-before the increment that observes completion), so
// no sequentially-consistent fence sits on the path.  Called by all 32 lanes
// of one warp after t1/t2 are final.
__device__ __forceinline__ void finish_item(const TsParams& p, int slot_y, int tr, int tc, bool second,
                                            int slot2, double t1, double t2, int lane) {
    const int T = p.T;
    const int tiles = T * T;
    int fin0 = -1, fin1 = -1;
    if (lane == 0) {
        p.tile_sums[static_cast<int64_t>(slot_y) * tiles + tr * T + tc] = t1;
        if (second) p.tile_sums[static_cast<int64_t>(slot2) * tiles + tc * T + tr] = t2;
        if (second && slot2 == slot_y) {
            if (atom_add_acq_rel(p.block_done + slot_y, 2u) + 2u == static_cast<unsigned>(tiles)) fin0 = slot_y;
        } else {
            if (atom_add_acq_rel(p.block_done + slot_y, 1u) + 1u == static_cast<unsigned>(tiles)) fin0 = slot_y;
            if (second && atom_add_acq_rel(p.block_done + slot2, 1u) + 1u == static_cast<unsigned>(tiles))
                fin1 = slot2;
        }
    }
    fin0 = __shfl_sync(0xffffffffu, fin0, 0);
    fin1 = __shfl_sync(0xffffffffu, fin1, 0);
    for (int f = 0; f < 2; ++f) {
        const int slot = f ? fin1 : fin0;
        if (slot < 0) continue;
        const double bs = warp_fold(p.tile_sums + static_cast<int64_t>(slot) * tiles, tiles, lane);
        int last = 0;
        if (lane == 0) {
            p.block_sums[slot] = bs;
            p.block_done[slot] = 0;  // re-arm for the next run (nobody touches it again this run)
            last = atom_add_acq_rel(p.all_done, 1u) + 1u == static_cast<unsigned>(p.nslots);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {  // this CTA completed the last block
            const double tot = warp_fold(p.block_sums, p.nslots, lane);
            if (lane == 0) {
                if (p.total) *p.total = tot;
                *p.all_done = 0;
            }
        }
    }
}

// Everything a consumer and the epilogue need about one staged item, filled
// by the producer so the consumer path touches no global metadata.
struct StageRec {
    double* y;
    double* y2;      // second output tile's block (y itself for a diagonal block)
    int tr, tc;
    int slot_y, slot2;
    int second;      // 1 when the item also produces the transposed tile
    int live;        // 0 = sentinel
};

__global__ void __launch_bounds__(kTmaThreads, 1)
    ts_kernel_tma(const TsParams p, const __grid_constant__ TsMaps maps) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[kStages];   // producer -> consumers (TMA bytes landed)
    __shared__ __align__(8) uint64_t empty_bar[kStages];  // consumers -> producer (tiles read)
    __shared__ __align__(8) uint64_t sum_full[kStages];   // consumers -> epilogue (partials written)
    __shared__ __align__(8) uint64_t sum_empty[kStages];  // epilogue -> consumers (partials read)
    __shared__ StageRec stage_rec[kStages];
    __shared__ StageRec sum_rec[kStages];
    __shared__ double part[kStages][2][kWarps];
    // 128-byte swizzled boxes need 1024-byte aligned destinations; the item
    // offset table follows the tile ring.
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                           ~static_cast<uintptr_t>(1023));
    const int64_t* item_off = p.item_off;
    if (p.ntasks + 1 <= kSmemOffsets) {
        int64_t* tab = reinterpret_cast<int64_t*>(smem + kStages * 2ull * kTileBytes);
        for (int i = threadIdx.x; i <= p.ntasks; i += blockDim.x) tab[i] = p.item_off[i];
        item_off = tab;
    }

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            m4d::ptx::mbar_init(&full_bar[s], 1);
            m4d::ptx::mbar_init(&empty_bar[s], kWarps);
            m4d::ptx::mbar_init(&sum_full[s], kWarps);
            m4d::ptx::mbar_init(&sum_empty[s], 1);
        }
        m4d::ptx::fence_mbar_init();
    }
    __syncthreads();

    const int64_t b = p.b;
    if (warp == kWarps) {
        // ---------------- producer warp: items blockIdx.x, +grid, ... ----------------
        if (lane == 0) {
            int task = 0;
            int k = 0;
            // Item streams share the grid: one per peer GPU whose tiles are read
            // over NVLink, then the local one.  The first remote_ctas CTAs start
            // spread over the peer streams (so every peer is read at once and no
            // peer's links become a hotspot), the rest on the local stream; a CTA
            // whose stream runs dry moves on to the next, so NVLink and HBM stay
            // busy together until the end.
            const int S = p.nstreams - 1;  // peer streams
            int st = (static_cast<int>(blockIdx.x) < p.remote_ctas && S > 0) ? static_cast<int>(blockIdx.x) % S : S;
            unsigned dry = 0;
            for (int q = 0; q < p.nstreams; ++q)
                if (p.stream_off[q] == p.stream_off[q + 1] || (q < S && static_cast<int>(blockIdx.x) >= p.remote_cap))
                    dry |= 1u << q;
            auto claim = [&]() -> int64_t {
                for (int tries = 0; tries < p.nstreams; ++tries, st = st + 1 == p.nstreams ? 0 : st + 1) {
                    if (dry >> st & 1u) continue;
                    const int64_t v = p.stream_off[st] + static_cast<int64_t>(atomicAdd(p.work + st, 1ull));
                    if (v < p.stream_off[st + 1]) return v;
                    dry |= 1u << st;
                }
                return p.items;
            };
            int64_t next = p.dynamic ? claim() : blockIdx.x;
            for (;; ++k) {
                const int64_t item = next;
                if (item < p.items)  // claim the following item early: its latency overlaps this one
                    next = p.dynamic ? claim() : item + gridDim.x;
                const int s = k % kStages;
                const uint32_t ph = (k / kStages) & 1;
                m4d::ptx::mbar_wait(&empty_bar[s], ph ^ 1);
                StageRec& rec = stage_rec[s];
                if (item >= p.items) {
                    rec.live = 0;  // sentinel: no more items
                    __threadfence_block();
                    m4d::ptx::mbar_arrive(&full_bar[s]);
                    break;
                }
                if (item < item_off[task]) task = 0;  // moved to an earlier stream
                while (item_off[task + 1] <= item) ++task;  // items ascend within a stream: walk forward
                const m4d_ts_task t = p.tasks[task];
                const int4 ref = p.refs[task];
                int64_t local = item - item_off[task];
                int tr, tc;
                const int T = p.T;
                if (t.diag) {
                    tr = 0;
                    while (local >= T - tr) { local -= T - tr; ++tr; }
                    tc = tr + static_cast<int>(local);
                } else {
                    tr = static_cast<int>(local / T);
                    tc = static_cast<int>(local % T);
                }
                rec.y = t.y;
                rec.y2 = t.diag ? t.y : t.y2;
                rec.tr = tr;
                rec.tc = tc;
                rec.slot_y = t.slot_y;
                rec.slot2 = t.diag ? t.slot_y : t.slot_y2;
                rec.second = t.diag ? (tr != tc) : (t.y2 != nullptr);
                rec.live = 1;
                __threadfence_block();  // publish the record before the phase can complete
                unsigned char* sA = smem + static_cast<size_t>(s) * 2 * kTileBytes;
                unsigned char* sB = sA + kTileBytes;
                m4d::ptx::mbar_arrive_expect_tx(&full_bar[s], 2 * kTileBytes);
                const void* ma = &maps.m[ref.x];
                const void* mb = &maps.m[ref.z];
                const int R0 = tr * kTile, C0 = tc * kTile;
                const int rowa = ref.y * static_cast<int>(b) + R0;  // x(i,j): rows R0.., cols C0..
                const int rowb = ref.w * static_cast<int>(b) + C0;  // x(j,i): rows C0.., cols R0..
#pragma unroll
                for (int q = 0; q < kBoxes; ++q) {
                    m4d::ptx::tma_load_2d(sA + q * kBoxBytes, ma, C0 + q * kBoxCols, rowa, &full_bar[s]);
                    m4d::ptx::tma_load_2d(sB + q * kBoxBytes, mb, R0 + q * kBoxCols, rowb, &full_bar[s]);
                }
            }
        }
        __syncwarp();
    } else if (warp == kWarps + 1) {
        // ---------------- epilogue warp: tile sums, block completion ----------------
        for (int k = 0;; ++k) {
            const int s = k % kStages;
            const uint32_t ph = (k / kStages) & 1;
            m4d::ptx::mbar_wait(&sum_full[s], ph);
            const StageRec rec = sum_rec[s];
            double t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) { t1 += part[s][0][w]; t2 += part[s][1][w]; }
            __syncwarp();
            if (lane == 0) m4d::ptx::mbar_arrive(&sum_empty[s]);
            if (!rec.live) break;
            if (p.fold_inline) {
                finish_item(p, rec.slot_y, rec.tr, rec.tc, rec.second != 0, rec.slot2, t1, t2, lane);
            } else if (lane == 0) {
                const int T = p.T;
                p.tile_sums[static_cast<int64_t>(rec.slot_y) * T * T + rec.tr * T + rec.tc] = t1;
                if (rec.second) p.tile_sums[static_cast<int64_t>(rec.slot2) * T * T + rec.tc * T + rec.tr] = t2;
            }
        }
    } else {
        // ---------------- consumer warps: transpose-add-store ----------------
        for (int k = 0;; ++k) {
            const int s = k % kStages;
            const uint32_t ph = (k / kStages) & 1;
            m4d::ptx::mbar_wait(&full_bar[s], ph);
            const StageRec rec = stage_rec[s];
            double s1 = 0.0, s2 = 0.0;
            if (rec.live) {
                const SwizzledTile A{smem + static_cast<size_t>(s) * 2 * kTileBytes};
                const SwizzledTile B{A.base + kTileBytes};
                transpose_add_tile(A, B, rec.y, rec.y2, rec.second != 0, b, static_cast<int64_t>(rec.tr) * kTile,
                                   static_cast<int64_t>(rec.tc) * kTile, warp, lane, s1, s2);
            }
            __syncwarp();
            if (lane == 0) m4d::ptx::mbar_arrive(&empty_bar[s]);  // tiles of this stage consumed
            s1 = warp_sum(s1);
            s2 = warp_sum(s2);
            m4d::ptx::mbar_wait(&sum_empty[s], ph ^ 1);  // epilogue has read this slot's partials
            if (lane == 0) {
                part[s][0][warp] = s1;
                part[s][1][warp] = s2;
                if (warp == 0) sum_rec[s] = rec;
                __threadfence_block();
                m4d::ptx::mbar_arrive(&sum_full[s]);
            }
            if (!rec.live) break;
        }
    }
    __syncthreads();
    if (p.dynamic && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.exits, 1u) + 1u == gridDim.x) {  // last CTA out re-arms the cursor
            for (int q = 0; q < p.nstreams; ++q) p.work[q] = 0;
            *p.exits = 0;
        }
    }
}

// Second launch of a step when the fold is not inline: CTA s folds block s's
// tile sums (fixed order), the last CTA folds the block sums.
__global__ void __launch_bounds__(256) ts_fold_kernel(const TsParams p) {
    const int slot = blockIdx.x;
    const int tiles = p.T * p.T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int last;
    if (warp == 0) {
        const double bs = warp_fold(p.tile_sums + static_cast<int64_t>(slot) * tiles, tiles, lane);
        if (lane == 0) {
            p.block_sums[slot] = bs;
            last = atom_add_acq_rel(p.all_done, 1u) + 1u == static_cast<unsigned>(p.nslots);
        }
        __syncwarp();
        if (last) {
            const double tot = warp_fold(p.block_sums, p.nslots, lane);
            if (lane == 0) {
                if (p.total) *p.total = tot;
                *p.all_done = 0;
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads, 3) ts_kernel_ldg(const TsParams p) {
    extern __shared__ double smem_ldg[];
    double* sA = smem_ldg;
    double* sB = smem_ldg + kTile * kPitchLdg;
    __shared__ double part[2][kWarps];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Item it = decode_item(p, blockIdx.x);
    const m4d_ts_task task = p.tasks[it.task];
    const int tr = it.tr, tc = it.tc;
    const bool second = task.diag ? (tr != tc) : (task.y2 != nullptr);
    double* const y2 = task.diag ? task.y : task.y2;
    const int slot2 = task.diag ? task.slot_y : task.slot_y2;
    const int64_t b = p.b;
    const int64_t R0 = static_cast<int64_t>(tr) * kTile;
    const int64_t C0 = static_cast<int64_t>(tc) * kTile;

#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            double av = 0.0, bv = 0.0;
            if (R0 + r < b && C0 + c < b) av = __ldcs(task.a + (R0 + r) * b + (C0 + c));
            if (C0 + r < b && R0 + c < b) bv = __ldcs(task.bt + (C0 + r) * b + (R0 + c));
            sA[r * kPitchLdg + c] = av;
            sB[r * kPitchLdg + c] = bv;
        }
    }
    __syncthreads();
    double s1 = 0.0, s2 = 0.0;
    transpose_add_tile(PaddedTile{sA}, PaddedTile{sB}, task.y, y2, second, b, R0, C0, warp, lane, s1, s2);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
        part[0][warp] = s1;
        part[1][warp] = s2;
    }
    __syncthreads();
    if (warp == 0) {
        double t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) { t1 += part[0][w]; t2 += part[1][w]; }
        finish_item(p, task.slot_y, tr, tc, second, slot2, t1, t2, lane);
    }
}

__global__ void fill_block_kernel(double* dst, int64_t n, int64_t row0, int64_t col0, int64_t b,
                                  uint64_t seed) {
    const int64_t count = b * b;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / b, c = idx - (idx / b) * b;
        const uint64_t g = static_cast<uint64_t>(row0 + r) * static_cast<uint64_t>(n) +
                           static_cast<uint64_t>(col0 + c);
        dst[idx] = static_cast<double>(m4d_splitmix64(seed ^ g) >> 11) * 0x1.0p-53;
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_tiled_fn() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    });
    return fn;
}

// L2 promotion of peer-pool tensor maps (M4D_TS_REMOTE_PROMO = none|64|128|256).
CUtensorMapL2promotion remote_promotion() {
    const char* v = getenv("M4D_TS_REMOTE_PROMO");
    if (!v) return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (!strcmp(v, "none")) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    if (!strcmp(v, "64")) return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (!strcmp(v, "128")) return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// Groups the x-block pointers of the tasks into pools (a base plus whole
// blocks) and encodes one 2-D tensor map per pool: rows = slot * b + row,
// cols = col, 128-byte swizzled 64x16 boxes.  Returns false when the tasks
// cannot be expressed that way (the LDG kernel is used instead).
bool build_maps(const m4d_ts_task* tasks, int ntasks, int64_t b, TsMaps* maps, std::vector<int4>* refs) {
    if (b % 2 || b > 0x7fffffff / 2) return false;
    PFN_encodeTiled encode = encode_tiled_fn();
    if (!encode) return false;
    const uint64_t block_bytes = static_cast<uint64_t>(b) * b * sizeof(double);
    std::vector<uintptr_t> ptrs;
    std::map<uintptr_t, bool> remote;  // pointer -> read over NVLink
    for (int t = 0; t < ntasks; ++t) {
        ptrs.push_back(reinterpret_cast<uintptr_t>(tasks[t].a));
        ptrs.push_back(reinterpret_cast<uintptr_t>(tasks[t].bt));
        remote[reinterpret_cast<uintptr_t>(tasks[t].a)] |= false;
        remote[reinterpret_cast<uintptr_t>(tasks[t].bt)] |= tasks[t].remote != 0;
    }
    std::sort(ptrs.begin(), ptrs.end());
    ptrs.erase(std::unique(ptrs.begin(), ptrs.end()), ptrs.end());
    std::vector<uintptr_t> bases;
    std::vector<uint64_t> slots;  // max slot + 1 per base
    std::vector<bool> pool_remote;
    std::map<uintptr_t, std::pair<int, int>> where;
    for (uintptr_t p : ptrs) {
        if (p & 15) return false;
        int found = -1;
        for (size_t k = 0; k < bases.size(); ++k)
            if ((p - bases[k]) % block_bytes == 0 && pool_remote[k] == remote[p]) { found = static_cast<int>(k); break; }
        if (found < 0) {
            if (bases.size() == kMaxMaps) return false;
            bases.push_back(p);
            slots.push_back(0);
            pool_remote.push_back(remote[p]);
            found = static_cast<int>(bases.size()) - 1;
        }
        const uint64_t slot = (p - bases[found]) / block_bytes;
        if ((slot + 1) * b > 0x7fffffffull) return false;
        slots[found] = std::max<uint64_t>(slots[found], slot + 1);
        where[p] = {found, static_cast<int>(slot)};
    }
    for (size_t k = 0; k < bases.size(); ++k) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(b), static_cast<cuuint64_t>(slots[k] * b)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(b) * sizeof(double)};
        cuuint32_t box[2] = {kBoxCols, kTile};
        cuuint32_t estr[2] = {1, 1};
        if (encode(&maps->m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, reinterpret_cast<void*>(bases[k]), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   pool_remote[k] ? remote_promotion() : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    refs->resize(ntasks);
    for (int t = 0; t < ntasks; ++t) {
        auto a = where[reinterpret_cast<uintptr_t>(tasks[t].a)];
        auto bt = where[reinterpret_cast<uintptr_t>(tasks[t].bt)];
        (*refs)[t] = make_int4(a.first, a.second, bt.first, bt.second);
    }
    return true;
}

}  // namespace

struct m4d_ts_plan {
    int device = 0;
    int64_t b = 0;
    int T = 0;
    int ntasks = 0;
    int nslots = 0;
    int64_t items = 0;
    int64_t items_remote = 0;
    std::vector<int64_t> stream_off;  // nstreams + 1
    int remote_ctas = 0;
    int remote_cap = 1 << 30;
    m4d_ts_task* d_tasks = nullptr;
    int4* d_refs = nullptr;
    int64_t* d_off = nullptr;
    double* d_tile_sums = nullptr;
    unsigned* d_counters = nullptr;  // nslots block counters, all_done, exits
    unsigned long long* d_work = nullptr;
    bool tma = false;                // TMA-fed persistent kernel usable
    int sms = 148;
    int dynamic = 1;                 // M4D_TS_SCHED=static: round-robin items (ablation)
    int fold_inline = 0;             // M4D_TS_FOLD=inline: in-kernel block completion (ablation)
    TsMaps maps;
};

using m4d::fail;

extern "C" {

m4d_status m4d_fill_block_f64(double* dst, int64_t n, int64_t row0, int64_t col0, int64_t b,
                              uint64_t seed, void* stream) {
    if (b <= 0 || n <= 0 || row0 < 0 || col0 < 0 || row0 + b > n || col0 + b > n)
        return fail(M4D_ERR_USAGE, "block (%lld,%lld)+%lld outside %lld^2 array", (long long)row0,
                    (long long)col0, (long long)b, (long long)n);
    const int64_t count = b * b;
    int64_t grid = std::min<int64_t>((count + 255) / 256, 148 * 16);
    fill_block_kernel<<<static_cast<unsigned>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        dst, n, row0, col0, b, seed);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}


m4d_status m4d_ts_plan_create(int device, const m4d_ts_task* tasks_in, int ntasks, int64_t block,
                              int nslots, m4d_ts_plan** plan_out) {
    *plan_out = nullptr;
    if (ntasks > 0 && !tasks_in) return fail(M4D_ERR_USAGE, "null task array");
    // Tasks grouped into item streams: one per distinct non-zero `remote` id
    // (the peer the partner tile is read from), ascending, then the local tasks.
    std::vector<int> groups;
    for (int t = 0; t < ntasks; ++t)
        if (tasks_in[t].remote && std::find(groups.begin(), groups.end(), tasks_in[t].remote) == groups.end())
            groups.push_back(tasks_in[t].remote);
    std::sort(groups.begin(), groups.end());
    if (static_cast<int>(groups.size()) >= kMaxStreams) return fail(M4D_ERR_USAGE, "more than %d peer groups", kMaxStreams - 1);
    std::vector<m4d_ts_task> sorted;
    std::vector<int> stream_tasks(groups.size() + 2, 0);  // task prefix per stream
    sorted.reserve(ntasks > 0 ? ntasks : 0);
    for (size_t g = 0; g <= groups.size(); ++g) {
        for (int t = 0; t < ntasks; ++t)
            if (g < groups.size() ? tasks_in[t].remote == groups[g] : tasks_in[t].remote == 0)
                sorted.push_back(tasks_in[t]);
        stream_tasks[g + 1] = static_cast<int>(sorted.size());
    }
    const m4d_ts_task* tasks = sorted.data();
    const int nremote = stream_tasks[groups.size()];
    if (block <= 0) return fail(M4D_ERR_USAGE, "block edge must be positive");
    if (ntasks < 0 || nslots < 0) return fail(M4D_ERR_USAGE, "negative task or slot count");
    const int64_t T64 = (block + kTile - 1) / kTile;
    if (T64 > 46340) return fail(M4D_ERR_USAGE, "block edge %lld too large", (long long)block);
    const int T = static_cast<int>(T64);
    const int64_t tiles = T64 * T64;

    // Every output block must be covered by exactly T*T tiles.
    std::vector<int64_t> cover(static_cast<size_t>(nslots), 0);
    std::vector<int64_t> off(static_cast<size_t>(ntasks) + 1, 0);
    for (int t = 0; t < ntasks; ++t) {
        const m4d_ts_task& k = tasks[t];
        if (!k.a || !k.bt || !k.y) return fail(M4D_ERR_USAGE, "task %d has a null pointer", t);
        if (k.slot_y < 0 || k.slot_y >= nslots)
            return fail(M4D_ERR_USAGE, "task %d slot_y %d outside [0,%d)", t, k.slot_y, nslots);
        int64_t n_items;
        if (k.diag) {
            if (k.a != k.bt || k.y2)
                return fail(M4D_ERR_USAGE, "diagonal task %d needs a == bt and y2 == NULL", t);
            n_items = T64 * (T64 + 1) / 2;
            cover[k.slot_y] += tiles;
        } else {
            n_items = tiles;
            cover[k.slot_y] += tiles;
            if (k.y2) {
                if (k.slot_y2 < 0 || k.slot_y2 >= nslots || k.slot_y2 == k.slot_y)
                    return fail(M4D_ERR_USAGE, "task %d slot_y2 %d invalid", t, k.slot_y2);
                cover[k.slot_y2] += tiles;
            }
        }
        off[t + 1] = off[t] + n_items;
    }
    for (int s = 0; s < nslots; ++s)
        if (cover[s] != tiles)
            return fail(M4D_ERR_USAGE, "output slot %d covered by %lld tiles, expected %lld", s,
                        (long long)cover[s], (long long)tiles);
    if (off[ntasks] > 0x7fffffffll) return fail(M4D_ERR_USAGE, "too many tile items");

    auto* plan = new m4d_ts_plan();
    plan->device = device;
    plan->b = block;
    plan->T = T;
    plan->ntasks = ntasks;
    plan->nslots = nslots;
    plan->items = off[ntasks];
    plan->items_remote = off[nremote];
    for (size_t g = 0; g < stream_tasks.size(); ++g) plan->stream_off.push_back(off[stream_tasks[g]]);
    auto cleanup = [&](int code) {
        m4d_ts_plan_destroy(plan);
        return code;
    };
    cudaError_t e;
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cleanup(m4d::cuda_fail(e, "cudaSetDevice"));
    std::vector<int4> refs;
    // M4D_TS_FORCE_LDG=1 selects the fallback kernel (tests cover both).
    plan->tma = !getenv("M4D_TS_FORCE_LDG") && ntasks > 0 && build_maps(tasks, ntasks, block, &plan->maps, &refs);
    if (const char* v = getenv("M4D_TS_SCHED")) plan->dynamic = strcmp(v, "static") != 0;
    if (const char* v = getenv("M4D_TS_FOLD")) plan->fold_inline = strcmp(v, "inline") == 0;
    if (ntasks) {
        if ((e = cudaMalloc(&plan->d_tasks, sizeof(m4d_ts_task) * ntasks)) != cudaSuccess ||
            (e = cudaMemcpy(plan->d_tasks, tasks, sizeof(m4d_ts_task) * ntasks, cudaMemcpyHostToDevice)) !=
                cudaSuccess)
            return cleanup(m4d::cuda_fail(e, "plan tasks"));
        if (plan->tma &&
            ((e = cudaMalloc(&plan->d_refs, sizeof(int4) * ntasks)) != cudaSuccess ||
             (e = cudaMemcpy(plan->d_refs, refs.data(), sizeof(int4) * ntasks, cudaMemcpyHostToDevice)) !=
                 cudaSuccess))
            return cleanup(m4d::cuda_fail(e, "plan tensor refs"));
    }
    if ((e = cudaMalloc(&plan->d_off, sizeof(int64_t) * (ntasks + 1))) != cudaSuccess ||
        (e = cudaMemcpy(plan->d_off, off.data(), sizeof(int64_t) * (ntasks + 1), cudaMemcpyHostToDevice)) !=
            cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "plan offsets"));
    if ((e = cudaMalloc(&plan->d_tile_sums, sizeof(double) * std::max<int64_t>(1, tiles * nslots))) !=
            cudaSuccess ||
        (e = cudaMalloc(&plan->d_counters, sizeof(unsigned) * (nslots + 2))) != cudaSuccess ||
        (e = cudaMemset(plan->d_counters, 0, sizeof(unsigned) * (nslots + 2))) != cudaSuccess ||
        (e = cudaMalloc(&plan->d_work, kMaxStreams * sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMemset(plan->d_work, 0, kMaxStreams * sizeof(unsigned long long))) != cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "plan scratch"));
    if ((e = cudaFuncSetAttribute(ts_kernel_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemLdg))) != cudaSuccess ||
        (e = cudaFuncSetAttribute(ts_kernel_ldg, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) !=
            cudaSuccess ||
        (e = cudaFuncSetAttribute(ts_kernel_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemTma))) != cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "ts kernel attributes"));
    if ((e = cudaDeviceGetAttribute(&plan->sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "SM count"));
    // CTAs that start on the peer streams: their share of the items, leaned
    // 15% toward NVLink (N=4: 111 -> 130 CTAs, 4.21 -> 4.08 ms per launch;
    // flat at N=2; tools/ts_remote_sweep.sh).  M4D_TS_REMOTE_CTAS overrides.
    plan->remote_ctas = plan->items ? static_cast<int>(std::min<int64_t>(
                                          plan->sms, (plan->sms * plan->items_remote * 115 / 100 + plan->items - 1) / plan->items))
                                    : 0;
    if (const char* v = getenv("M4D_TS_REMOTE_CTAS")) plan->remote_ctas = atoi(v);
    if (const char* v = getenv("M4D_TS_REMOTE_CAP")) plan->remote_cap = atoi(v);
    *plan_out = plan;
    return M4D_OK;
}

m4d_status m4d_ts_run(m4d_ts_plan* plan, double* block_sums, double* total, void* stream) {
    if (!plan) return fail(M4D_ERR_USAGE, "null plan");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (plan->items == 0) {
        if (total) M4D_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(double), s));
        return M4D_OK;
    }
    if (!block_sums) return fail(M4D_ERR_USAGE, "block_sums must not be NULL");
    M4D_CUDA_TRY(cudaSetDevice(plan->device));  // the stream belongs to the plan's device
    TsParams p;
    p.tasks = plan->d_tasks;
    p.refs = plan->d_refs;
    p.item_off = plan->d_off;
    p.ntasks = plan->ntasks;
    p.T = plan->T;
    p.b = plan->b;
    p.nslots = plan->nslots;
    p.items = plan->items;
    p.items_remote = plan->items_remote;
    p.remote_ctas = plan->remote_ctas;
    p.remote_cap = plan->remote_cap;
    p.nstreams = static_cast<int>(plan->stream_off.size()) - 1;
    for (int q = 0; q <= p.nstreams; ++q) p.stream_off[q] = plan->stream_off[q];
    p.tile_sums = plan->d_tile_sums;
    p.block_done = plan->d_counters;
    p.all_done = plan->d_counters + plan->nslots;
    p.exits = plan->d_counters + plan->nslots + 1;
    p.work = plan->d_work;
    p.block_sums = block_sums;
    p.total = total;
    p.dynamic = plan->dynamic;
    p.fold_inline = plan->fold_inline;
    if (plan->tma) {
        const int64_t grid = std::min<int64_t>(plan->sms, plan->items);
        ts_kernel_tma<<<static_cast<unsigned>(grid), kTmaThreads, kSmemTma, s>>>(p, plan->maps);
        if (!plan->fold_inline) ts_fold_kernel<<<plan->nslots, 256, 0, s>>>(p);
    } else {
        ts_kernel_ldg<<<static_cast<unsigned>(plan->items), kThreads, kSmemLdg, s>>>(p);
    }
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

int m4d_ts_launches_per_run(const m4d_ts_plan* plan) {
    if (!plan || plan->items == 0) return 0;
    return plan->tma && !plan->fold_inline ? 2 : 1;
}

int m4d_ts_plan_uses_tma(const m4d_ts_plan* plan) { return plan && plan->tma ? 1 : 0; }

m4d_status m4d_ts_plan_destroy(m4d_ts_plan* plan) {
    if (!plan) return M4D_OK;
    cudaFree(plan->d_tasks);
    cudaFree(plan->d_refs);
    cudaFree(plan->d_off);
    cudaFree(plan->d_tile_sums);
    cudaFree(plan->d_counters);
    cudaFree(plan->d_work);
    delete plan;
    return M4D_OK;
}

}  // extern "C"
