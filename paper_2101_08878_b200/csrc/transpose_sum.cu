// K3/K4: fused transpose-add-reduce for sum(x + x.T) over a chunked fp64
// array, plus the deterministic input
// generator of BASELINE.md §3.
//
// Work decomposition.  Every output block y(i,j) = x(i,j) + x(j,i)^T is cut
// into 64x64 fp64 tiles.  One CTA (256 threads) handles one tile item:
//   * paired item  : y(i,j) tile (tr,tc) AND y(j,i) tile (tc,tr).  Both x tiles
//                    are staged once in shared memory, so x is read exactly
//                    once for both outputs (16 B of HBM per output element).
//   * single item  : y(i,j) tile only; the x(j,i) tile may live on a peer B200
//                    and is read straight over NVLink through its IPC mapping.
//   * diagonal     : y(i,i) tiles (tr,tc) and (tc,tr) of the same block.
// Global access is one 256 B coalesced row segment per warp instruction
// (8 B per lane, streaming .cs hints); the transposed read comes out of a
// padded shared tile (pitch 65 doubles -> conflict-free 64-bit column reads).
//
// Reduction.  Each tile's sum is accumulated in a fixed thread/element order
// that does not depend on whether the tile was computed paired or single, so
// per-block sums are bit-identical for any worker count.  The last CTA to
// finish a block folds its tile sums in fixed order (threadfence-reduction
// pattern), and the last block folds the block sums, so one launch per step.
#include <cuda_runtime.h>

#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "m4d_internal.h"
#include "ptx.cuh"

namespace {

constexpr int kTile = 64;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerWarp = kTile / kWarps;  // 8

// v1 (LDG) path: padded pitch 65 -> conflict-free 64-bit column reads.
constexpr int kPitchLdg = kTile + 1;
constexpr size_t kSmemLdg = 2ull * kTile * kPitchLdg * sizeof(double);

// v2 (TMA bulk) path: rows must be 16-byte aligned -> pitch 66 (2-way conflicts
// on the transposed read, far below the smem bandwidth budget).
constexpr int kPitchTma = kTile + 2;
constexpr int kStages = 3;
constexpr int kTmaThreads = kThreads + 32;  // 8 consumer warps + 1 producer warp
constexpr size_t kTileBytesTma = static_cast<size_t>(kTile) * kPitchTma * sizeof(double);
constexpr size_t kSmemTma = kStages * 2 * kTileBytesTma;

struct TsParams {
    const m4d_ts_task* tasks;
    const int64_t* item_off;  // ntasks + 1 prefix offsets of tile items
    int ntasks;
    int T;                    // tiles per block edge
    int64_t b;                // block edge (elements)
    int64_t items;            // total tile items
    int nslots;
    double* tile_sums;        // [nslots][T*T]
    unsigned* block_done;     // [nslots]
    unsigned* all_done;       // [1]
    unsigned long long* work; // [1] dynamic item cursor (TMA path)
    unsigned* exits;          // [1] CTAs done (TMA path)
    double* block_sums;       // [nslots]
    double* total;            // [1] or null
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

// y(i,j)[R0+r][C0+c] = sA[r][c] + sB[c][r];  y(j,i)[C0+r][R0+c] = sB[r][c] + sA[c][r].
// Thread (warp w, lane l) owns rows w*8..w*8+7, columns l and l+32 of both
// output tiles and accumulates them in that fixed order (the determinism
// contract: identical per-tile sums for paired and single computation).
template <int PITCH>
__device__ __forceinline__ void transpose_add_tile(const double* sA, const double* sB, double* y, double* y2,
                                                   bool second, int64_t b, int64_t R0, int64_t C0, int warp,
                                                   int lane, double& s1, double& s2) {
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            if (R0 + r < b && C0 + c < b) {
                const double v = sA[r * PITCH + c] + sB[c * PITCH + r];
                __stcs(y + (R0 + r) * b + (C0 + c), v);
                s1 += v;
            }
            if (second && C0 + r < b && R0 + c < b) {
                const double w = sB[r * PITCH + c] + sA[c * PITCH + r];
                __stcs(y2 + (C0 + r) * b + (R0 + c), w);
                s2 += w;
            }
        }
    }
}

// Records one item's tile sums; the CTA that completes an output block folds
// its tile sums, and the one completing the last block folds the block sums.
// Called by all 32 lanes of one warp after t1/t2 are final.
__device__ __forceinline__ void finish_item(const TsParams& p, const m4d_ts_task& task, int tr, int tc,
                                            bool second, int slot2, double t1, double t2, int lane) {
    const int T = p.T;
    const int tiles = T * T;
    int fin0 = -1, fin1 = -1;
    if (lane == 0) {
        p.tile_sums[static_cast<int64_t>(task.slot_y) * tiles + tr * T + tc] = t1;
        if (second) p.tile_sums[static_cast<int64_t>(slot2) * tiles + tc * T + tr] = t2;
        __threadfence();
        if (second && slot2 == task.slot_y) {
            if (atomicAdd(p.block_done + task.slot_y, 2u) + 2u == static_cast<unsigned>(tiles)) fin0 = task.slot_y;
        } else {
            if (atomicAdd(p.block_done + task.slot_y, 1u) + 1u == static_cast<unsigned>(tiles)) fin0 = task.slot_y;
            if (second && atomicAdd(p.block_done + slot2, 1u) + 1u == static_cast<unsigned>(tiles)) fin1 = slot2;
        }
        __threadfence();
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
            p.block_done[slot] = 0;  // re-arm for the next run
            __threadfence();
            last = atomicAdd(p.all_done, 1u) + 1u == static_cast<unsigned>(p.nslots);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {  // this CTA completed the last block
            __threadfence();
            const double tot = warp_fold(p.block_sums, p.nslots, lane);
            if (lane == 0) {
                if (p.total) *p.total = tot;
                *p.all_done = 0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// v2: persistent, warp-specialised, TMA-fed.  One CTA per SM; a producer warp
// claims items from a global cursor and streams both x tiles of each item into
// a 3-stage shared-memory ring with cp.async.bulk row copies (mbarrier
// complete_tx); 8 consumer warps transpose-add-store and reduce.  Two tile
// pairs stay in flight while the third is consumed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTmaThreads, 1) ts_kernel_tma(TsParams p) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) uint64_t full_bar[kStages];
    __shared__ __align__(8) uint64_t empty_bar[kStages];
    __shared__ int4 stage_info[kStages];
    __shared__ double part[kStages][2][kWarps];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            m4d::ptx::mbar_init(&full_bar[s], 1);
            m4d::ptx::mbar_init(&empty_bar[s], kWarps);
        }
        m4d::ptx::fence_mbar_init();
    }
    __syncthreads();

    const int64_t b = p.b;
    if (warp == kWarps) {
        // ---------------- producer warp ----------------
        for (int k = 0;; ++k) {
            const int s = k % kStages;
            const uint32_t ph = (k / kStages) & 1;
            m4d::ptx::mbar_wait(&empty_bar[s], ph ^ 1);
            unsigned long long item = 0;
            if (lane == 0) item = atomicAdd(p.work, 1ull);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= static_cast<unsigned long long>(p.items)) {
                if (lane == 0) {
                    stage_info[s] = make_int4(-1, 0, 0, 0);
                    m4d::ptx::mbar_arrive(&full_bar[s]);
                }
                break;
            }
            const Item it = decode_item(p, static_cast<int64_t>(item));
            const m4d_ts_task& task = p.tasks[it.task];
            const int64_t R0 = static_cast<int64_t>(it.tr) * kTile;
            const int64_t C0 = static_cast<int64_t>(it.tc) * kTile;
            const int64_t rows_a = (b - R0 < kTile ? b - R0 : (int64_t)kTile), cols_a = (b - C0 < kTile ? b - C0 : (int64_t)kTile);
            const int64_t rows_b = cols_a, cols_b = rows_a;  // B tile = x(j,i) rows C0.., cols R0..
            const uint32_t bytes = static_cast<uint32_t>((rows_a * cols_a + rows_b * cols_b) * sizeof(double));
            double* sA = smem + static_cast<size_t>(s) * 2 * kTile * kPitchTma;
            double* sB = sA + kTile * kPitchTma;
            if (lane == 0) {
                stage_info[s] = make_int4(it.task, it.tr, it.tc, 1);
                m4d::ptx::mbar_arrive_expect_tx(&full_bar[s], bytes);
            }
            __syncwarp();
            for (int r = lane; r < rows_a; r += 32)
                m4d::ptx::bulk_g2s(sA + r * kPitchTma, task.a + (R0 + r) * b + C0,
                                   static_cast<uint32_t>(cols_a * sizeof(double)), &full_bar[s]);
            for (int r = lane; r < rows_b; r += 32)
                m4d::ptx::bulk_g2s(sB + r * kPitchTma, task.bt + (C0 + r) * b + R0,
                                   static_cast<uint32_t>(cols_b * sizeof(double)), &full_bar[s]);
        }
    } else {
        // ---------------- consumer warps ----------------
        for (int k = 0;; ++k) {
            const int s = k % kStages;
            const uint32_t ph = (k / kStages) & 1;
            m4d::ptx::mbar_wait(&full_bar[s], ph);
            const int4 info = stage_info[s];
            if (info.w < 0) break;
            const m4d_ts_task task = p.tasks[info.x];
            const int tr = info.y, tc = info.z;
            const bool second = task.diag ? (tr != tc) : (task.y2 != nullptr);
            double* const y2 = task.diag ? task.y : task.y2;
            const int slot2 = task.diag ? task.slot_y : task.slot_y2;
            const double* sA = smem + static_cast<size_t>(s) * 2 * kTile * kPitchTma;
            const double* sB = sA + kTile * kPitchTma;
            double s1 = 0.0, s2 = 0.0;
            transpose_add_tile<kPitchTma>(sA, sB, task.y, y2, second, b, static_cast<int64_t>(tr) * kTile,
                                          static_cast<int64_t>(tc) * kTile, warp, lane, s1, s2);
            __syncwarp();
            if (lane == 0) m4d::ptx::mbar_arrive(&empty_bar[s]);  // this warp is done with the stage
            s1 = warp_sum(s1);
            s2 = warp_sum(s2);
            if (lane == 0) {
                part[s][0][warp] = s1;
                part[s][1][warp] = s2;
            }
            m4d::ptx::named_barrier(1, kThreads);
            if (warp == 0) {
                double t1 = 0.0, t2 = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) { t1 += part[s][0][w]; t2 += part[s][1][w]; }
                finish_item(p, task, tr, tc, second, slot2, t1, t2, lane);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.exits, 1u) + 1u == gridDim.x) {  // last CTA out re-arms the cursor
            *p.work = 0;
            *p.exits = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// v1: one CTA per tile item, LDG-staged (fallback for odd block edges or
// pointers that are not 16-byte aligned, which TMA rows cannot express).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 3) ts_kernel_ldg(TsParams p) {
    extern __shared__ double smem[];
    double* sA = smem;
    double* sB = smem + kTile * kPitchLdg;
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
    transpose_add_tile<kPitchLdg>(sA, sB, task.y, y2, second, b, R0, C0, warp, lane, s1, s2);
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
        finish_item(p, task, tr, tc, second, slot2, t1, t2, lane);
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

}  // namespace

struct m4d_ts_plan {
    int device = 0;
    int64_t b = 0;
    int T = 0;
    int ntasks = 0;
    int nslots = 0;
    int64_t items = 0;
    m4d_ts_task* d_tasks = nullptr;
    int64_t* d_off = nullptr;
    double* d_tile_sums = nullptr;
    unsigned* d_counters = nullptr;  // nslots block counters, all_done, exits
    unsigned long long* d_work = nullptr;
    bool tma = false;                // TMA-fed persistent kernel usable
    int sms = 148;
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

int m4d_ts_launches_per_run(void) { return 1; }

m4d_status m4d_ts_plan_create(int device, const m4d_ts_task* tasks, int ntasks, int64_t block,
                              int nslots, m4d_ts_plan** plan_out) {
    *plan_out = nullptr;
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
    auto cleanup = [&](int code) {
        m4d_ts_plan_destroy(plan);
        return code;
    };
    cudaError_t e;
    if ((e = cudaSetDevice(device)) != cudaSuccess) return cleanup(m4d::cuda_fail(e, "cudaSetDevice"));
    if (ntasks) {
        if ((e = cudaMalloc(&plan->d_tasks, sizeof(m4d_ts_task) * ntasks)) != cudaSuccess ||
            (e = cudaMemcpy(plan->d_tasks, tasks, sizeof(m4d_ts_task) * ntasks, cudaMemcpyHostToDevice)) !=
                cudaSuccess)
            return cleanup(m4d::cuda_fail(e, "plan tasks"));
    }
    if ((e = cudaMalloc(&plan->d_off, sizeof(int64_t) * (ntasks + 1))) != cudaSuccess ||
        (e = cudaMemcpy(plan->d_off, off.data(), sizeof(int64_t) * (ntasks + 1), cudaMemcpyHostToDevice)) !=
            cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "plan offsets"));
    if ((e = cudaMalloc(&plan->d_tile_sums, sizeof(double) * std::max<int64_t>(1, tiles * nslots))) !=
            cudaSuccess ||
        (e = cudaMalloc(&plan->d_counters, sizeof(unsigned) * (nslots + 2))) != cudaSuccess ||
        (e = cudaMemset(plan->d_counters, 0, sizeof(unsigned) * (nslots + 2))) != cudaSuccess ||
        (e = cudaMalloc(&plan->d_work, sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMemset(plan->d_work, 0, sizeof(unsigned long long))) != cudaSuccess)
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
    // TMA rows need 16-byte aligned row starts and sizes: even block edge and
    // 16-byte aligned block bases.  M4D_TS_FORCE_LDG=1 selects the v1 kernel.
    plan->tma = (block % 2 == 0) && !getenv("M4D_TS_FORCE_LDG");
    for (int t = 0; t < ntasks && plan->tma; ++t)
        if ((reinterpret_cast<uintptr_t>(tasks[t].a) | reinterpret_cast<uintptr_t>(tasks[t].bt)) & 15)
            plan->tma = false;
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
    TsParams p;
    p.tasks = plan->d_tasks;
    p.item_off = plan->d_off;
    p.ntasks = plan->ntasks;
    p.T = plan->T;
    p.b = plan->b;
    p.nslots = plan->nslots;
    p.items = plan->items;
    p.tile_sums = plan->d_tile_sums;
    p.block_done = plan->d_counters;
    p.all_done = plan->d_counters + plan->nslots;
    p.exits = plan->d_counters + plan->nslots + 1;
    p.work = plan->d_work;
    p.block_sums = block_sums;
    p.total = total;
    if (plan->tma) {
        const int64_t grid = std::min<int64_t>(plan->sms, plan->items);
        ts_kernel_tma<<<static_cast<unsigned>(grid), kTmaThreads, kSmemTma, s>>>(p);
    } else {
        ts_kernel_ldg<<<static_cast<unsigned>(plan->items), kThreads, kSmemLdg, s>>>(p);
    }
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

m4d_status m4d_ts_plan_destroy(m4d_ts_plan* plan) {
    if (!plan) return M4D_OK;
    cudaFree(plan->d_tasks);
    cudaFree(plan->d_off);
    cudaFree(plan->d_tile_sums);
    cudaFree(plan->d_counters);
    cudaFree(plan->d_work);
    delete plan;
    return M4D_OK;
}

}  // extern "C"
