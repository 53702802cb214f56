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

#include <algorithm>
#include <vector>

#include "m4d_internal.h"

namespace {

constexpr int kTile = 64;
constexpr int kPitch = kTile + 1;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerWarp = kTile / kWarps;  // 8
constexpr size_t kSmemBytes = 2ull * kTile * kPitch * sizeof(double);

struct TsParams {
    const m4d_ts_task* tasks;
    const int64_t* item_off;  // ntasks + 1 prefix offsets of tile items
    int ntasks;
    int T;                    // tiles per block edge
    int64_t b;                // block edge (elements)
    int nslots;
    double* tile_sums;        // [nslots][T*T]
    unsigned* block_done;     // [nslots]
    unsigned* all_done;       // [1]
    double* block_sums;       // [nslots]
    double* total;            // [1] or null
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

__global__ void __launch_bounds__(kThreads, 3) ts_kernel(TsParams p) {
    extern __shared__ double smem[];
    double* sA = smem;                   // sA[r][c] = x(i,j)[R0+r][C0+c]
    double* sB = smem + kTile * kPitch;  // sB[r][c] = x(j,i)[C0+r][R0+c]
    __shared__ double part[2][kWarps];
    __shared__ int finished[2];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t item = blockIdx.x;

    // Locate the task owning this item (prefix offsets, binary search).
    int lo = 0, hi = p.ntasks - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (p.item_off[mid] <= item) lo = mid; else hi = mid - 1;
    }
    const m4d_ts_task task = p.tasks[lo];
    int64_t local = item - p.item_off[lo];
    const int T = p.T;
    int tr, tc;
    if (task.diag) {  // upper triangle of the tile grid, row by row
        tr = 0;
        while (local >= T - tr) { local -= T - tr; ++tr; }
        tc = tr + static_cast<int>(local);
    } else {
        tr = static_cast<int>(local / T);
        tc = static_cast<int>(local % T);
    }
    const bool second = task.diag ? (tr != tc) : (task.y2 != nullptr);
    double* const y2 = task.diag ? task.y : task.y2;
    const int slot2 = task.diag ? task.slot_y : task.slot_y2;

    const int64_t b = p.b;
    const int64_t R0 = static_cast<int64_t>(tr) * kTile;
    const int64_t C0 = static_cast<int64_t>(tc) * kTile;

    // Phase 1: stage both x tiles (coalesced rows, streaming loads).
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            double av = 0.0;
            if (R0 + r < b && C0 + c < b) av = __ldcs(task.a + (R0 + r) * b + (C0 + c));
            sA[r * kPitch + c] = av;
        }
    }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            double bv = 0.0;
            if (C0 + r < b && R0 + c < b) bv = __ldcs(task.bt + (C0 + r) * b + (R0 + c));
            sB[r * kPitch + c] = bv;
        }
    }
    __syncthreads();

    // Phase 2: y(i,j)[R0+r][C0+c] = sA[r][c] + sB[c][r];
    //          y(j,i)[C0+r][R0+c] = sB[r][c] + sA[c][r]   (paired / diagonal).
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
        const int r = warp * kRowsPerWarp + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = lane + 32 * h;
            if (R0 + r < b && C0 + c < b) {
                const double v = sA[r * kPitch + c] + sB[c * kPitch + r];
                __stcs(task.y + (R0 + r) * b + (C0 + c), v);
                s1 += v;
            }
            if (second && C0 + r < b && R0 + c < b) {
                const double w = sB[r * kPitch + c] + sA[c * kPitch + r];
                __stcs(y2 + (C0 + r) * b + (R0 + c), w);
                s2 += w;
            }
        }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
        part[0][warp] = s1;
        part[1][warp] = s2;
    }
    __syncthreads();

    const int tiles = T * T;
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) { t1 += part[0][w]; t2 += part[1][w]; }
        p.tile_sums[static_cast<int64_t>(task.slot_y) * tiles + tr * T + tc] = t1;
        if (second) p.tile_sums[static_cast<int64_t>(slot2) * tiles + tc * T + tr] = t2;
        __threadfence();
        finished[0] = finished[1] = -1;
        if (second && slot2 == task.slot_y) {
            if (atomicAdd(p.block_done + task.slot_y, 2u) + 2u == static_cast<unsigned>(tiles))
                finished[0] = task.slot_y;
        } else {
            if (atomicAdd(p.block_done + task.slot_y, 1u) + 1u == static_cast<unsigned>(tiles))
                finished[0] = task.slot_y;
            if (second && atomicAdd(p.block_done + slot2, 1u) + 1u == static_cast<unsigned>(tiles))
                finished[1] = slot2;
        }
        __threadfence();
    }
    __syncthreads();

    if (warp == 0) {
        for (int f = 0; f < 2; ++f) {
            const int slot = finished[f];
            if (slot < 0) continue;
            const double bs = warp_fold(p.tile_sums + static_cast<int64_t>(slot) * tiles, tiles, lane);
            if (lane == 0) {
                p.block_sums[slot] = bs;
                p.block_done[slot] = 0;  // re-arm for the next run
                __threadfence();
                finished[f] = (atomicAdd(p.all_done, 1u) + 1u == static_cast<unsigned>(p.nslots)) ? -2 : -1;
            }
            __syncwarp();
            if (finished[f] == -2) {  // this CTA completed the last block
                __threadfence();
                const double tot = warp_fold(p.block_sums, p.nslots, lane);
                if (lane == 0) {
                    if (p.total) *p.total = tot;
                    *p.all_done = 0;
                }
            }
        }
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
    unsigned* d_counters = nullptr;  // nslots block counters + 1 global counter
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
        (e = cudaMalloc(&plan->d_counters, sizeof(unsigned) * (nslots + 1))) != cudaSuccess ||
        (e = cudaMemset(plan->d_counters, 0, sizeof(unsigned) * (nslots + 1))) != cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "plan scratch"));
    if ((e = cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes))) != cudaSuccess ||
        (e = cudaFuncSetAttribute(ts_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) !=
            cudaSuccess)
        return cleanup(m4d::cuda_fail(e, "ts_kernel attributes"));
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
    p.tile_sums = plan->d_tile_sums;
    p.block_done = plan->d_counters;
    p.all_done = plan->d_counters + plan->nslots;
    p.block_sums = block_sums;
    p.total = total;
    ts_kernel<<<static_cast<unsigned>(plan->items), kThreads, kSmemBytes, s>>>(p);
    M4D_CUDA_TRY(cudaGetLastError());
    return M4D_OK;
}

m4d_status m4d_ts_plan_destroy(m4d_ts_plan* plan) {
    if (!plan) return M4D_OK;
    cudaFree(plan->d_tasks);
    cudaFree(plan->d_off);
    cudaFree(plan->d_tile_sums);
    cudaFree(plan->d_counters);
    delete plan;
    return M4D_OK;
}

}  // extern "C"
