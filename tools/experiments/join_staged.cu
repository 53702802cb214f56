// Experiment (rejected): TMA-staged key_merge join with a fingerprint table.
// 1e8 rows/side, one B200: 1.99 ms vs 1.58 ms for the register-fed chained join
// (1.26 G vs 0.95 G warp instructions; warps spin on the tile mbarrier: two 32 KB
// tiles cannot keep enough bytes in flight per SM).  Kept for the record; it was a
// drop-in for join_kernel inside csrc/key_merge.cu.

// Staged join (default).  One CTA per partition streams the partition's rows
// through shared memory with TMA bulk copies -- build rows, then probe rows,
// one 2048-row tile ahead of the one being processed -- so no warp waits on
// a global load while building or probing.  The table keeps per build row a
// 32-bit fingerprint and a 16-bit chain link (16384 heads): 6 bytes a row
// instead of the full key, which is what frees the room for the two tiles.
// A fingerprint match is a candidate; the emit step reads the build row from
// global memory (L2: the partition was just streamed), keeps the exact key
// matches (warp ballot), reserves output rows with one atomic per round and
// writes (key, lval, rval) plus the digest.  Partitions above kSJChunk build
// rows are joined in balanced chunks (probe rows streamed once per chunk).
constexpr int kSJThreads = 1024;
constexpr int kSJTile = 2048;
constexpr int kSJChunk = 13000;
constexpr int kSJStage = 64;
constexpr size_t kSJSmem = 2 * kSJTile * sizeof(longlong2) + kSlots * sizeof(uint32_t) +
                           kSJChunk * (sizeof(uint32_t) + sizeof(uint16_t)) +
                           (kSJThreads / 32) * kSJStage * sizeof(uint32_t);
static_assert(kSJSmem + 2048 <= 227 * 1024, "staged join shared memory");
static_assert(kSJChunk < (1 << kIdxBits) && kIdxBits + 11 <= 32, "staged join candidate packing");

__device__ __forceinline__ void sj_hash(int64_t key, uint32_t* slot, uint32_t* fp) {
    const uint64_t x = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull;
    *slot = static_cast<uint32_t>(x >> (64 - kSlotBits));
    *fp = static_cast<uint32_t>(x >> 18);
}

__global__ void __launch_bounds__(kSJThreads, 1)
    join_staged_kernel(const longlong2* __restrict__ build, const int64_t* __restrict__ loff,
                       const longlong2* __restrict__ probe, const int64_t* __restrict__ roff, int64_t* __restrict__ ok,
                       int64_t* __restrict__ ol, int64_t* __restrict__ orr, int64_t capacity,
                       unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ digest) {
    extern __shared__ __align__(128) unsigned char smem[];
    longlong2* stage = reinterpret_cast<longlong2*>(smem);              // [2][kSJTile]
    uint32_t* head = reinterpret_cast<uint32_t*>(stage + 2 * kSJTile);  // [kSlots]
    uint32_t* bfp = head + kSlots;                                      // [kSJChunk]
    uint32_t* est_all = bfp + kSJChunk;                                 // [warps][kSJStage]
    uint16_t* link = reinterpret_cast<uint16_t*>(est_all + (kSJThreads / 32) * kSJStage);  // [kSJChunk]
    __shared__ uint64_t bar[2];
    __shared__ unsigned long long red[kSJThreads / 32][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* est = est_all + warp * kSJStage;
    unsigned long long cnt = 0, hsum = 0, ksum = 0;
    const int part = blockIdx.x;
    const longlong2* brow = build + loff[part];
    const longlong2* prow = probe + roff[part];
    if (loff[part + 1] - loff[part] > INT32_MAX || roff[part + 1] - roff[part] > INT32_MAX) __trap();
    const int bn = static_cast<int>(loff[part + 1] - loff[part]);
    const int pn = static_cast<int>(roff[part + 1] - roff[part]);
    const int nch = (bn && pn) ? (bn + kSJChunk - 1) / kSJChunk : 0;
    const int csz = nch ? (bn + nch - 1) / nch : 0;
    const int ptiles = (pn + kSJTile - 1) / kSJTile;
    const int btiles = (csz + kSJTile - 1) / kSJTile;  // per chunk (the last chunk may need fewer)
    const int per_chunk = btiles + ptiles;
    const int total = nch * per_chunk;
    // tile k of the sequence [chunk 0: build tiles, probe tiles][chunk 1: ...]
    auto tile = [&](int k, bool* is_probe, int* c0, int* off, int* rows) {
        const int ch = k / per_chunk, q = k % per_chunk;
        *c0 = ch * csz;
        const int cn = bn - *c0 < csz ? bn - *c0 : csz;
        if (q < btiles) {
            *is_probe = false;
            *off = q * kSJTile;  // chunk-relative
            *rows = cn - *off < kSJTile ? cn - *off : kSJTile;
        } else {
            *is_probe = true;
            *off = (q - btiles) * kSJTile;
            *rows = pn - *off < kSJTile ? pn - *off : kSJTile;
        }
    };
    auto issue = [&](int k) {
        bool pr;
        int c0, off, rows;
        tile(k, &pr, &c0, &off, &rows);
        uint64_t* b = &bar[k & 1];
        if (rows <= 0) {  // an empty build tile of a short last chunk: complete the phase without bytes
            m4d::ptx::mbar_arrive(b);
            return;
        }
        m4d::ptx::mbar_arrive_expect_tx(b, static_cast<uint32_t>(rows) * 16u);
        m4d::ptx::bulk_g2s(stage + (k & 1) * kSJTile, pr ? prow + off : brow + c0 + off, rows * 16u, b);
    };
    if (threadIdx.x == 0) {
        m4d::ptx::mbar_init(&bar[0], 1);
        m4d::ptx::mbar_init(&bar[1], 1);
        m4d::ptx::fence_mbar_init();
        if (total) {
            // the whole partition streams into L2 while the first tiles are consumed
            const uint32_t lb = static_cast<uint32_t>((bn < (1 << 20) ? bn : (1 << 20)) * 16);
            const uint32_t rb = static_cast<uint32_t>((pn < (1 << 20) ? pn : (1 << 20)) * 16);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(brow), "r"(lb) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(prow), "r"(rb) : "memory");
            issue(0);
        }
    }
    __syncthreads();
    for (int k = 0; k < total; ++k) {
        bool is_probe;
        int c0, off, rows;
        tile(k, &is_probe, &c0, &off, &rows);
        if (!is_probe && off == 0) {  // a chunk starts: empty table (the previous tile's barrier passed)
            for (int sl = threadIdx.x; sl < kSlots; sl += kSJThreads) head[sl] = kEmpty;
            __syncthreads();
        }
        if (threadIdx.x == 0 && k + 1 < total) issue(k + 1);  // buffer (k+1)&1 was released by tile k-1
        m4d::ptx::mbar_wait(&bar[k & 1], (k >> 1) & 1);
        const longlong2* tl = stage + (k & 1) * kSJTile;
        if (!is_probe) {
#pragma unroll
            for (int u = 0; u < kSJTile / kSJThreads; ++u) {
                const int r = u * kSJThreads + threadIdx.x;
                if (r < rows) {
                    const int i = off + r;
                    uint32_t slot, fp;
                    sj_hash(tl[r].x, &slot, &fp);
                    bfp[i] = fp;
                    const uint32_t old = atomicExch(&head[slot], static_cast<uint32_t>(i));
                    link[i] = old == kEmpty ? kNil : static_cast<uint16_t>(old);
                }
            }
        } else {
            constexpr int kPer = kSJTile / kSJThreads;
            uint32_t info[kPer], fpv[kPer], cand = 0;
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                info[u] = 0;
                fpv[u] = 0;
                const int j = u * kSJThreads + threadIdx.x;
                if (j >= rows) continue;
                uint32_t slot;
                sj_hash(tl[j].x, &slot, &fpv[u]);
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
            for (uint32_t win = 0; win < warp_total; win += kSJStage) {  // warp-uniform rounds
                if (cand && e0 < win + kSJStage && e0 + cand > win) {
                    uint32_t e = e0;
#pragma unroll
                    for (int u = 0; u < kPer; ++u) {
                        const uint32_t c = info[u] >> 16;
                        if (!c) continue;
                        const uint32_t loc = static_cast<uint32_t>(u * kSJThreads + threadIdx.x) << kIdxBits;
                        const uint32_t first = info[u] & 0xffffu;
                        if (c == 1) {
                            if (e >= win && e < win + kSJStage) est[e - win] = loc | first;
                            ++e;
                            continue;
                        }
                        for (uint32_t i = first; i != kNil; i = link[i]) {
                            if (bfp[i] != fpv[u]) continue;
                            if (e >= win && e < win + kSJStage) est[e - win] = loc | i;
                            ++e;
                        }
                    }
                }
                __syncwarp();
                const uint32_t n = warp_total - win < kSJStage ? warp_total - win : kSJStage;
                for (uint32_t q0 = 0; q0 < n; q0 += 32) {  // verify, compact, reserve, store
                    const uint32_t q = q0 + lane;
                    int64_t key = 0, lv = 0, rv = 0;
                    bool hit = false;
                    if (q < n) {
                        const uint32_t ent = est[q];
                        const longlong2 b = brow[c0 + static_cast<int>(ent & ((1u << kIdxBits) - 1))];
                        const longlong2 pr = tl[ent >> kIdxBits];
                        hit = b.x == pr.x;
                        key = b.x;
                        lv = b.y;
                        rv = pr.y;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (!m) continue;
                    unsigned long long at = 0;
                    if (lane == 0) at = atomicAdd(cursor, static_cast<unsigned long long>(__popc(m)));
                    at = __shfl_sync(0xffffffffu, at, 0);
                    if (hit) {
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
        }
        __syncthreads();  // tile buffer free; inserts visible before probing
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
            atomicAdd(digest + 0, cnt);
            atomicAdd(digest + 1, hsum);
            atomicAdd(digest + 2, ksum);
        }
    }
}

