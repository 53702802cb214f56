// Experiment (rejected): two 512-thread join CTAs per SM with a 6-byte fingerprint table and
// 16-bit CAS-inserted heads, fingerprint matches confirmed on the full key by a load of the
// build row in the counting walk.  1e8 rows/side, one B200: 2.84 ms vs 1.58 ms for the
// one-CTA chained join (ncu: long-scoreboard stalls 7.9 per issue from the confirm loads,
// 1.40 G warp instructions, DRAM read 4.6 GB).  Parity held (key_merge GPU tests).

// Paired join (default): two independent 512-thread CTAs per SM, each joining a
// whole partition, so one CTA's build / probe / emit phases -- and the tail
// when its slowest warp finishes -- overlap the other's (the one-CTA-per-SM
// join spends ~20 % of its stall samples at barriers and EXIT).  Half the
// shared memory per CTA needs a compact table: per build row a 32-bit
// fingerprint and a 16-bit link, 8192 16-bit chain heads (inserted with a
// 32-bit CAS on the head pair).  A fingerprint match is confirmed on the full
// key with a load of the build row (L2: the partition was just read) in the
// counting walk, so the output reservation counts exact matches only.
constexpr int kPJThreads = 512;
constexpr int kPJHeadBits = 13;
constexpr int kPJHeads = 1 << kPJHeadBits;
constexpr int kPJChunk = 13000;
constexpr int kPJStage = 128;
constexpr int kPJPer = 4;  // rows per thread per batch (2048 rows)
constexpr size_t kPJSmem = kPJChunk * (sizeof(uint32_t) + sizeof(uint16_t)) + kPJHeads * sizeof(uint16_t) +
                           (kPJThreads / 32) * kPJStage * sizeof(uint32_t);
static_assert(2 * (kPJSmem + 1024) <= 228 * 1024, "two paired-join CTAs per SM");
static_assert(kPJChunk < (1 << kIdxBits) && kIdxBits + 11 <= 32 && kPJThreads * kPJPer <= (1 << 11), "packing");

__device__ __forceinline__ void pj_hash(int64_t key, uint32_t* slot, uint32_t* fp) {
    const uint64_t x = static_cast<uint64_t>(key) * 0x9E3779B97F4A7C15ull;
    *slot = static_cast<uint32_t>(x >> (64 - kPJHeadBits));
    *fp = static_cast<uint32_t>(x >> 20);
}

__global__ void __launch_bounds__(kPJThreads, 2)
    join_pair_kernel(const longlong2* __restrict__ build, const int64_t* __restrict__ loff,
                     const longlong2* __restrict__ probe, const int64_t* __restrict__ roff, int64_t* __restrict__ ok,
                     int64_t* __restrict__ ol, int64_t* __restrict__ orr, int64_t capacity,
                     unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ digest) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* bfp = reinterpret_cast<uint32_t*>(smem);                       // [kPJChunk]
    uint32_t* stage_all = bfp + kPJChunk;                                    // [warps][kPJStage]
    uint16_t* link = reinterpret_cast<uint16_t*>(stage_all + (kPJThreads / 32) * kPJStage);  // [kPJChunk]
    uint16_t* head = link + kPJChunk;                                        // [kPJHeads]
    uint32_t* head2 = reinterpret_cast<uint32_t*>(head);                     // head pairs (CAS)
    __shared__ unsigned long long red[kPJThreads / 32][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int T = kPJThreads;
    uint32_t* stage = stage_all + warp * kPJStage;
    unsigned long long cnt = 0, hsum = 0, ksum = 0;
    const int part = blockIdx.x;
    const longlong2* brow = build + loff[part];
    const longlong2* prow = probe + roff[part];
    if (threadIdx.x == 0) {  // both sides of the partition stream into L2 while the table is built
        const int64_t ln = loff[part + 1] - loff[part], rn = roff[part + 1] - roff[part];
        const uint32_t lb = static_cast<uint32_t>((ln < (1 << 20) ? ln : (1 << 20)) * 16);
        const uint32_t rb = static_cast<uint32_t>((rn < (1 << 20) ? rn : (1 << 20)) * 16);
        if (lb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(brow), "r"(lb) : "memory");
        if (rb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(prow), "r"(rb) : "memory");
    }
    if (loff[part + 1] - loff[part] > INT32_MAX || roff[part + 1] - roff[part] > INT32_MAX) __trap();
    const int bn = static_cast<int>(loff[part + 1] - loff[part]);
    const int pn = static_cast<int>(roff[part + 1] - roff[part]);
    const int nch = (bn && pn) ? (bn + kPJChunk - 1) / kPJChunk : 0;
    const int csz = nch ? (bn + nch - 1) / nch : 0;
    for (int ch = 0; ch < nch; ++ch) {
        const int c0 = ch * csz, cn = bn - c0 < csz ? bn - c0 : csz;
        const longlong2* crow = brow + c0;
        if (ch) __syncthreads();  // every warp is done probing the previous chunk's table
        for (int w = threadIdx.x; w < kPJHeads / 2; w += T) head2[w] = 0xffffffffu;
        __syncthreads();
        for (int base = 0; base < cn; base += T * kPJPer) {
            int64_t k[kPJPer];
#pragma unroll
            for (int u = 0; u < kPJPer; ++u) {
                const int i = base + u * T + threadIdx.x;
                k[u] = i < cn ? crow[i].x : 0;
            }
#pragma unroll
            for (int u = 0; u < kPJPer; ++u) {
                const int i = base + u * T + threadIdx.x;
                if (i >= cn) break;
                uint32_t slot, fp;
                pj_hash(k[u], &slot, &fp);
                bfp[i] = fp;
                const uint32_t sh = (slot & 1u) * 16u;
                uint32_t* w = &head2[slot >> 1];
                uint32_t old = *w, assumed;
                do {
                    assumed = old;
                    old = atomicCAS(w, assumed, (assumed & ~(0xffffu << sh)) | (static_cast<uint32_t>(i) << sh));
                } while (old != assumed);
                link[i] = static_cast<uint16_t>(assumed >> sh);
            }
        }
        __syncthreads();
        for (int base = 0; base < pn; base += T * kPJPer) {
            int64_t r[kPJPer];
#pragma unroll
            for (int u = 0; u < kPJPer; ++u) {
                const int j = base + u * T + threadIdx.x;
                r[u] = j < pn ? prow[j].x : 0;
            }
            uint32_t info[kPJPer];  // first matching build row | min(matches, 0xffff) << 16
            uint32_t fpv[kPJPer];
            uint32_t mine = 0;
#pragma unroll
            for (int u = 0; u < kPJPer; ++u) {  // (1) count exact matches
                info[u] = 0;
                fpv[u] = 0;
                if (base + u * T + static_cast<int>(threadIdx.x) >= pn) continue;
                uint32_t slot;
                pj_hash(r[u], &slot, &fpv[u]);
                uint32_t c = 0, first = 0;
                for (uint32_t i = head[slot]; i != kNil; i = link[i])
                    if (bfp[i] == fpv[u] && crow[i].x == r[u]) {
                        first = c ? first : i;
                        ++c;
                    }
                info[u] = first | (c < 0xffffu ? c : 0xffffu) << 16;
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
            for (uint32_t win = 0; win < warp_total; win += kPJStage) {  // warp-uniform rounds
                if (mine && my0 < win + kPJStage && my0 + mine > win) {  // (3) stage
                    uint32_t e = my0;
#pragma unroll
                    for (int u = 0; u < kPJPer; ++u) {
                        const uint32_t c = info[u] >> 16;
                        if (!c) continue;
                        const uint32_t loc = static_cast<uint32_t>(u * T + threadIdx.x) << kIdxBits;
                        const uint32_t first = info[u] & 0xffffu;
                        if (c == 1) {
                            if (e >= win && e < win + kPJStage) stage[e - win] = loc | first;
                            ++e;
                            continue;
                        }
                        for (uint32_t i = first; i != kNil; i = link[i]) {
                            if (bfp[i] != fpv[u] || crow[i].x != r[u]) continue;
                            if (e >= win && e < win + kPJStage) stage[e - win] = loc | i;
                            ++e;
                        }
                    }
                }
                __syncwarp();
                const uint32_t n = warp_total - win < kPJStage ? warp_total - win : kPJStage;
                for (uint32_t q = lane; q < n; q += 32) {  // (4) emit, all lanes
                    const uint32_t ent = stage[q];
                    const longlong2 b = crow[ent & ((1u << kIdxBits) - 1)];
                    const int64_t rv = prow[base + static_cast<int>(ent >> kIdxBits)].y;
                    const unsigned long long pos = wbase + win + q;
                    if (static_cast<int64_t>(pos) < capacity) {
                        ok[pos] = b.x;
                        ol[pos] = b.y;
                        orr[pos] = rv;
                    }
                    ++cnt;
                    hsum += row_hash(b.x, b.y, rv);
                    ksum += static_cast<unsigned long long>(b.x);
                }
                __syncwarp();
            }
        }
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
        cnt = lane < kPJThreads / 32 ? red[lane][0] : 0;
        hsum = lane < kPJThreads / 32 ? red[lane][1] : 0;
        ksum = lane < kPJThreads / 32 ? red[lane][2] : 0;
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

