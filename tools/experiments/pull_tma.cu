// Experiment (rejected): a TMA pull kernel for rendezvous device frames -- one CTA per
// SM, one thread driving a ring of shared-memory slots (cp.async.bulk peer HBM -> smem,
// smem -> local HBM).  2 x B200 osu_bw (GB/s at 4 / 16 / 64 MiB), run back to back with
// the LDG kernel: 4 x 32 KB slots 671 / 725 / 788, 16 x 8 KB slots 680 / 729 / 788,
// LDG kernel 689-702 / 761-762 / 786.  The pull kernel is not what limits 4 MiB windows
// (receiver posting takes ~200 us of a ~390 us window).  Drop-in for pull.cu.
// TMA pull: one CTA per SM, one thread drives a 4-slot shared-memory ring of
// 32 KB chunks -- cp.async.bulk reads from the peer's HBM (NVLink) into a slot,
// cp.async.bulk writes the slot to the local destination -- keeping three
// chunk reads (96 KB) in flight per SM with no registers holding data.  All
// messages of the batch must be 16-byte aligned at both ends with a length
// that is a multiple of 16 (launch_pull_batch checks; the LDG kernel below
// takes the rest).  Chunk c of the batch (messages cut into 32 KB pieces,
// concatenated) goes to CTA c mod grid.
constexpr int kTmaChunk = 8 * 1024;
constexpr int kTmaSlots = 16;

__global__ void __launch_bounds__(32, 1) pull_tma_kernel(m4d::PullBatch batch) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ uint64_t bar[kTmaSlots];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kTmaSlots; ++s) m4d::ptx::mbar_init(&bar[s], 1);
    m4d::ptx::fence_mbar_init();
    size_t first[m4d::kMaxPull + 1];  // first chunk of each message
    first[0] = 0;
    for (int k = 0; k < batch.n; ++k) first[k + 1] = first[k] + (batch.d[k].len + kTmaChunk - 1) / kTmaChunk;
    const size_t chunks = first[batch.n];
    const size_t mine = chunks > blockIdx.x ? (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto locate = [&](size_t j, const uint8_t** src, uint8_t** dst, uint32_t* bytes) {
        const size_t c = blockIdx.x + j * gridDim.x;
        int k = 0;
        while (first[k + 1] <= c) ++k;
        const size_t off = (c - first[k]) * kTmaChunk;
        const size_t left = batch.d[k].len - off;
        *src = batch.d[k].src + off;
        *dst = batch.d[k].dst + off;
        *bytes = static_cast<uint32_t>(left < kTmaChunk ? left : kTmaChunk);
    };
    auto load = [&](size_t j) {
        const uint8_t* src;
        uint8_t* dst;
        uint32_t bytes;
        locate(j, &src, &dst, &bytes);
        const int s = static_cast<int>(j % kTmaSlots);
        m4d::ptx::mbar_arrive_expect_tx(&bar[s], bytes);
        m4d::ptx::bulk_g2s(ring + s * kTmaChunk, src, bytes, &bar[s]);
    };
    for (size_t j = 0; j < mine && j < kTmaSlots; ++j) load(j);
    for (size_t j = 0; j < mine; ++j) {
        const int s = static_cast<int>(j % kTmaSlots);
        m4d::ptx::mbar_wait(&bar[s], static_cast<uint32_t>((j / kTmaSlots) & 1));
        const uint8_t* src;
        uint8_t* dst;
        uint32_t bytes;
        locate(j, &src, &dst, &bytes);
        m4d::ptx::bulk_s2g(dst, ring + s * kTmaChunk, bytes);
        m4d::ptx::bulk_commit();
        // refill the slot of chunk j - 1 once its write has read the slot (the write
        // of chunk j may still be reading its own)
        if (j >= 1 && j - 1 + kTmaSlots < mine) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            load(j - 1 + kTmaSlots);
        }
    }
    m4d::ptx::bulk_wait_all();
}

