// K1 rendezvous data mover: the receiver pulls a batch of matched messages from
// peer B200 memory (CUDA-IPC mappings) with one SM copy kernel.
//
// Measured on 2 x B200 (NV18), back-to-back transfers into distinct buffers
// (tools/probes/peer_probe.cu): copy-engine pulls reach 266-380 / 524-634 /
// 681-769 GB/s at 4 / 16 / 64 MiB, this kernel on 4 round-robin streams
// 576 / 769 / 788 GB/s.  Each launch moves up to kMaxPull messages so the
// per-launch ramp is shared when several messages are matched together.
#include <cuda_runtime.h>

#include <cstdlib>

#include "m4d_internal.h"

namespace {

// kIlp: each thread moves kIlp 16-byte words per round, all loads issued before
// any store (the stores may alias the loads as far as the compiler knows, so
// without this it keeps one load in flight per thread).
template <int kIlp>
__global__ void __launch_bounds__(512) pull_kernel(m4d::PullBatch batch) {
    const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (int k = 0; k < batch.n; ++k) {
        const uint8_t* src = batch.d[k].src;
        uint8_t* dst = batch.d[k].dst;
        const size_t len = batch.d[k].len;
        // Vector body when both ends share 16-byte alignment; bytes for the rest.
        size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
        if (((reinterpret_cast<uintptr_t>(src) ^ reinterpret_cast<uintptr_t>(dst)) & 15) != 0) head = len;
        if (head > len) head = len;
        const size_t body = (len - head) / 16;
        const int4* s16 = reinterpret_cast<const int4*>(src + head);
        int4* d16 = reinterpret_cast<int4*>(dst + head);
        size_t i = tid;
        for (; i + (kIlp - 1) * stride < body; i += kIlp * stride) {
            int4 v[kIlp];
#pragma unroll
            for (int u = 0; u < kIlp; ++u) v[u] = __ldcs(s16 + i + u * stride);
#pragma unroll
            for (int u = 0; u < kIlp; ++u) d16[i + u * stride] = v[u];
        }
        for (; i < body; i += stride) d16[i] = __ldcs(s16 + i);
        for (size_t i = tid; i < head; i += stride) dst[i] = src[i];
        for (size_t i = head + body * 16 + tid; i < len; i += stride) dst[i] = src[i];
    }
}

__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kProxyThreads = 512;  // 64 KiB: 128 threads 13.4 us RTT, 512 9.6 (tools/probes/proxy_probe.cu)

// Warp 0, lanes 0-2: read the three words of the slot of command `seq`; true (on
// every lane) when all three carry its tag, the values (untagged) then in w[].
__device__ __forceinline__ bool proxy_fetch(const m4d::ProxyQueue* q, uint64_t seq, uint64_t* w) {
    const uint64_t* slot = q->cmd[seq % m4d::kProxySlots].w;
    const int lane = threadIdx.x;
    const uint64_t v = lane < 3 ? ld_relaxed_sys(slot + lane) : 0;
    const bool ok = lane >= 3 || (v >> m4d::kProxyTagShift) == (seq & 0xffff);
    if (!__all_sync(0xffffffffu, ok)) return false;
    if (lane < 3) w[lane] = v & ((uint64_t(1) << m4d::kProxyTagShift) - 1);
    return true;
}

// The resident eager-copy proxy: one CTA that polls the host-mapped queue,
// copies each command's payload (into a peer's ring over NVLink) and publishes
// its sequence number (system-scope release after a system fence), in order.
// After `idle_ns` without a command it clears q->alive, looks once more
// (Dekker with the host, which stores the command, fences, then reads alive)
// and exits.
__global__ void __launch_bounds__(kProxyThreads) eager_proxy_kernel(m4d::ProxyQueue* q, uint64_t* state,
                                                                   uint64_t* done, uint64_t idle_ns) {
    __shared__ uint64_t cmd[3];
    __shared__ int verdict;  // 1: command in cmd[], 2: exit
    uint64_t seq = *state;
    uint64_t idle_since = globaltimer();
    for (;;) {
        if (threadIdx.x < 32) {
            int v = 0;
            while (!v) {
                if (proxy_fetch(q, seq + 1, cmd)) {
                    v = 1;
                } else if (globaltimer() - idle_since > idle_ns) {
                    if (threadIdx.x == 0) st_relaxed_sys32(&q->alive, 0);
                    __syncwarp();
                    asm volatile("fence.sc.sys;" ::: "memory");
                    if (proxy_fetch(q, seq + 1, cmd)) {
                        if (threadIdx.x == 0) st_relaxed_sys32(&q->alive, 1);
                        v = 1;
                    } else {
                        v = 2;
                    }
                }
            }
            if (threadIdx.x == 0) verdict = v;
        }
        __syncthreads();
        if (verdict == 2) break;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(cmd[0]);
        uint8_t* dst = reinterpret_cast<uint8_t*>(cmd[1]);
        const uint64_t len = cmd[2];
        __syncthreads();  // cmd[] read by every thread before warp 0 polls again
        if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
            const uint64_t body = len / 16;
            for (uint64_t i = threadIdx.x; i < body; i += kProxyThreads)
                reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
            for (uint64_t i = body * 16 + threadIdx.x; i < len; i += kProxyThreads) dst[i] = src[i];
        } else {
            for (uint64_t i = threadIdx.x; i < len; i += kProxyThreads) dst[i] = src[i];
        }
        __threadfence_system();
        __syncthreads();
        ++seq;
        if (threadIdx.x == 0) {
            st_release_sys(done, seq);
            st_relaxed_sys(&q->head, seq);
        }
        idle_since = globaltimer();
    }
    if (threadIdx.x == 0) *state = seq;
}

}  // namespace

namespace m4d {

int launch_eager_proxy(ProxyQueue* q, uint64_t* state, uint64_t* done, uint64_t idle_ns, cudaStream_t stream) {
    eager_proxy_kernel<<<1, kProxyThreads, 0, stream>>>(q, state, done, idle_ns);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? M4D_OK : cuda_fail(e, "eager proxy launch");
}

int pull_batch() {
    static const int b = [] {
        const char* v = getenv("M4D_PULL_BATCH");
        const int x = v ? atoi(v) : 8;
        return x < 1 ? 1 : x > kMaxPull ? kMaxPull : x;
    }();
    return b;
}

// A launch also closes once it holds this many bytes (M4D_PULL_BATCH_BYTES,
// default 16 MiB): 4 x 4 MiB per launch beat 8 x 4 MiB (osu_bw 705 vs 684 GB/s,
// profiles/r1_p2p_batch_sweep.txt) while 1 MiB messages keep 8 per launch
// (a count cap of 4 cut them from 317 to 240 GB/s).
uint64_t pull_batch_bytes() {
    static const uint64_t b = [] {
        const char* v = getenv("M4D_PULL_BATCH_BYTES");
        return v && atoll(v) > 0 ? static_cast<uint64_t>(atoll(v)) : uint64_t(16) << 20;
    }();
    return b;
}

static int pull_ilp() {
    static const int k = [] {
        const char* v = getenv("M4D_PULL_ILP");
        const int x = v ? atoi(v) : 1;
        return x >= 4 ? 4 : x >= 2 ? 2 : 1;
    }();
    return k;
}

int launch_pull_batch(const PullBatch& batch, cudaStream_t stream, int max_ctas) {
    size_t total = 0;
    for (int k = 0; k < batch.n; ++k) total += batch.d[k].len;
    // 2 CTAs of 512 threads per SM saturate NVLink; tiny batches use fewer CTAs.
    // max_ctas caps the grid so pulls can share the GPU with compute kernels.
    const unsigned cap = static_cast<unsigned>(max_ctas > 0 ? max_ctas : 296);
    unsigned grid = static_cast<unsigned>((total + 8191) / 8192);
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    switch (pull_ilp()) {
        case 4: pull_kernel<4><<<grid, 512, 0, stream>>>(batch); break;
        case 2: pull_kernel<2><<<grid, 512, 0, stream>>>(batch); break;
        default: pull_kernel<1><<<grid, 512, 0, stream>>>(batch);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? M4D_OK : cuda_fail(e, "pull kernel launch");
}

}  // namespace m4d
