// Probe: host-observed round trip through a resident polling kernel (the eager
// proxy's mechanism, csrc/pull.cu), one process, GPU 0 (peer GPU 1 if present):
//   doorbell  host stores seq into pinned mapped memory; the kernel (polling it
//             with ld.relaxed.sys) answers by storing seq into another pinned word;
//             host spins on the answer.  = PCIe poll + PCIe posted write floor.
//   local     same, plus a 1 B .. 64 KiB copy into local HBM and __threadfence_system
//   peer      same, copy into GPU 1's HBM over NVLink
// Each mode: 20000 round trips after 2000 warm-up, mean and min of one-way (RTT)
// in us (one trip host->GPU->host; the proxy path's one-way latency adds the
// receiving host's poll of the answer, which is this same PCIe write).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o proxy_probe proxy_probe.cu
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

struct Ctl {
    alignas(64) volatile uint64_t cmd;   // host -> gpu: seq (0 = none yet), ~0 = stop
    alignas(64) volatile uint64_t len;   // bytes to copy for this command
    alignas(64) volatile uint64_t ack;   // gpu -> host
};

__device__ __forceinline__ uint64_t ld_sys(const volatile uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads) poller(Ctl* c, const uint8_t* src, uint8_t* dst, int fence) {
    __shared__ uint64_t s_seq, s_len;
    uint64_t last = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            uint64_t v;
            do { v = ld_sys(&c->cmd); } while (v == last);
            s_seq = v;
            s_len = v == ~0ull ? 0 : ld_sys(&c->len);
        }
        __syncthreads();
        const uint64_t seq = s_seq, len = s_len;
        __syncthreads();
        if (seq == ~0ull) return;
        last = seq;
        const uint64_t body = len / 16;
        for (uint64_t i = threadIdx.x; i < body; i += kThreads)
            reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
        for (uint64_t i = body * 16 + threadIdx.x; i < len; i += kThreads) dst[i] = src[i];
        if (fence) __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&c->ack), "l"(seq) : "memory");
    }
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int kThreads>
static void run(const char* name, Ctl* c, Ctl* cd, const uint8_t* src, uint8_t* dst, uint64_t len, int fence) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    c->cmd = 0;
    c->ack = 0;
    poller<kThreads><<<1, kThreads, 0, s>>>(cd, src, dst, fence);
    CK(cudaGetLastError());
    const int warm = 2000, iters = 20000;
    double sum = 0, best = 1e9;
    for (int k = 1; k <= warm + iters; ++k) {
        c->len = len;
        const double t0 = now_us();
        __atomic_store_n(&c->cmd, (uint64_t)k, __ATOMIC_SEQ_CST);
        while (__atomic_load_n(&c->ack, __ATOMIC_ACQUIRE) != (uint64_t)k) {
        }
        const double dt = now_us() - t0;
        if (k > warm) {
            sum += dt;
            if (dt < best) best = dt;
        }
    }
    c->cmd = ~0ull;
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamDestroy(s));
    printf("%-9s %3d thr %6llu B  RTT mean %6.2f us  min %6.2f us\n", name, kThreads, (unsigned long long)len,
           sum / iters, best);
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    CK(cudaSetDevice(0));
    if (ndev > 1) CK(cudaDeviceEnablePeerAccess(1, 0));
    Ctl* c = nullptr;
    CK(cudaHostAlloc(&c, sizeof(Ctl), cudaHostAllocMapped));
    Ctl* cd = nullptr;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&cd), c, 0));
    uint8_t *src, *dst, *peer = nullptr;
    CK(cudaMalloc(&src, 1 << 20));
    CK(cudaMalloc(&dst, 1 << 20));
    if (ndev > 1) {
        CK(cudaSetDevice(1));
        CK(cudaMalloc(&peer, 1 << 20));
        CK(cudaSetDevice(0));
    }
    run<128>("doorbell", c, cd, src, dst, 0, 0);
    run<128>("doorbell", c, cd, src, dst, 0, 1);
    for (uint64_t len : {1ull, 4096ull, 65536ull}) {
        run<128>("local", c, cd, src, dst, len, 1);
        if (peer) {
            run<128>("peer", c, cd, src, peer, len, 1);
            run<512>("peer", c, cd, src, peer, len, 1);
            run<1024>("peer", c, cd, src, peer, len, 1);
        }
    }
    return 0;
}
