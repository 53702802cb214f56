// Internal helpers shared by the libm4d translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "m4d.h"

namespace m4d {

// Records a formatted message for m4d_last_error() and returns `code`.
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

// Allocation containing `ptr`: base, size and the driver's unique buffer id.
int alloc_info(const void* ptr, uint64_t* base, uint64_t* size, uint64_t* buffer_id);

// Rendezvous pulls launched as one SM copy kernel (pull.cu).
constexpr int kMaxPull = 32;  // array capacity; messages per launch = pull_batch() (M4D_PULL_BATCH, default 8)
int pull_batch();
uint64_t pull_batch_bytes();  // a launch also closes at this many bytes (M4D_PULL_BATCH_BYTES)
struct PullDesc {
    const uint8_t* src;
    uint8_t* dst;
    size_t len;
};
struct PullBatch {
    PullDesc d[kMaxPull];
    int n;
};
int launch_pull_batch(const PullBatch& batch, cudaStream_t stream, int max_ctas);

// Eager device copies through a resident proxy kernel (pull.cu): the host writes
// a command into a host-mapped queue, the kernel (one CTA) polls it over PCIe,
// copies the payload into the peer's device ring and then publishes the
// command's sequence number in host memory -- no launch, no event per message.
// A command slot holds three words, each tagged in its top 16 bits with the
// command's sequence number (so a torn read is detected): src, dst, len.
constexpr int kProxySlots = 256;
struct alignas(64) ProxyCmd {
    uint64_t w[3];
    uint64_t pad[5];
};
struct ProxyQueue {
    alignas(64) uint64_t head;   // commands consumed (the kernel writes)
    alignas(64) uint32_t alive;  // a proxy kernel is running (kernel clears it when it idles out)
    alignas(64) ProxyCmd cmd[kProxySlots];
};
constexpr uint64_t kProxyTagShift = 48;
// Launches the proxy kernel on `stream`.  q: device view of the queue; state:
// device word holding the commands done (kept across launches); done: device view
// of the host word that receives each finished command's sequence number.
int launch_eager_proxy(ProxyQueue* q, uint64_t* state, uint64_t* done, uint64_t idle_ns, cudaStream_t stream);

// m4d_free hook: true when a transport took over the free of an allocation it exported
// (deferred until every peer that mapped it closed the mapping; transport.cpp).
bool release_exported(void* ptr);

inline int cuda_fail(cudaError_t err, const char* what) {
    return fail(M4D_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
}

}  // namespace m4d

#define M4D_CUDA_TRY(expr)                                         \
    do {                                                           \
        cudaError_t m4d_err__ = (expr);                            \
        if (m4d_err__ != cudaSuccess) return m4d::cuda_fail(m4d_err__, #expr); \
    } while (0)

// splitmix64 finaliser with the golden-ratio increment (Steele et al. 2014);
// the generator of BASELINE.md §3 / SURVEY.md §8(d).
__host__ __device__ __forceinline__ uint64_t m4d_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
