// Device plumbing exported through the C ABI: errors, streams, events,
// allocation and legacy CUDA IPC (export/import of allocations so a peer
// process on another B200 can read or write them over NVLink).
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <mutex>

#include "m4d_internal.h"

namespace m4d {

static thread_local char g_last_error[512];

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof g_last_error, fmt, ap);
    va_end(ap);
    return code;
}

// cuMemGetAddressRange through the runtime's driver entry point, so the
// library never links libcuda directly (it must load on GPU-less hosts).
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_getAddressRange address_range_fn() {
    static PFN_getAddressRange fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_getAddressRange>(p);
    });
    return fn;
}

typedef CUresult (*PFN_pointerGetAttribute)(void*, CUpointer_attribute, CUdeviceptr);
static PFN_pointerGetAttribute pointer_attribute_fn() {
    static PFN_pointerGetAttribute fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_pointerGetAttribute>(p);
    });
    return fn;
}

typedef CUresult (*PFN_pointerGetAttributes)(unsigned, CUpointer_attribute*, void**, CUdeviceptr);
static PFN_pointerGetAttributes pointer_attributes_fn() {
    static PFN_pointerGetAttributes fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuPointerGetAttributes", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_pointerGetAttributes>(p);
    });
    return fn;
}

int alloc_info(const void* ptr, uint64_t* base, uint64_t* size, uint64_t* buffer_id) {
    // One driver call for range start, range size and buffer id (every device
    // send of the rendezvous path asks); anything it cannot answer takes the
    // two-call path below, which also produces the errors.
    if (PFN_pointerGetAttributes all = pointer_attributes_fn()) {
        CUdeviceptr b = 0;
        size_t sz = 0;
        unsigned long long id = 0;
        CUpointer_attribute which[3] = {CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, CU_POINTER_ATTRIBUTE_RANGE_SIZE,
                                        CU_POINTER_ATTRIBUTE_BUFFER_ID};
        void* out[3] = {&b, &sz, &id};
        if (all(3, which, out, reinterpret_cast<CUdeviceptr>(ptr)) == CUDA_SUCCESS && b && sz && id &&
            reinterpret_cast<uint64_t>(ptr) >= static_cast<uint64_t>(b) &&
            reinterpret_cast<uint64_t>(ptr) < static_cast<uint64_t>(b) + sz) {
            *base = static_cast<uint64_t>(b);
            *size = sz;
            *buffer_id = id;
            return M4D_OK;
        }
    }
    PFN_getAddressRange range = address_range_fn();
    PFN_pointerGetAttribute attr = pointer_attribute_fn();
    if (!range || !attr) return fail(M4D_ERR_CUDA, "driver entry points unavailable");
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (range(&b, &sz, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(M4D_ERR_USAGE, "pointer %p is not a device allocation", ptr);
    unsigned long long id = 0;
    if (attr(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(M4D_ERR_CUDA, "cuPointerGetAttribute(BUFFER_ID) failed for %p", ptr);
    *base = static_cast<uint64_t>(b);
    *size = sz;
    *buffer_id = id;
    return M4D_OK;
}

}  // namespace m4d

using namespace m4d;

extern "C" {

size_t m4d_last_error(char* buf, size_t n) {
    size_t len = strlen(g_last_error);
    if (buf && n) {
        size_t c = len < n - 1 ? len : n - 1;
        memcpy(buf, g_last_error, c);
        buf[c] = 0;
    }
    return len;
}

int m4d_version(void) { return (1 << 16) | 0; }

m4d_status m4d_pointer_device(const void* ptr, int* device) {
    cudaPointerAttributes a;
    M4D_CUDA_TRY(cudaPointerGetAttributes(&a, ptr));
    *device = (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? a.device : -1;
    return M4D_OK;
}

m4d_status m4d_mem_get_info(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    size_t f = 0, t = 0;
    M4D_CUDA_TRY(cudaMemGetInfo(&f, &t));
    *free_bytes = f;
    *total_bytes = t;
    return M4D_OK;
}

int m4d_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

m4d_status m4d_set_device(int device) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    return M4D_OK;
}

m4d_status m4d_stream_create(int device, void** stream_out) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s;
    M4D_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream_out = s;
    return M4D_OK;
}

m4d_status m4d_stream_destroy(void* stream) {
    M4D_CUDA_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
    return M4D_OK;
}

m4d_status m4d_stream_sync(void* stream) {
    M4D_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return M4D_OK;
}

m4d_status m4d_device_sync(int device) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    M4D_CUDA_TRY(cudaDeviceSynchronize());
    return M4D_OK;
}

m4d_status m4d_event_create(void** ev_out) {
    cudaEvent_t e;
    M4D_CUDA_TRY(cudaEventCreate(&e));
    *ev_out = e;
    return M4D_OK;
}

m4d_status m4d_event_destroy(void* ev) {
    M4D_CUDA_TRY(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
    return M4D_OK;
}

m4d_status m4d_event_record(void* ev, void* stream) {
    M4D_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)));
    return M4D_OK;
}

m4d_status m4d_stream_wait_event(void* stream, void* ev) {
    M4D_CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0));
    return M4D_OK;
}

m4d_status m4d_event_sync(void* ev) {
    M4D_CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(ev)));
    return M4D_OK;
}

m4d_status m4d_event_elapsed_ms(void* start, void* stop, float* ms_out) {
    M4D_CUDA_TRY(cudaEventElapsedTime(ms_out, static_cast<cudaEvent_t>(start),
                                      static_cast<cudaEvent_t>(stop)));
    return M4D_OK;
}

m4d_status m4d_malloc(int device, size_t nbytes, void** ptr_out) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    // Whole 2 MiB granules: small cudaMallocs can share one driver chunk, and
    // legacy CUDA IPC then refuses to map a second allocation of that chunk in
    // the peer (cudaErrorAlreadyMapped).  Every m4d allocation is exportable.
    const size_t granule = 2u << 20;
    const size_t rounded = ((nbytes ? nbytes : 1) + granule - 1) / granule * granule;
    M4D_CUDA_TRY(cudaMalloc(ptr_out, rounded));
    return M4D_OK;
}

m4d_status m4d_free(void* ptr) {
    if (m4d::release_exported(ptr)) return M4D_OK;  // freed once the importers unmapped it
    M4D_CUDA_TRY(cudaFree(ptr));
    return M4D_OK;
}

m4d_status m4d_host_alloc(size_t nbytes, void** ptr_out) {
    M4D_CUDA_TRY(cudaHostAlloc(ptr_out, nbytes ? nbytes : 1, cudaHostAllocPortable));
    return M4D_OK;
}

m4d_status m4d_host_free(void* ptr) {
    M4D_CUDA_TRY(cudaFreeHost(ptr));
    return M4D_OK;
}

m4d_status m4d_memcpy(void* dst, const void* src, size_t nbytes, void* stream) {
    if (!nbytes) return M4D_OK;
    M4D_CUDA_TRY(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    return M4D_OK;
}

m4d_status m4d_memset(void* dst, int value, size_t nbytes, void* stream) {
    if (!nbytes) return M4D_OK;
    M4D_CUDA_TRY(cudaMemsetAsync(dst, value, nbytes, static_cast<cudaStream_t>(stream)));
    return M4D_OK;
}

m4d_status m4d_ipc_export(const void* ptr, uint8_t handle_out[64], uint64_t* offset_out) {
    PFN_getAddressRange range = address_range_fn();
    if (!range) return fail(M4D_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(M4D_ERR_USAGE, "pointer %p is not a device allocation", ptr);
    cudaIpcMemHandle_t h;
    M4D_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle_out, &h, 64);
    *offset_out = reinterpret_cast<uint64_t>(ptr) - static_cast<uint64_t>(base);
    return M4D_OK;
}

m4d_status m4d_ipc_import(int device, const uint8_t handle[64], void** base_out) {
    M4D_CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    M4D_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
    return M4D_OK;
}

m4d_status m4d_ipc_close(void* base) {
    M4D_CUDA_TRY(cudaIpcCloseMemHandle(base));
    return M4D_OK;
}

m4d_status m4d_enable_peer(int device, int peer_device) {
    if (device == peer_device) return M4D_OK;
    int ok = 0;
    M4D_CUDA_TRY(cudaDeviceCanAccessPeer(&ok, device, peer_device));
    if (!ok) return fail(M4D_ERR_CONFIGURATION, "device %d cannot access peer %d", device, peer_device);
    M4D_CUDA_TRY(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return M4D_OK;
    }
    M4D_CUDA_TRY(e);
    return M4D_OK;
}

}  // extern "C"
