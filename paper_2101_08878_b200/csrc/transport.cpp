// libm4d transport: the B200 replacement of the reference Transport
// (pkg/src/commshim/transport/base.py:199-306; sim.py / tcp.py behaviour).
//
// One process per GPU (or several ranks in one process for tests).  Every
// rank publishes a POSIX shared-memory segment holding one single-producer /
// single-consumer byte ring per sending peer; the peers map it.  All traffic
// from rank s to rank r goes through ring (s -> r) in post order, so per-key
// FIFO across every protocol follows from ring order, and matching happens at
// the receiver exactly on (channel, source, tag) with no wildcards.
//
// Protocols, chosen per post:
//   * host payload  -> EAGER: the bytes are copied into the ring (fragments
//     of <= frag_bytes) and the send completes as soon as the last fragment
//     is in; an unmatched message is buffered at the receiver.
//   * device payload -> RENDEZVOUS over NVLink: the sender publishes an RTS
//     carrying the CUDA-IPC handle (+ offset) of the allocation; the matching
//     receiver maps it once (cached) and pulls the bytes device-to-device
//     with a copy-engine cudaMemcpyAsync on its own stream, then answers FIN.
//     Device bytes never touch host memory (device_aware = True).
// Truncation fails the receive and, for rendezvous, the send too (the
// reference simulated-fabric semantics, sim.py:115-122).  No host threads:
// everything advances inside m4d_transport_progress (cooperative progress,
// PAPER.md:82).
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <stdlib.h>
#include <fcntl.h>
#include <signal.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <array>
#include <atomic>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "m4d_internal.h"

using m4d::fail;

namespace {

constexpr uint32_t kSegMagic = 0x4D344453;  // "M4DS"
constexpr uint32_t kSegVersion = 3;
constexpr uint64_t kHeaderBytes = 4096;
// Consumer heads of the eager device rings (one u64 per source rank) live in
// the segment header from this offset.
constexpr uint64_t kDevHeadsOff = 1024;
constexpr int kMaxEagerWorld = static_cast<int>((kHeaderBytes - kDevHeadsOff) / 8);
constexpr uint64_t kDevSlotAlign = 256;
constexpr int kStateInit = 0, kStateReady = 1, kStateClosed = 2;

double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}

struct alignas(64) RingCtl {
    std::atomic<uint64_t> tail;  // bytes ever produced (producer writes)
    char pad0[56];
    std::atomic<uint64_t> head;  // bytes ever consumed (consumer writes)
    char pad1[56];
};

struct SegHeader {
    uint32_t magic;
    uint32_t version;
    int32_t world;
    int32_t rank;
    int32_t pid;
    int32_t device;
    std::atomic<int32_t> state;
    int32_t reserved;
    uint64_t ring_bytes;
    uint64_t ring_stride;
    // eager device ring: one device allocation of world * dev_ring_bytes, the
    // region of source s at s * dev_ring_bytes (published once allocated)
    std::atomic<int32_t> dev_ring_ok;
    int32_t reserved2;
    uint64_t dev_ring_bytes;
    uint64_t dev_ring_id;  // driver buffer id (the peers' mapping-cache key)
    uint64_t dev_ring_addr;  // its address in the owner process (peers in the same process use it)
    uint8_t dev_ring_handle[64];
    // eager proxy: sequence number of the last eager device copy this rank's
    // proxy kernel finished (written by the GPU through a host mapping)
    alignas(64) std::atomic<uint64_t> proxy_done;
};
static_assert(sizeof(SegHeader) <= kDevHeadsOff, "segment header fields overlap the device-ring heads");

inline std::atomic<uint64_t>* dev_heads(SegHeader* h) {
    return reinterpret_cast<std::atomic<uint64_t>*>(reinterpret_cast<uint8_t*>(h) + kDevHeadsOff);
}

enum Kind : uint16_t { kPad = 0, kMsg = 1, kCont = 2, kRts = 3, kFin = 4, kBye = 5, kUnmap = 6, kUnmapAck = 7,
                       kEagerDev = 8 };

struct RecHdr {
    uint32_t bytes;  // whole record, 8-byte multiple
    uint16_t kind;
    uint16_t flags;
};

struct MsgRec {  // first (or only) fragment of an eager message; payload follows
    RecHdr h;
    uint32_t channel, tag;
    uint64_t total;
    uint32_t frag;
    uint32_t domain;
};

struct ContRec {  // continuation fragment; payload follows
    RecHdr h;
    uint32_t frag;
    uint32_t reserved;
};

struct RtsRec {
    RecHdr h;
    uint32_t channel, tag;
    uint64_t len;
    uint64_t send_id;
    uint64_t src_ptr;  // sender-process pointer (used when both ranks share a process)
    uint64_t offset;   // ptr - allocation base
    int32_t pid;
    int32_t device;
    uint64_t buffer_id;  // driver-unique id of the allocation (mapping cache key)
    uint8_t handle[64];
};

// An eager device message: its bytes are in the receiver's device ring (region
// of this source) at absolute position pos (ring offset pos % size) -- already
// when the record is written, or (flags bit 1, proxy) once the sender's
// proxy_done reaches seq.
struct EagerDevRec {
    RecHdr h;
    uint32_t channel, tag;
    uint64_t len;
    uint64_t pos;
    uint32_t domain;
    uint32_t reserved;
    uint64_t seq;
};
constexpr uint16_t kEagerFailed = 1, kEagerProxied = 2;

struct FinRec {
    RecHdr h;
    int32_t status;
    uint32_t reserved;
    uint64_t send_id;
    uint64_t bytes;
};

// Allocation lifetime across processes: a sender about to free an allocation it
// exported asks every peer that saw it to close the mapping (kUnmap: exporter
// pid, buffer id, exporter base); the peer closes it once no pull reads it and
// answers kUnmapAck(base); the allocation is cudaFree'd when the last answer
// arrives (cuda_runtime_api.h: an exporter must not free before importers close).
struct UnmapRec {
    RecHdr h;
    int32_t pid;
    uint32_t reserved;
    uint64_t buffer_id;
    uint64_t base;  // exporter-process address, echoed in the ack
};
static_assert(sizeof(UnmapRec) == sizeof(FinRec), "control records share the fin queue");

inline uint64_t align8(uint64_t n) { return (n + 7) & ~7ull; }

struct Ring {
    RingCtl* ctl = nullptr;
    uint8_t* data = nullptr;
    uint64_t cap = 0;
    uint64_t cursor = 0;  // producer: cached tail / consumer: cached head

    uint64_t free_bytes() const { return cap - (cursor - ctl->head.load(std::memory_order_acquire)); }

    // Producer side: room for a record of `bytes` (plus wrap padding)?  Returns
    // the write pointer or nullptr; commit() publishes it.
    uint8_t* reserve(uint64_t bytes) {
        uint64_t pos = cursor % cap;
        uint64_t head = ctl->head.load(std::memory_order_acquire);
        uint64_t used = cursor - head;
        if (pos + bytes > cap) {  // would wrap: pad to the end first
            uint64_t pad = cap - pos;
            if (used + pad + bytes > cap) return nullptr;
            RecHdr* p = reinterpret_cast<RecHdr*>(data + pos);
            p->bytes = static_cast<uint32_t>(pad);
            p->kind = kPad;
            p->flags = 0;
            cursor += pad;
            ctl->tail.store(cursor, std::memory_order_release);
            pos = 0;
            used += pad;
        }
        if (used + bytes > cap) return nullptr;
        return data + pos;
    }

    void commit(uint64_t bytes) {
        cursor += bytes;
        ctl->tail.store(cursor, std::memory_order_release);
    }
};

enum ReqKind { kSend = 0, kRecv = 1 };

struct Req {
    uint64_t id;
    int kind;
    uint32_t channel, tag;
    int peer;
    uint8_t* ptr;
    uint64_t len;
    int domain;
    bool device;        // pointer is device memory (send: rendezvous; recv: H2D / D2D target)
    // send progress
    uint64_t sent = 0;
    bool started = false;
    RtsRec rts;
    // eager device send: the copy into the peer's ring, published when it is done
    bool eager_dev = false;
    bool proxied = false;      // copied by the proxy kernel (no event)
    uint64_t dev_pos = 0;
    cudaEvent_t dev_ev = nullptr;
    uint64_t proxy_seq = 0;
    // receive: an eager device message may complete it by loan (no copy)
    bool loan_ok = false;
    // loan-only receive (no buffer of its own): a rendezvous message is pulled into a
    // transport-owned receive slot, which is then lent like an eager message
    bool loan_only = false;
    // queue membership
    bool in_posted = false;
    bool in_outq = false;
};

struct Unexpected {
    bool rts = false;
    bool eager_dev = false;   // bytes wait in our device ring at dev_pos
    uint64_t dev_pos = 0;
    RtsRec rec;               // rendezvous descriptor
    std::vector<uint8_t> data;  // eager payload so far
    uint64_t total = 0;
    bool complete = false;
};

// Where the fragments of the eager message currently arriving from a peer go.
struct Inbound {
    bool active = false;
    Req* recv = nullptr;                  // matched receive, or
    std::shared_ptr<Unexpected> buf;      // buffered unexpected message, or neither: discard
    uint64_t total = 0, got = 0;
};

struct MapKey {
    int pid = 0;
    uint64_t buffer_id = 0;
    bool mapped = false;  // the source is a CUDA-IPC mapping (not a same-process pointer)
    bool operator<(const MapKey& o) const { return pid != o.pid ? pid < o.pid : buffer_id < o.buffer_id; }
};

struct Copy {
    Req* recv;
    int peer;
    uint64_t send_id;
    uint64_t bytes;
    MapKey src;
};

// One pull launch (or copy-engine copy) and the messages its event completes.
// Launches on one stream finish in order, so only the oldest of each stream
// is ever queried.
struct Launch {
    cudaEvent_t ev;
    std::vector<Copy> msgs;
};

struct PendingPull {
    Req* recv;
    int peer;
    uint64_t send_id;
    const uint8_t* src;
    uint64_t len;
    MapKey key;
};

// A peer allocation mapped through CUDA IPC.
struct PeerMap {
    void* base = nullptr;
    int inflight = 0;          // pulls reading it right now
    bool unmap_requested = false;
    int unmap_peer = -1;       // who asked (gets the ack)
    uint64_t exporter_base = 0;
};

// Largest lone pull that takes the copy engine (M4D_LONE_CE_MAX, bytes; 0 = never).
static uint64_t lone_ce_max() {
    static const uint64_t v = [] {
        const char* e = getenv("M4D_LONE_CE_MAX");
        return e && atoll(e) >= 0 ? static_cast<uint64_t>(atoll(e)) : uint64_t(1) << 20;  // negative: default
    }();
    return v;
}

// Below this a copy-engine memcpy is cheaper than a launch (M4D_SMALL_PULL overrides, bytes).
static uint64_t small_pull() {
    static const uint64_t v = [] {
        const char* e = getenv("M4D_SMALL_PULL");
        return e && atoll(e) >= 0 ? static_cast<uint64_t>(atoll(e)) : uint64_t(64 * 1024);  // negative: default
    }();
    return v;
}

// Eager device protocol: device payloads a sender marks
// eager-capable and of at most M4D_EAGER_DEVICE_MAX bytes (default 64 KiB; 0
// disables) are copied by the SENDER into its region of the receiver's device
// ring and announced by a ring record once the copy is done; larger ones, and
// any that find the ring full, take the rendezvous.  Per source region:
// M4D_EAGER_DEVICE_RING bytes (default 4 MiB).
static uint64_t eager_device_max() {
    static const uint64_t v = [] {
        const char* e = getenv("M4D_EAGER_DEVICE_MAX");
        return e && atoll(e) >= 0 ? static_cast<uint64_t>(atoll(e)) : uint64_t(64) << 10;
    }();
    return v;
}

// The resident proxy kernel moves eager device payloads (M4D_EAGER_PROXY=0: copy
// engine + event per message instead); it exits after M4D_EAGER_PROXY_IDLE_US
// (default 100) without a command and is relaunched by the next one.
static bool eager_proxy_enabled() {
    static const bool v = [] {
        const char* e = getenv("M4D_EAGER_PROXY");
        return !e || strcmp(e, "0") != 0;
    }();
    return v;
}

static uint64_t eager_proxy_idle_ns() {
    static const uint64_t v = [] {
        const char* e = getenv("M4D_EAGER_PROXY_IDLE_US");
        return (e && atoll(e) > 0 ? static_cast<uint64_t>(atoll(e)) : uint64_t(100)) * 1000;
    }();
    return v;
}

static uint64_t eager_ring_bytes() {
    static const uint64_t v = [] {
        const char* e = getenv("M4D_EAGER_DEVICE_RING");
        uint64_t b = e && atoll(e) > 0 ? static_cast<uint64_t>(atoll(e)) : uint64_t(4) << 20;
        b = (b + (1u << 20) - 1) & ~uint64_t((1u << 20) - 1);
        const uint64_t floor_b = ((4 * eager_device_max() + (1u << 20) - 1) >> 20) << 20;
        return b < floor_b ? floor_b : b;
    }();
    return v;
}

inline uint64_t ckey(uint32_t channel, uint32_t tag) { return (static_cast<uint64_t>(channel) << 32) | tag; }

struct DevSlot {
    uint64_t pos, bytes;
    bool released;
};

// An eager device message copied out of our ring into a posted device buffer.
struct EagerCopy {
    Req* recv;
    int peer;
    uint64_t pos;
    uint64_t len;
    cudaEvent_t ev;
};

struct Peer {
    SegHeader* seg = nullptr;  // peer's segment (we produce into ring me->peer inside it)
    size_t seg_len = 0;
    Ring out;                  // ring in the peer's segment, we are the producer
    Ring in;                   // ring in our segment, the peer produces
    int pid = 0;
    bool dead = false;
    bool said_bye = false;
    std::deque<Req*> outq;     // sends not yet fully in the ring, post order
    std::deque<FinRec> fins;   // control records (fin, unmap, unmap ack) waiting for ring space
    std::unordered_map<uint64_t, std::deque<Req*>> posted;
    std::unordered_map<uint64_t, std::deque<std::shared_ptr<Unexpected>>> unexpected;
    Inbound inbound;
    // eager device ring, sender side: our region in the peer's ring (mapped), cursor
    uint8_t* dev_out = nullptr;
    uint64_t dev_out_cap = 0;
    uint64_t dev_prod = 0;
    // receiver side: slots of the peer's region of our ring, in arrival order
    std::deque<DevSlot> dev_in;
    uint64_t dev_in_end = 0;
};

}  // namespace

struct m4d_transport {
    int world = 1, rank = 0, device = -1;
    uint64_t ring_bytes = 0, frag_bytes = 0;
    std::string session;
    std::string seg_name;
    SegHeader* me = nullptr;
    size_t me_len = 0;
    std::vector<Peer> peers;
    std::unordered_map<uint64_t, std::unique_ptr<Req>> reqs;  // live requests by id
    std::unordered_map<uint64_t, Req*> awaiting_fin;           // rendezvous sends by id
    std::vector<std::deque<Launch>> inflight;                   // per pull stream, launch order
    size_t inflight_launches = 0;
    std::vector<PendingPull> pending_pulls;
    bool use_ce = false;                                        // M4D_PULL_ENGINE=ce: copy engine only
    int pull_ctas = 296;                                        // pull-kernel grid cap (M4D_PULL_CTAS / setter)
    std::vector<cudaEvent_t> spare_events;
    std::vector<m4d_completion> done;
    std::map<MapKey, PeerMap> ipc_maps;                         // (pid, buffer id) -> mapping
    std::unordered_map<uint64_t, std::pair<uint64_t, std::array<uint8_t, 64>>> exports;  // buffer id -> (base, handle)
    cudaStream_t stream = nullptr;                             // (kept: first of the pull streams)
    uint8_t* dev_ring = nullptr;                                // eager device ring (our inbound regions)
    uint64_t dev_ring_bytes = 0;                                // per source
    cudaStream_t eager_stream = nullptr;                        // eager copies (into peers' rings, out of ours)
    // eager proxy (pull.cu): host-mapped command queue, its device view, the
    // kernel's persistent state, the device view of me->proxy_done
    m4d::ProxyQueue* pq = nullptr;
    m4d::ProxyQueue* pq_dev = nullptr;
    uint64_t* proxy_state = nullptr;
    uint64_t* proxy_done_dev = nullptr;
    cudaStream_t proxy_stream = nullptr;
    bool me_registered = false;
    bool proxy_broken = false;                                  // a launch failed: copy engine from then on
    uint64_t proxy_seq = 0;                                     // commands issued
    std::deque<Req*> proxy_sends;                               // issued, copy not yet done (seq order)
    std::vector<EagerCopy> eager_copies;
    std::unordered_map<uint64_t, std::pair<uint64_t, uint64_t>> loans;  // recv id -> (device address, token)
    // receive slots of loan-only receives that arrive by rendezvous: kRecvSlot-byte
    // slots carved from kRecvSlab allocations; larger messages get their own
    std::vector<void*> recv_slabs;
    std::vector<uint8_t*> recv_free;
    std::unordered_map<uint64_t, void*> recv_big;
    std::vector<cudaStream_t> pull_streams;                     // copies round-robin over these
    size_t next_stream = 0;
    double last_liveness = 0.0;
    double last_map_attempt = 0.0;
    int unmapped = 0;
    m4d_transport_stats stats{};
};

namespace {

// The eager proxy's queue (host, mapped), state word, stream, and the device view
// of our header (proxy_done).  Failure leaves the copy-engine eager path.
void setup_proxy(m4d_transport* t) {
    void* q = nullptr;
    void* q_dev = nullptr;
    void* me_dev = nullptr;
    void* state = nullptr;
    cudaError_t e = cudaHostAlloc(&q, sizeof(m4d::ProxyQueue), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&q_dev, q, 0);
    if (e == cudaSuccess) {
        e = cudaHostRegister(t->me, kHeaderBytes, cudaHostRegisterMapped);
        t->me_registered = e == cudaSuccess;
    }
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&me_dev, t->me, 0);
    if (e == cudaSuccess) e = cudaMalloc(&state, sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMemset(state, 0, sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->proxy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (q) cudaFreeHost(q);
        if (state) cudaFree(state);
        if (t->me_registered) cudaHostUnregister(t->me);
        t->me_registered = false;
        t->proxy_stream = nullptr;
        return;
    }
    memset(q, 0, sizeof(m4d::ProxyQueue));
    t->pq = static_cast<m4d::ProxyQueue*>(q);
    t->pq_dev = static_cast<m4d::ProxyQueue*>(q_dev);
    t->proxy_state = static_cast<uint64_t*>(state);
    const uint64_t off = reinterpret_cast<uint8_t*>(&t->me->proxy_done) - reinterpret_cast<uint8_t*>(t->me);
    t->proxy_done_dev = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(me_dev) + off);
}

std::string seg_name_for(const std::string& session, int rank) { return "/m4d_" + session + "_" + std::to_string(rank); }

bool pid_alive(int pid) { return pid > 0 && (kill(pid, 0) == 0 || errno != ESRCH); }

uint64_t ring_stride(uint64_t ring_bytes) { return (sizeof(RingCtl) + ring_bytes + 4095) & ~4095ull; }

Ring ring_in(SegHeader* seg, int src) {
    Ring r;
    uint8_t* base = reinterpret_cast<uint8_t*>(seg) + kHeaderBytes + seg->ring_stride * static_cast<uint64_t>(src);
    r.ctl = reinterpret_cast<RingCtl*>(base);
    r.data = base + sizeof(RingCtl);
    r.cap = seg->ring_bytes;
    return r;
}

void complete(m4d_transport* t, Req* r, int status, uint64_t bytes) {
    m4d_completion c;
    c.req_id = r->id;
    c.status = status;
    c.kind = r->kind;
    c.bytes = bytes;
    t->done.push_back(c);
    if (status == M4D_OK) {
        if (r->kind == kSend) {
            t->stats.sends_completed++;
            t->stats.bytes_sent += bytes;
        } else {
            t->stats.recvs_completed++;
            t->stats.bytes_received += bytes;
        }
    }
    t->reqs.erase(r->id);  // frees r
}

cudaEvent_t grab_event(m4d_transport* t) {
    if (!t->spare_events.empty()) {
        cudaEvent_t ev = t->spare_events.back();
        t->spare_events.pop_back();
        return ev;
    }
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return ev;
}

constexpr uint64_t kRecvSlot = 64 << 10, kRecvSlab = 2 << 20;
constexpr uint64_t kPoolToken = uint64_t(1) << 63;  // loan token of a receive slot: bit 63 | address

uint8_t* recv_slot_get(m4d_transport* t, uint64_t len) {
    cudaSetDevice(t->device);
    if (len > kRecvSlot) {
        void* p = nullptr;
        if (cudaMalloc(&p, len) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        t->recv_big[reinterpret_cast<uint64_t>(p)] = p;
        return static_cast<uint8_t*>(p);
    }
    if (t->recv_free.empty()) {
        void* slab = nullptr;
        if (cudaMalloc(&slab, kRecvSlab) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        t->recv_slabs.push_back(slab);
        for (uint64_t off = 0; off < kRecvSlab; off += kRecvSlot) t->recv_free.push_back(static_cast<uint8_t*>(slab) + off);
    }
    uint8_t* p = t->recv_free.back();
    t->recv_free.pop_back();
    return p;
}

void recv_slot_put(m4d_transport* t, uint8_t* p) {
    auto it = t->recv_big.find(reinterpret_cast<uint64_t>(p));
    if (it != t->recv_big.end()) {
        cudaFree(it->second);
        t->recv_big.erase(it);
        return;
    }
    t->recv_free.push_back(p);
}

// A receive whose rendezvous pull finished (or failed): a loan-only receive lends
// its slot (or gives it back on failure), then the receive completes.
void finish_pulled(m4d_transport* t, Req* r, int status, uint64_t bytes) {
    if (r->loan_only) {
        if (status == M4D_OK)
            t->loans[r->id] = std::make_pair(reinterpret_cast<uint64_t>(r->ptr), kPoolToken | reinterpret_cast<uint64_t>(r->ptr));
        else
            recv_slot_put(t, r->ptr);
    }
    complete(t, r, status, bytes);
}

// Receiver: the slot at `pos` of `peer`'s region of our ring is free; the head
// the sender sees advances over every freed slot at the front.
void dev_release(m4d_transport* t, int peer, uint64_t pos) {
    Peer& p = t->peers[peer];
    for (DevSlot& sl : p.dev_in)
        if (sl.pos == pos) {
            sl.released = true;
            break;
        }
    while (!p.dev_in.empty() && p.dev_in.front().released) {
        p.dev_in_end = p.dev_in.front().pos + p.dev_in.front().bytes;
        p.dev_in.pop_front();
    }
    const uint64_t head = p.dev_in.empty() ? p.dev_in_end : p.dev_in.front().pos;
    dev_heads(t->me)[peer].store(head, std::memory_order_release);
}

// Receiver: deliver an eager device message (pos, len) of `peer` to receive r:
// by loan (r accepts one: the ring bytes themselves), by a device-to-device copy
// out of the ring, or by a copy to host memory.
void deliver_eager(m4d_transport* t, int peer, Req* r, uint64_t pos, uint64_t len, bool failed) {
    if (failed) {
        dev_release(t, peer, pos);
        fail(M4D_ERR_TRANSFER, "rank %d's eager device copy failed", peer);
        complete(t, r, M4D_ERR_TRANSFER, 0);
        return;
    }
    if (len > r->len) {
        dev_release(t, peer, pos);
        fail(M4D_ERR_TRUNCATION, "incoming %llu bytes exceed posted buffer of %llu", (unsigned long long)len,
             (unsigned long long)r->len);
        complete(t, r, M4D_ERR_TRUNCATION, 0);
        return;
    }
    uint8_t* src = t->dev_ring + static_cast<uint64_t>(peer) * t->dev_ring_bytes + pos % t->dev_ring_bytes;
    if (r->loan_ok) {
        t->loans[r->id] = std::make_pair(reinterpret_cast<uint64_t>(src), (static_cast<uint64_t>(peer) << 48) | pos);
        t->stats.eager_device_loans++;
        complete(t, r, M4D_OK, len);
        return;
    }
    cudaSetDevice(t->device);
    if (r->device) {
        cudaEvent_t ev = grab_event(t);
        cudaError_t e = ev ? cudaMemcpyAsync(r->ptr, src, len, cudaMemcpyDeviceToDevice, t->eager_stream)
                           : cudaErrorMemoryAllocation;
        if (e == cudaSuccess) e = cudaEventRecord(ev, t->eager_stream);
        if (e != cudaSuccess) {
            if (ev) t->spare_events.push_back(ev);
            m4d::cuda_fail(e, "eager device delivery");
            dev_release(t, peer, pos);
            complete(t, r, M4D_ERR_CUDA, 0);
            return;
        }
        t->eager_copies.push_back(EagerCopy{r, peer, pos, len, ev});
        return;
    }
    const cudaError_t e = cudaMemcpy(r->ptr, src, len, cudaMemcpyDeviceToHost);
    dev_release(t, peer, pos);
    if (e != cudaSuccess) {
        m4d::cuda_fail(e, "eager device delivery to host memory");
        complete(t, r, M4D_ERR_CUDA, 0);
        return;
    }
    complete(t, r, M4D_OK, len);
}

int poll_eager_copies(m4d_transport* t) {
    int n = 0;
    for (size_t i = 0; i < t->eager_copies.size();) {
        EagerCopy& c = t->eager_copies[i];
        const cudaError_t e = cudaEventQuery(c.ev);
        if (e == cudaErrorNotReady) {
            ++i;
            continue;
        }
        if (e != cudaSuccess) m4d::cuda_fail(e, "eager device delivery");
        dev_release(t, c.peer, c.pos);
        complete(t, c.recv, e == cudaSuccess ? M4D_OK : M4D_ERR_CUDA, e == cudaSuccess ? c.len : 0);
        t->spare_events.push_back(c.ev);
        t->eager_copies[i] = t->eager_copies.back();
        t->eager_copies.pop_back();
        ++n;
    }
    return n;
}

// Sends whose proxy copy finished (me->proxy_done passed their sequence number).
int poll_proxy_sends(m4d_transport* t) {
    const uint64_t done = t->me->proxy_done.load(std::memory_order_acquire);
    int n = 0;
    while (!t->proxy_sends.empty() && t->proxy_sends.front()->proxy_seq <= done) {
        Req* r = t->proxy_sends.front();
        t->proxy_sends.pop_front();
        complete(t, r, M4D_OK, r->len);
        ++n;
    }
    return n;
}

int copy_in(m4d_transport* t, Req* r, uint64_t at, const void* src, uint64_t n) {
    if (!n) return M4D_OK;
    if (r->device) {
        cudaError_t e = cudaMemcpy(r->ptr + at, src, n, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return m4d::cuda_fail(e, "eager host->device delivery");
    } else {
        memcpy(r->ptr + at, src, n);
    }
    return M4D_OK;
}

void queue_fin(m4d_transport* t, int peer, uint64_t send_id, int status, uint64_t bytes) {
    FinRec f{};
    f.h.bytes = sizeof(FinRec);
    f.h.kind = kFin;
    f.status = status;
    f.send_id = send_id;
    f.bytes = bytes;
    t->peers[peer].fins.push_back(f);
}

void queue_unmap(m4d_transport* t, int peer, int kind, int32_t pid, uint64_t buffer_id, uint64_t base) {
    UnmapRec u{};
    u.h.bytes = sizeof(UnmapRec);
    u.h.kind = static_cast<uint16_t>(kind);
    u.pid = pid;
    u.buffer_id = buffer_id;
    u.base = base;
    FinRec f;
    memcpy(&f, &u, sizeof f);
    t->peers[peer].fins.push_back(f);
}

// -- process-wide registry of exported allocations (sender side) --------------------------

struct ExportHold {
    m4d_transport* t;
    int peer;
};
struct ExportEntry {
    uint64_t buffer_id = 0;
    std::vector<ExportHold> holds;  // (transport, peer) pairs that were sent an RTS for it
    int acks_pending = 0;           // > 0: the owner freed it; cudaFree when the last ack arrives
};
std::mutex g_exp_mu;
std::unordered_map<uint64_t, ExportEntry> g_exports;  // allocation base -> entry

void note_export(m4d_transport* t, int peer, uint64_t base, uint64_t buffer_id) {
    std::lock_guard<std::mutex> lk(g_exp_mu);
    ExportEntry& e = g_exports[base];
    if (e.buffer_id != buffer_id) e = ExportEntry{buffer_id, {}, 0};  // a new allocation at a reused address
    for (const ExportHold& h : e.holds)
        if (h.t == t && h.peer == peer) return;
    e.holds.push_back(ExportHold{t, peer});
}

// One awaited answer for `base` will never come (ack arrived, peer gone, transport closed).
void settle_export(uint64_t base) {
    std::lock_guard<std::mutex> lk(g_exp_mu);
    auto it = g_exports.find(base);
    if (it == g_exports.end() || it->second.acks_pending <= 0) return;
    if (--it->second.acks_pending == 0) {
        cudaFree(reinterpret_cast<void*>(base));
        g_exports.erase(it);
    }
}

// Drops `t`'s holds (peer == -1: every peer); holds whose answer was awaited settle.
void drop_holds(m4d_transport* t, int peer) {
    std::vector<uint64_t> settle;
    {
        std::lock_guard<std::mutex> lk(g_exp_mu);
        for (auto it = g_exports.begin(); it != g_exports.end();) {
            ExportEntry& e = it->second;
            for (size_t i = 0; i < e.holds.size();) {
                if (e.holds[i].t == t && (peer < 0 || e.holds[i].peer == peer)) {
                    if (e.acks_pending > 0) settle.push_back(it->first);
                    e.holds.erase(e.holds.begin() + static_cast<long>(i));
                } else {
                    ++i;
                }
            }
            if (e.holds.empty() && e.acks_pending == 0) it = g_exports.erase(it);
            else ++it;
        }
    }
    for (uint64_t b : settle) settle_export(b);
}

// Receiver: close a mapping nobody reads any more and answer the exporter.
void close_mapping(m4d_transport* t, std::map<MapKey, PeerMap>::iterator it) {
    cudaIpcCloseMemHandle(it->second.base);
    if (it->second.unmap_requested && it->second.unmap_peer >= 0 && !t->peers[it->second.unmap_peer].dead)
        queue_unmap(t, it->second.unmap_peer, kUnmapAck, 0, it->first.buffer_id, it->second.exporter_base);
    t->ipc_maps.erase(it);
}

void* map_peer_allocation(m4d_transport* t, const RtsRec& rts, MapKey* key, int* status) {
    *status = M4D_OK;
    key->pid = rts.pid;
    key->buffer_id = rts.buffer_id;
    key->mapped = false;
    if (rts.pid == static_cast<int32_t>(getpid())) return reinterpret_cast<void*>(rts.src_ptr);
    key->mapped = true;
    auto it = t->ipc_maps.find(*key);
    if (it != t->ipc_maps.end()) {
        it->second.inflight++;
        return static_cast<uint8_t*>(it->second.base) + rts.offset;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, rts.handle, 64);
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaErrorAlreadyMapped) {
        cudaGetLastError();
        *status = fail(M4D_ERR_CUDA, "rendezvous source shares a driver chunk with an allocation already mapped "
                                     "from rank pid %d: allocate device frames with m4d_malloc (2 MiB granules)",
                       rts.pid);
        return nullptr;
    }
    if (e != cudaSuccess) {
        *status = m4d::cuda_fail(e, "cudaIpcOpenMemHandle (rendezvous source)");
        return nullptr;
    }
    PeerMap& m = t->ipc_maps[*key];
    m.base = base;
    m.inflight = 1;
    return static_cast<uint8_t*>(base) + rts.offset;
}

// A pull from a mapped source finished: close the mapping if its exporter asked.
void pull_done(m4d_transport* t, const MapKey& key) {
    if (!key.mapped) return;
    auto it = t->ipc_maps.find(key);
    if (it == t->ipc_maps.end()) return;
    if (--it->second.inflight <= 0 && it->second.unmap_requested) close_mapping(t, it);
}

// Matched rendezvous: pull the peer's bytes device-to-device (or D2H for a
// host receive buffer), complete on the event.
void start_pull(m4d_transport* t, int peer, Req* r, const RtsRec& rts) {
    if (rts.len > r->len) {
        queue_fin(t, peer, rts.send_id, M4D_ERR_TRUNCATION, 0);
        fail(M4D_ERR_TRUNCATION, "incoming %llu bytes exceed posted buffer of %llu",
             (unsigned long long)rts.len, (unsigned long long)r->len);
        complete(t, r, M4D_ERR_TRUNCATION, 0);
        return;
    }
    if (rts.len == 0) {
        queue_fin(t, peer, rts.send_id, M4D_OK, 0);
        complete(t, r, M4D_OK, 0);
        return;
    }
    int st;
    MapKey key;
    void* src = map_peer_allocation(t, rts, &key, &st);
    if (st != M4D_OK) {
        queue_fin(t, peer, rts.send_id, M4D_ERR_TRANSFER, 0);
        complete(t, r, M4D_ERR_CUDA, 0);
        return;
    }
    if (r->loan_only) {
        r->ptr = recv_slot_get(t, rts.len);
        if (!r->ptr) {
            pull_done(t, key);
            m4d::fail(M4D_ERR_CUDA, "no device memory for a %llu-byte receive slot", (unsigned long long)rts.len);
            queue_fin(t, peer, rts.send_id, M4D_ERR_TRANSFER, 0);
            complete(t, r, M4D_ERR_CUDA, 0);
            return;
        }
    }
    t->pending_pulls.push_back(PendingPull{r, peer, rts.send_id, static_cast<const uint8_t*>(src), rts.len, key});
    t->stats.rendezvous_pulls++;
    t->stats.nvlink_bytes += rts.len;
}

// Issues every pull matched since the last call.  Large ones go out as SM
// copy kernels, up to kMaxPull messages per launch, round-robin over the pull
// streams (several launches in flight); small ones use the copy engine, whose
// fixed cost is lower than a launch.  One event per launch or copy.
void flush_pulls(m4d_transport* t) {
    if (t->pending_pulls.empty()) return;
    cudaSetDevice(t->device);
    auto take_event = [&](cudaEvent_t* ev) -> cudaError_t {
        if (!t->spare_events.empty()) {
            *ev = t->spare_events.back();
            t->spare_events.pop_back();
            return cudaSuccess;
        }
        return cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    };
    auto fail_all = [&](size_t from, size_t to, cudaError_t e) {
        m4d::cuda_fail(e, "rendezvous pull");
        for (size_t i = from; i < to; ++i) {
            PendingPull& pp = t->pending_pulls[i];
            pull_done(t, pp.key);
            queue_fin(t, pp.peer, pp.send_id, M4D_ERR_TRANSFER, 0);
            finish_pulled(t, pp.recv, M4D_ERR_CUDA, 0);
        }
    };
    std::vector<PendingPull>& v = t->pending_pulls;
    size_t i = 0;
    while (i < v.size()) {
        const size_t si = t->next_stream++ % t->pull_streams.size();
        cudaStream_t s = t->pull_streams[si];
        cudaEvent_t ev = nullptr;
        cudaError_t e = take_event(&ev);
        size_t j = i + 1;
        // The SM kernel needs a device destination; host buffers use the copy engine.
        // A lone pull (nothing else pending or in flight: a ping-pong) of up to
        // 1 MiB rides the copy engine, whose latency is lower than a launch's
        // (osu_latency 64 KiB / 256 KiB / 1 MiB: 20.5 / 21.5 / 22.7 us via the
        // kernel, 14.8 / 14.8 / 16.4 us via the copy engine); pulls that arrive
        // together keep the batched kernel, which carries more per window.
        const bool lone = v.size() == 1 && t->inflight_launches == 0;
        auto via_kernel = [&](const PendingPull& pp) {
            return !t->use_ce && pp.len >= small_pull() && pp.recv->device && !(lone && pp.len <= lone_ce_max());
        };
        if (e == cudaSuccess && !via_kernel(v[i])) {
            e = cudaMemcpyAsync(v[i].recv->ptr, v[i].src, v[i].len, cudaMemcpyDefault, s);
        } else if (e == cudaSuccess) {
            m4d::PullBatch batch;
            batch.n = 0;
            uint64_t bytes = 0;
            for (j = i; j < v.size() && batch.n < m4d::pull_batch() && via_kernel(v[j]) &&
                        (batch.n == 0 || bytes + v[j].len <= m4d::pull_batch_bytes());
                 ++j) {
                batch.d[batch.n++] = m4d::PullDesc{v[j].src, v[j].recv->ptr, v[j].len};
                bytes += v[j].len;
            }
            if (m4d::launch_pull_batch(batch, s, t->pull_ctas) != M4D_OK) e = cudaErrorLaunchFailure;
            else t->stats.pull_kernel_launches++;
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev, s);
        if (e != cudaSuccess) {
            if (ev) t->spare_events.push_back(ev);
            fail_all(i, j, e);
        } else {
            Launch l{ev, {}};
            l.msgs.reserve(j - i);
            for (size_t k = i; k < j; ++k)
                l.msgs.push_back(Copy{v[k].recv, v[k].peer, v[k].send_id, v[k].len, v[k].key});
            t->inflight[si].push_back(std::move(l));
            ++t->inflight_launches;
        }
        i = j;
    }
    v.clear();
}

// A receive meets a buffered unexpected message.
void deliver_unexpected(m4d_transport* t, int peer, Req* r, std::shared_ptr<Unexpected> u) {
    if (u->eager_dev) {
        deliver_eager(t, peer, r, u->dev_pos, u->total, u->rec.h.flags & 1);
        return;
    }
    if (u->rts) {
        start_pull(t, peer, r, u->rec);
        return;
    }
    Inbound& in = t->peers[peer].inbound;
    const bool arriving = in.active && in.buf == u;
    if (u->total > r->len) {
        fail(M4D_ERR_TRUNCATION, "incoming %llu bytes exceed posted buffer of %llu",
             (unsigned long long)u->total, (unsigned long long)r->len);
        if (arriving) in.buf.reset();  // remaining fragments are discarded
        complete(t, r, M4D_ERR_TRUNCATION, 0);
        return;
    }
    int st = copy_in(t, r, 0, u->data.data(), u->data.size());
    if (st != M4D_OK) {
        complete(t, r, st, 0);
        return;
    }
    if (arriving) {  // the rest streams straight into the receive buffer
        in.buf.reset();
        in.recv = r;
        return;
    }
    complete(t, r, M4D_OK, u->total);
}

void fail_peer(m4d_transport* t, int peer, int status, const char* why) {
    Peer& p = t->peers[peer];
    if (p.dead) return;
    p.dead = true;
    fail(status, "rank %d %s", peer, why);
    std::vector<Req*> victims;
    for (auto& kv : p.posted)
        for (Req* r : kv.second) victims.push_back(r);
    p.posted.clear();
    if (p.inbound.active && p.inbound.recv) victims.push_back(p.inbound.recv);
    p.inbound = Inbound{};
    for (Req* r : p.outq) victims.push_back(r);
    p.outq.clear();
    for (auto it = t->awaiting_fin.begin(); it != t->awaiting_fin.end();) {
        if (it->second->peer == peer) {
            victims.push_back(it->second);
            it = t->awaiting_fin.erase(it);
        } else {
            ++it;
        }
    }
    for (Req* r : victims) complete(t, r, M4D_ERR_TRANSFER, r->kind == kSend ? r->sent : 0);
    drop_holds(t, peer);  // its answers to unmap requests will never come
}

// -- producer side ---------------------------------------------------------------------

bool flush_fins(m4d_transport* t, Peer& p) {
    while (!p.fins.empty()) {
        uint8_t* w = p.out.reserve(sizeof(FinRec));
        if (!w) return false;
        memcpy(w, &p.fins.front(), sizeof(FinRec));
        p.out.commit(sizeof(FinRec));
        p.fins.pop_front();
    }
    return true;
}

// The proxy kernel is running, or launched now.  Called after a command was
// stored: store, fence, then read `alive` (the kernel clears alive, fences, then
// looks for a command once more), so a command is never left without a kernel.
int ensure_proxy(m4d_transport* t) {
    std::atomic_thread_fence(std::memory_order_seq_cst);
    volatile uint32_t* alive = &t->pq->alive;
    if (*alive) return M4D_OK;
    *alive = 1;
    cudaSetDevice(t->device);
    t->stats.eager_proxy_launches++;
    return m4d::launch_eager_proxy(t->pq_dev, t->proxy_state, t->proxy_done_dev, eager_proxy_idle_ns(),
                                   t->proxy_stream);
}

// An eager device send through the proxy: the command goes into the queue and
// the record into the ring at once (in post order with every other record); the
// receiver takes the record once our proxy_done reaches its sequence number.
bool push_proxied(m4d_transport* t, Peer& p, Req* r) {
    const uint64_t seq = t->proxy_seq + 1;
    if (seq - reinterpret_cast<volatile uint64_t*>(&t->pq->head)[0] > static_cast<uint64_t>(m4d::kProxySlots))
        return false;  // queue full: the kernel is behind
    uint8_t* w = p.out.reserve(sizeof(EagerDevRec));
    if (!w) return false;
    const uint64_t tag = (seq & 0xffff) << m4d::kProxyTagShift;
    const uint64_t cap = p.dev_out_cap;
    const uint64_t pos = r->dev_pos;
    volatile uint64_t* slot = t->pq->cmd[seq % m4d::kProxySlots].w;
    slot[0] = reinterpret_cast<uint64_t>(r->ptr) | tag;
    slot[1] = reinterpret_cast<uint64_t>(p.dev_out + pos % cap) | tag;
    slot[2] = r->len | tag;
    t->proxy_seq = seq;
    const int st = ensure_proxy(t);
    if (st != M4D_OK) {
        // no kernel: void the command (a later kernel must never run it -- the receiver
        // frees the slot of a failed record) and send eager copies by the copy engine
        slot[2] = r->len | ((seq + 1) & 0xffff) << m4d::kProxyTagShift;
        t->proxy_broken = true;
    }
    EagerDevRec* rec = reinterpret_cast<EagerDevRec*>(w);
    rec->h.bytes = sizeof(EagerDevRec);
    rec->h.kind = kEagerDev;
    rec->h.flags = st == M4D_OK ? kEagerProxied : kEagerFailed;
    rec->channel = r->channel;
    rec->tag = r->tag;
    rec->len = r->len;
    rec->pos = pos;
    rec->domain = static_cast<uint32_t>(r->domain);
    rec->reserved = 0;
    rec->seq = seq;
    p.out.commit(sizeof(EagerDevRec));
    r->proxy_seq = seq;
    r->sent = st == M4D_OK ? r->len : 0;
    return true;
}

// Writes as much of the send at the head of the queue as fits; true when the
// whole send is in the ring.
bool push_send(m4d_transport* t, Peer& p, Req* r) {
    if (r->proxied) return push_proxied(t, p, r);
    if (r->eager_dev) {  // publish once the copy into the peer's ring is done
        const cudaError_t e = cudaEventQuery(r->dev_ev);
        if (e == cudaErrorNotReady) return false;
        uint8_t* w = p.out.reserve(sizeof(EagerDevRec));
        if (!w) return false;
        EagerDevRec* rec = reinterpret_cast<EagerDevRec*>(w);
        rec->h.bytes = sizeof(EagerDevRec);
        rec->h.kind = kEagerDev;
        rec->h.flags = e == cudaSuccess ? 0 : 1;  // 1: the copy failed (the receiver frees the slot)
        rec->channel = r->channel;
        rec->tag = r->tag;
        rec->len = r->len;
        rec->pos = r->dev_pos;
        rec->domain = static_cast<uint32_t>(r->domain);
        rec->reserved = 0;
        p.out.commit(sizeof(EagerDevRec));
        if (e != cudaSuccess) m4d::cuda_fail(e, "eager device copy");
        t->spare_events.push_back(r->dev_ev);
        r->dev_ev = nullptr;
        r->sent = e == cudaSuccess ? r->len : 0;
        return true;
    }
    if (r->device) {
        uint8_t* w = p.out.reserve(sizeof(RtsRec));
        if (!w) return false;
        memcpy(w, &r->rts, sizeof(RtsRec));
        p.out.commit(sizeof(RtsRec));
        return true;
    }
    while (!r->started || r->sent < r->len) {
        const uint64_t remaining = r->len - r->sent;
        const uint64_t frag = remaining < t->frag_bytes ? remaining : t->frag_bytes;
        const uint64_t head = r->started ? sizeof(ContRec) : sizeof(MsgRec);
        const uint64_t bytes = align8(head + frag);
        uint8_t* w = p.out.reserve(bytes);
        if (!w) return false;
        if (!r->started) {
            MsgRec* m = reinterpret_cast<MsgRec*>(w);
            m->h.bytes = static_cast<uint32_t>(bytes);
            m->h.kind = kMsg;
            m->h.flags = 0;
            m->channel = r->channel;
            m->tag = r->tag;
            m->total = r->len;
            m->frag = static_cast<uint32_t>(frag);
            m->domain = static_cast<uint32_t>(r->domain);
        } else {
            ContRec* c = reinterpret_cast<ContRec*>(w);
            c->h.bytes = static_cast<uint32_t>(bytes);
            c->h.kind = kCont;
            c->h.flags = 0;
            c->frag = static_cast<uint32_t>(frag);
            c->reserved = 0;
        }
        if (frag) memcpy(w + head, r->ptr + r->sent, frag);
        p.out.commit(bytes);
        r->sent += frag;
        r->started = true;
        t->stats.eager_bytes += frag;
    }
    return true;
}

int flush_peer(m4d_transport* t, int peer) {
    Peer& p = t->peers[peer];
    if (p.dead || !p.seg) return 0;
    if (!flush_fins(t, p)) return 0;
    int progressed = 0;
    while (!p.outq.empty()) {
        Req* r = p.outq.front();
        if (!push_send(t, p, r)) break;
        p.outq.pop_front();
        r->in_outq = false;
        ++progressed;
        if (r->device && !r->eager_dev) {
            t->awaiting_fin[r->id] = r;
        } else if (r->proxied && r->sent == r->len) {
            t->proxy_sends.push_back(r);  // completes once the proxy copied it
        } else if (r->eager_dev && r->sent != r->len) {
            complete(t, r, M4D_ERR_CUDA, 0);
        } else {
            complete(t, r, M4D_OK, r->len);  // eager: complete once the bytes are in the ring
        }
    }
    return progressed;
}

// Sender: start an eager device send -- reserve a slot in our region of the
// peer's device ring and copy the payload into it on the eager stream; the
// record goes out (push_send) once the copy is done.  False: rendezvous instead
// (no ring, or not enough room).
bool try_eager(m4d_transport* t, int q, Req* r) {
    Peer& p = t->peers[q];
    if (!p.seg || p.dead || t->world > kMaxEagerWorld) return false;
    if (!p.dev_out) {
        if (!p.seg->dev_ring_ok.load(std::memory_order_acquire)) return false;
        void* base = nullptr;
        if (p.pid == static_cast<int32_t>(getpid())) {  // ranks sharing this process
            base = reinterpret_cast<void*>(p.seg->dev_ring_addr);
        } else {
            const MapKey key{p.pid, p.seg->dev_ring_id, true};
            auto it = t->ipc_maps.find(key);
            if (it != t->ipc_maps.end()) {
                base = it->second.base;
            } else {
                cudaIpcMemHandle_t h;
                memcpy(&h, p.seg->dev_ring_handle, 64);
                cudaSetDevice(t->device);
                if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    return false;
                }
                t->ipc_maps[key].base = base;
            }
        }
        p.dev_out = static_cast<uint8_t*>(base) + static_cast<uint64_t>(t->rank) * p.seg->dev_ring_bytes;
        p.dev_out_cap = p.seg->dev_ring_bytes;
    }
    const uint64_t cap = p.dev_out_cap;
    const uint64_t need = (r->len + kDevSlotAlign - 1) & ~(kDevSlotAlign - 1);
    uint64_t pos = p.dev_prod, off = pos % cap;
    if (off + need > cap) {  // no wrap inside a slot: skip to the start of the region
        pos += cap - off;
        off = 0;
    }
    const uint64_t head = dev_heads(p.seg)[t->rank].load(std::memory_order_acquire);
    if (pos + need - head > cap) return false;  // full: the receiver still holds those slots
    const uint64_t top = uint64_t(1) << m4d::kProxyTagShift;
    if (t->pq && !t->proxy_broken && reinterpret_cast<uint64_t>(r->ptr) < top && reinterpret_cast<uint64_t>(p.dev_out + off) < top &&
        r->len < top) {
        p.dev_prod = pos + need;
        t->stats.eager_device_sends++;
        t->stats.eager_proxy_copies++;
        r->eager_dev = true;
        r->proxied = true;
        r->dev_pos = pos;
        r->started = true;
        return true;
    }
    cudaEvent_t ev = grab_event(t);
    if (!ev) return false;
    cudaSetDevice(t->device);
    cudaError_t e = cudaMemcpyAsync(p.dev_out + off, r->ptr, r->len, cudaMemcpyDefault, t->eager_stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev, t->eager_stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        t->spare_events.push_back(ev);
        return false;
    }
    p.dev_prod = pos + need;
    t->stats.eager_device_sends++;
    r->eager_dev = true;
    r->dev_pos = pos;
    r->dev_ev = ev;
    r->started = true;  // the slot is taken: the send can no longer be retracted
    return true;
}

// -- consumer side -----------------------------------------------------------------------

void on_msg(m4d_transport* t, int peer, const MsgRec* m) {
    Peer& p = t->peers[peer];
    const uint8_t* payload = reinterpret_cast<const uint8_t*>(m) + sizeof(MsgRec);
    const uint64_t key = ckey(m->channel, m->tag);
    Inbound in;
    in.active = m->frag < m->total;
    in.total = m->total;
    in.got = m->frag;
    auto q = p.posted.find(key);
    if (q != p.posted.end() && !q->second.empty()) {
        Req* r = q->second.front();
        q->second.pop_front();
        if (q->second.empty()) p.posted.erase(q);
        r->in_posted = false;
        if (m->total > r->len) {
            fail(M4D_ERR_TRUNCATION, "incoming %llu bytes exceed posted buffer of %llu",
                 (unsigned long long)m->total, (unsigned long long)r->len);
            complete(t, r, M4D_ERR_TRUNCATION, 0);
            // in.recv stays null: remaining fragments are discarded
        } else {
            int st = copy_in(t, r, 0, payload, m->frag);
            if (st != M4D_OK) {
                complete(t, r, st, 0);
            } else if (!in.active) {
                complete(t, r, M4D_OK, m->total);
            } else {
                in.recv = r;
            }
        }
    } else {
        auto u = std::make_shared<Unexpected>();
        u->total = m->total;
        u->data.assign(payload, payload + m->frag);
        u->complete = !in.active;
        p.unexpected[key].push_back(u);
        if (in.active) in.buf = u;
        t->stats.unexpected_messages++;
    }
    p.inbound = in;
}

void on_cont(m4d_transport* t, int peer, const ContRec* c) {
    Peer& p = t->peers[peer];
    Inbound& in = p.inbound;
    if (!in.active) return;  // stray continuation (stream already failed)
    const uint8_t* payload = reinterpret_cast<const uint8_t*>(c) + sizeof(ContRec);
    if (in.recv) {
        int st = copy_in(t, in.recv, in.got, payload, c->frag);
        if (st != M4D_OK) {
            complete(t, in.recv, st, in.got);
            in.recv = nullptr;
        }
    } else if (in.buf) {
        in.buf->data.insert(in.buf->data.end(), payload, payload + c->frag);
    }
    in.got += c->frag;
    if (in.got >= in.total) {
        if (in.recv) complete(t, in.recv, M4D_OK, in.total);
        if (in.buf) in.buf->complete = true;
        in = Inbound{};
    }
}

void on_rts(m4d_transport* t, int peer, const RtsRec* rts) {
    Peer& p = t->peers[peer];
    const uint64_t key = ckey(rts->channel, rts->tag);
    auto q = p.posted.find(key);
    if (q != p.posted.end() && !q->second.empty()) {
        Req* r = q->second.front();
        q->second.pop_front();
        if (q->second.empty()) p.posted.erase(q);
        r->in_posted = false;
        start_pull(t, peer, r, *rts);
        return;
    }
    auto u = std::make_shared<Unexpected>();
    u->rts = true;
    u->rec = *rts;
    u->total = rts->len;
    u->complete = true;
    p.unexpected[key].push_back(u);
    t->stats.unexpected_messages++;
}

void on_eager_dev(m4d_transport* t, int peer, const EagerDevRec* rec) {
    Peer& p = t->peers[peer];
    p.dev_in.push_back(DevSlot{rec->pos, (rec->len + kDevSlotAlign - 1) & ~(kDevSlotAlign - 1), false});
    const bool failed = rec->h.flags & 1;
    if (!failed) t->stats.nvlink_bytes += rec->len;  // device bytes that reached this rank (as for pulls)
    const uint64_t key = ckey(rec->channel, rec->tag);
    auto q = p.posted.find(key);
    if (q != p.posted.end() && !q->second.empty()) {
        Req* r = q->second.front();
        q->second.pop_front();
        if (q->second.empty()) p.posted.erase(q);
        r->in_posted = false;
        deliver_eager(t, peer, r, rec->pos, rec->len, failed);
        return;
    }
    auto u = std::make_shared<Unexpected>();
    u->eager_dev = true;
    u->dev_pos = rec->pos;
    u->rec.h.flags = failed ? 1 : 0;
    u->total = rec->len;
    u->complete = true;
    p.unexpected[key].push_back(u);
    t->stats.unexpected_messages++;
}

void on_fin(m4d_transport* t, const FinRec* f) {
    auto it = t->awaiting_fin.find(f->send_id);
    if (it == t->awaiting_fin.end()) return;
    Req* r = it->second;
    t->awaiting_fin.erase(it);
    if (f->status == M4D_ERR_TRUNCATION)
        fail(M4D_ERR_TRUNCATION, "peer buffer shorter than the %llu-byte message", (unsigned long long)r->len);
    else if (f->status == M4D_ERR_CANCELLED)
        fail(M4D_ERR_CANCELLED, "the matching receive side purged the message");
    else if (f->status != M4D_OK)
        fail(f->status, "peer failed to pull the message");
    complete(t, r, f->status, f->bytes);
}

void on_unmap(m4d_transport* t, int peer, const UnmapRec* u) {
    auto it = t->ipc_maps.find(MapKey{u->pid, u->buffer_id, true});
    if (it == t->ipc_maps.end()) {  // never mapped here (same process, or a purged send): answer now
        queue_unmap(t, peer, kUnmapAck, 0, u->buffer_id, u->base);
        return;
    }
    it->second.unmap_requested = true;
    it->second.unmap_peer = peer;
    it->second.exporter_base = u->base;
    if (it->second.inflight <= 0) close_mapping(t, it);
}

int drain_peer(m4d_transport* t, int peer) {
    Peer& p = t->peers[peer];
    Ring& ring = p.in;
    const uint64_t tail = ring.ctl->tail.load(std::memory_order_acquire);
    int n = 0;
    while (ring.cursor < tail) {
        const uint64_t pos = ring.cursor % ring.cap;
        const RecHdr* h = reinterpret_cast<const RecHdr*>(ring.data + pos);
        if (h->kind == kEagerDev && (h->flags & kEagerProxied) &&
            p.seg->proxy_done.load(std::memory_order_acquire) < reinterpret_cast<const EagerDevRec*>(h)->seq)
            break;  // its bytes are still on the way: later records wait behind it (FIFO)
        switch (h->kind) {
            case kMsg: on_msg(t, peer, reinterpret_cast<const MsgRec*>(h)); break;
            case kCont: on_cont(t, peer, reinterpret_cast<const ContRec*>(h)); break;
            case kRts: on_rts(t, peer, reinterpret_cast<const RtsRec*>(h)); break;
            case kFin: on_fin(t, reinterpret_cast<const FinRec*>(h)); break;
            case kBye: p.said_bye = true; break;
            case kUnmap: on_unmap(t, peer, reinterpret_cast<const UnmapRec*>(h)); break;
            case kUnmapAck: settle_export(reinterpret_cast<const UnmapRec*>(h)->base); break;
            case kEagerDev: on_eager_dev(t, peer, reinterpret_cast<const EagerDevRec*>(h)); break;
            default: break;  // kPad
        }
        ring.cursor += h->bytes;
        ++n;
    }
    if (n) ring.ctl->head.store(ring.cursor, std::memory_order_release);
    if (p.said_bye && !p.dead) fail_peer(t, peer, M4D_ERR_CLOSED, "closed the connection");
    return n;
}

int poll_copies(m4d_transport* t) {
    int n = 0;
    for (auto& q : t->inflight) {
        while (!q.empty()) {
            Launch& l = q.front();
            const cudaError_t e = cudaEventQuery(l.ev);
            if (e == cudaErrorNotReady) break;
            if (e != cudaSuccess) m4d::cuda_fail(e, "rendezvous copy");
            for (const Copy& c : l.msgs) {
                pull_done(t, c.src);
                if (e == cudaSuccess) {
                    queue_fin(t, c.peer, c.send_id, M4D_OK, c.bytes);
                    finish_pulled(t, c.recv, M4D_OK, c.bytes);
                } else {
                    queue_fin(t, c.peer, c.send_id, M4D_ERR_TRANSFER, 0);
                    finish_pulled(t, c.recv, M4D_ERR_CUDA, 0);
                }
                ++n;
            }
            t->spare_events.push_back(l.ev);
            q.pop_front();
            --t->inflight_launches;
        }
    }
    return n;
}

void check_liveness(m4d_transport* t) {
    const double now = now_s();
    if (now - t->last_liveness < 0.002) return;
    t->last_liveness = now;
    for (int q = 0; q < t->world; ++q) {
        if (q == t->rank || t->peers[q].dead || !t->peers[q].seg) continue;
        Peer& p = t->peers[q];
        if (p.seg->state.load(std::memory_order_acquire) == kStateClosed) {
            drain_peer(t, q);  // take what it sent before leaving
            flush_pulls(t);
            fail_peer(t, q, M4D_ERR_CLOSED, "closed the connection");
        } else if (!pid_alive(p.pid)) {
            fail_peer(t, q, M4D_ERR_TRANSFER, "died");
        }
    }
}

Req* find_req(m4d_transport* t, uint64_t id) {
    auto it = t->reqs.find(id);
    return it == t->reqs.end() ? nullptr : it->second.get();
}

int validate_peer(m4d_transport* t, int peer) {
    if (peer == t->rank) return fail(M4D_ERR_USAGE, "cannot address self");
    if (peer < 0 || peer >= t->world) return fail(M4D_ERR_USAGE, "peer %d outside world of size %d", peer, t->world);
    return M4D_OK;
}

// Maps peer q's segment if it exists and is ready (non-blocking).  Returns
// M4D_OK whether or not it is there yet; ConfigurationError on a mismatch.
int try_map_peer(m4d_transport* t, int q) {
    Peer& p = t->peers[q];
    if (p.seg) return M4D_OK;
    const std::string name = seg_name_for(t->session, q);
    int pfd = shm_open(name.c_str(), O_RDWR, 0600);
    if (pfd < 0) return M4D_OK;
    struct stat sb;
    if (fstat(pfd, &sb) != 0 || static_cast<size_t>(sb.st_size) < kHeaderBytes) {
        close(pfd);
        return M4D_OK;
    }
    void* pm = mmap(nullptr, sb.st_size, PROT_READ | PROT_WRITE, MAP_SHARED, pfd, 0);
    close(pfd);
    if (pm == MAP_FAILED) return M4D_OK;
    SegHeader* ph = static_cast<SegHeader*>(pm);
    if (ph->magic != kSegMagic || ph->state.load(std::memory_order_acquire) != kStateReady) {
        munmap(pm, sb.st_size);
        return M4D_OK;
    }
    if (ph->version != kSegVersion || ph->world != t->world || ph->rank != q || ph->ring_bytes != t->ring_bytes) {
        const int w = ph->world;
        const unsigned long long rb = ph->ring_bytes;
        munmap(pm, sb.st_size);
        return fail(M4D_ERR_CONFIGURATION, "rank %d's segment disagrees (world %d vs %d, ring %llu vs %llu)", q, w,
                    t->world, rb, (unsigned long long)t->ring_bytes);
    }
    p.seg = ph;
    p.seg_len = sb.st_size;
    p.pid = ph->pid;
    p.out = ring_in(p.seg, t->rank);  // we produce into (me -> q) inside q's segment
    return M4D_OK;
}

void map_missing_peers(m4d_transport* t) {
    const double now = now_s();
    if (now - t->last_map_attempt < 0.0005) return;
    t->last_map_attempt = now;
    for (int q = 0; q < t->world; ++q)
        if (q != t->rank && !t->peers[q].seg) try_map_peer(t, q);
}

}  // namespace

namespace m4d {

// m4d_free of an allocation a transport exported: every peer that was sent an RTS
// for it is asked to close its mapping, and the cudaFree waits for their answers
// (settle_export).  Returns true when the free was taken over (deferred).
bool release_exported(void* ptr) {
    const uint64_t base = reinterpret_cast<uint64_t>(ptr);
    std::vector<ExportHold> holds;
    uint64_t id = 0;
    {
        std::lock_guard<std::mutex> lk(g_exp_mu);
        auto it = g_exports.find(base);
        if (it == g_exports.end()) return false;
        if (it->second.acks_pending > 0) return true;  // already being released
        if (it->second.holds.empty()) {
            g_exports.erase(it);
            return false;
        }
        holds = it->second.holds;
        id = it->second.buffer_id;
        it->second.holds.clear();
        it->second.acks_pending = static_cast<int>(holds.size());
    }
    for (const ExportHold& h : holds) {
        h.t->exports.erase(id);
        if (h.t->peers[h.peer].dead) {
            settle_export(base);
            continue;
        }
        queue_unmap(h.t, h.peer, kUnmap, static_cast<int32_t>(getpid()), id, base);
        flush_peer(h.t, h.peer);
    }
    return true;
}

}  // namespace m4d

extern "C" {

m4d_status m4d_transport_open(const m4d_transport_config* cfg, m4d_transport** out) {
    *out = nullptr;
    if (!cfg || cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return fail(M4D_ERR_USAGE, "invalid world/rank");
    if (!cfg->session || !cfg->session[0] || strchr(cfg->session, '/'))
        return fail(M4D_ERR_CONFIGURATION, "transport session name must be non-empty and contain no '/'");
    if (cfg->ring_bytes < 65536 || cfg->ring_bytes % 4096)
        return fail(M4D_ERR_CONFIGURATION, "ring_bytes must be a multiple of 4096 and >= 64 KiB");
    std::unique_ptr<m4d_transport> t(new m4d_transport());
    t->world = cfg->world;
    t->rank = cfg->rank;
    t->device = cfg->device;
    t->ring_bytes = cfg->ring_bytes;
    t->frag_bytes = cfg->ring_bytes / 4 < (256u << 10) ? cfg->ring_bytes / 4 : (256u << 10);
    t->session = cfg->session;
    t->seg_name = seg_name_for(t->session, t->rank);
    t->peers.resize(t->world);

    // Own segment: header + one inbound ring per source rank.
    const uint64_t stride = ring_stride(t->ring_bytes);
    const size_t seg_len = kHeaderBytes + stride * t->world;
    int fd = -1;
    for (int attempt = 0; attempt < 2 && fd < 0; ++attempt) {
        fd = shm_open(t->seg_name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (fd >= 0 || errno != EEXIST) break;
        // Stale segment of a dead process, or a live rank collision?
        int ofd = shm_open(t->seg_name.c_str(), O_RDWR, 0600);
        if (ofd >= 0) {
            struct stat sb;
            bool live = false;
            if (fstat(ofd, &sb) == 0 && static_cast<size_t>(sb.st_size) >= sizeof(SegHeader)) {
                void* m = mmap(nullptr, sizeof(SegHeader), PROT_READ, MAP_SHARED, ofd, 0);
                if (m != MAP_FAILED) {
                    const SegHeader* h = static_cast<const SegHeader*>(m);
                    live = h->magic == kSegMagic && h->state.load() != kStateClosed && pid_alive(h->pid);
                    munmap(m, sizeof(SegHeader));
                }
            }
            close(ofd);
            if (live) return fail(M4D_ERR_CONFIGURATION, "rank %d already initialized in session %s (rank collision)",
                                  t->rank, t->session.c_str());
        }
        shm_unlink(t->seg_name.c_str());
    }
    if (fd < 0) return fail(M4D_ERR_STARTUP, "shm_open(%s): %s", t->seg_name.c_str(), strerror(errno));
    if (ftruncate(fd, static_cast<off_t>(seg_len)) != 0) {
        close(fd);
        shm_unlink(t->seg_name.c_str());
        return fail(M4D_ERR_STARTUP, "ftruncate(%s): %s", t->seg_name.c_str(), strerror(errno));
    }
    void* mem = mmap(nullptr, seg_len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mem == MAP_FAILED) {
        shm_unlink(t->seg_name.c_str());
        return fail(M4D_ERR_STARTUP, "mmap(%s): %s", t->seg_name.c_str(), strerror(errno));
    }
    t->me = static_cast<SegHeader*>(mem);
    t->me_len = seg_len;
    SegHeader* h = t->me;
    h->magic = kSegMagic;
    h->version = kSegVersion;
    h->world = t->world;
    h->rank = t->rank;
    h->pid = static_cast<int32_t>(getpid());
    h->device = t->device;
    h->ring_bytes = t->ring_bytes;
    h->ring_stride = stride;
    for (int s = 0; s < t->world; ++s) {
        Ring r = ring_in(h, s);
        new (r.ctl) RingCtl();
        r.ctl->tail.store(0);
        r.ctl->head.store(0);
    }
    h->state.store(kStateReady, std::memory_order_release);

    for (int q = 0; q < t->world; ++q)
        if (q != t->rank) t->peers[q].in = ring_in(t->me, q);  // inbound rings live in our segment
    (void)cfg->connect_timeout;  // peers are mapped lazily (m4d_transport_wait_ready blocks)
    for (int q = 0; q < t->world; ++q)
        if (q != t->rank) {
            int st = try_map_peer(t.get(), q);
            if (st) {
                m4d_transport* raw = t.release();
                m4d_transport_close(raw);
                return st;
            }
        }

    if (t->device >= 0) {
        cudaError_t e = cudaSetDevice(t->device);
        const int nstreams = getenv("M4D_PULL_STREAMS") ? atoi(getenv("M4D_PULL_STREAMS")) : 4;
        for (int k = 0; k < (nstreams > 0 ? nstreams : 1) && e == cudaSuccess; ++k) {
            cudaStream_t st = nullptr;
            e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
            if (e == cudaSuccess) t->pull_streams.push_back(st);
        }
        if (e == cudaSuccess) t->stream = t->pull_streams[0];
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->eager_stream, cudaStreamNonBlocking);
        // the eager device ring: one region per source rank, published in our header
        if (e == cudaSuccess && eager_device_max() > 0 && t->world > 1 && t->world <= kMaxEagerWorld) {
            const uint64_t rb = eager_ring_bytes();
            void* ring = nullptr;
            uint64_t base = 0, size = 0, id = 0;
            std::array<uint8_t, 64> handle;
            uint64_t off0 = 0;
            if (cudaMalloc(&ring, rb * t->world) == cudaSuccess &&
                m4d::alloc_info(ring, &base, &size, &id) == M4D_OK &&
                m4d_ipc_export(ring, handle.data(), &off0) == M4D_OK) {
                t->dev_ring = static_cast<uint8_t*>(ring);
                t->dev_ring_bytes = rb;
                t->me->dev_ring_bytes = rb;
                t->me->dev_ring_id = id;
                t->me->dev_ring_addr = reinterpret_cast<uint64_t>(ring);
                memcpy(t->me->dev_ring_handle, handle.data(), 64);
                t->me->dev_ring_ok.store(1, std::memory_order_release);
                if (eager_proxy_enabled()) setup_proxy(t.get());
            } else {
                if (ring) cudaFree(ring);
                cudaGetLastError();  // no ring: every device send takes the rendezvous
            }
        }
        t->inflight.resize(t->pull_streams.size());
        if (const char* eng = getenv("M4D_PULL_ENGINE")) t->use_ce = strcmp(eng, "ce") == 0;
        if (const char* c = getenv("M4D_PULL_CTAS")) t->pull_ctas = atoi(c) > 0 ? atoi(c) : 296;
        if (e != cudaSuccess) {
            m4d_transport* raw = t.release();
            m4d_transport_close(raw);
            return m4d::cuda_fail(e, "transport stream");
        }
        int n = 0;
        if (cudaGetDeviceCount(&n) == cudaSuccess)
            for (int d = 0; d < n; ++d)
                if (d != t->device) {
                    int ok = 0;
                    if (cudaDeviceCanAccessPeer(&ok, t->device, d) == cudaSuccess && ok)
                        cudaDeviceEnablePeerAccess(d, 0);
                }
        cudaGetLastError();
    }
    *out = t.release();
    return M4D_OK;
}

m4d_status m4d_transport_post_send(m4d_transport* t, uint32_t channel, int peer, uint32_t tag, const void* ptr,
                                   uint64_t len, int domain, int on_device, uint64_t req_id, m4d_completion* now) {
    now->status = -1;
    int st = validate_peer(t, peer);
    if (st) return st;
    Peer& p = t->peers[peer];
    auto r = std::make_unique<Req>();
    Req* raw = r.get();
    raw->id = req_id;
    raw->kind = kSend;
    raw->channel = channel;
    raw->tag = tag;
    raw->peer = peer;
    raw->ptr = static_cast<uint8_t*>(const_cast<void*>(ptr));
    raw->len = len;
    raw->domain = domain;
    raw->device = (on_device & 1) && len > 0;
    if (raw->device && t->device < 0) return fail(M4D_ERR_USAGE, "device payload on a host-only transport");
    if (p.dead) {
        fail(M4D_ERR_CLOSED, "rank %d connection closed", peer);
        now->req_id = req_id;
        now->status = M4D_ERR_CLOSED;
        now->kind = kSend;
        now->bytes = 0;
        return M4D_OK;
    }
    const bool eager = raw->device && (on_device & 2) && len <= eager_device_max() && try_eager(t, peer, raw);
    if (raw->device && !eager) {
        RtsRec& rts = raw->rts;
        memset(&rts, 0, sizeof rts);
        rts.h.bytes = sizeof(RtsRec);
        rts.h.kind = kRts;
        rts.channel = channel;
        rts.tag = tag;
        rts.len = len;
        rts.send_id = req_id;
        rts.src_ptr = reinterpret_cast<uint64_t>(ptr);
        rts.pid = static_cast<int32_t>(getpid());
        rts.device = t->device;
        uint64_t base = 0, size = 0;
        st = m4d::alloc_info(ptr, &base, &size, &rts.buffer_id);
        if (st) return st;
        rts.offset = reinterpret_cast<uint64_t>(ptr) - base;
        auto ex = t->exports.find(rts.buffer_id);
        if (ex == t->exports.end() || ex->second.first != base) {
            std::array<uint8_t, 64> h;
            uint64_t off0 = 0;
            st = m4d_ipc_export(reinterpret_cast<void*>(base), h.data(), &off0);
            if (st) return st;
            ex = t->exports.insert_or_assign(rts.buffer_id, std::make_pair(base, h)).first;
        }
        memcpy(rts.handle, ex->second.second.data(), 64);
        note_export(t, peer, base, rts.buffer_id);
    }
    t->reqs[req_id] = std::move(r);
    raw->in_outq = true;
    p.outq.push_back(raw);
    const size_t before = t->done.size();
    flush_peer(t, peer);
    // Report an immediate completion (eager send fully in the ring) inline.
    for (size_t i = before; i < t->done.size(); ++i)
        if (t->done[i].req_id == req_id) {
            *now = t->done[i];
            t->done.erase(t->done.begin() + static_cast<long>(i));
            break;
        }
    return M4D_OK;
}

m4d_status m4d_transport_post_recv(m4d_transport* t, uint32_t channel, int peer, uint32_t tag, void* ptr,
                                   uint64_t cap, int domain, int on_device, uint64_t req_id, m4d_completion* now) {
    now->status = -1;
    int st = validate_peer(t, peer);
    if (st) return st;
    Peer& p = t->peers[peer];
    drain_peer(t, peer);  // match against everything that already arrived
    auto r = std::make_unique<Req>();
    Req* raw = r.get();
    raw->id = req_id;
    raw->kind = kRecv;
    raw->channel = channel;
    raw->tag = tag;
    raw->peer = peer;
    raw->ptr = static_cast<uint8_t*>(ptr);
    raw->len = cap;
    raw->domain = domain;
    raw->device = (on_device & 1) && cap > 0;
    raw->loan_ok = (on_device & 2) != 0;  // an eager device message may complete it by loan
    raw->loan_only = (on_device & 4) != 0;
    if (raw->loan_only) {  // no buffer: the transport provides the memory it lends
        if (!(on_device & 1) || t->device < 0) return fail(M4D_ERR_USAGE, "loan-only receives are device receives");
        raw->loan_ok = true;
        raw->device = true;
        raw->ptr = nullptr;
    }
    if (raw->device && t->device < 0) return fail(M4D_ERR_USAGE, "device buffer on a host-only transport");
    t->reqs[req_id] = std::move(r);
    const size_t before = t->done.size();
    const uint64_t key = ckey(channel, tag);
    auto u = p.unexpected.find(key);
    if (u != p.unexpected.end() && !u->second.empty()) {
        std::shared_ptr<Unexpected> msg = u->second.front();
        u->second.pop_front();
        if (u->second.empty()) p.unexpected.erase(u);
        deliver_unexpected(t, peer, raw, msg);
        flush_peer(t, peer);  // a truncation / empty-rendezvous FIN leaves now
    } else if (p.dead) {
        fail(M4D_ERR_CLOSED, "rank %d connection closed", peer);
        complete(t, raw, M4D_ERR_CLOSED, 0);
    } else {
        raw->in_posted = true;
        p.posted[key].push_back(raw);
    }
    // Pulls matched here (this receive, or earlier posted receives whose RTS
    // drain_peer just took) are launched in batches: a window of posted
    // receives becomes a few multi-message launches, not one launch per post.
    // With no pull in flight they go at once, so the link starts while the
    // caller is still posting instead of at its next progress() (measured
    // osu_bw, 4 MiB messages, window 64: a fixed ~120 us per window before).
    if (!t->pending_pulls.empty()) {
        uint64_t bytes = 0;
        for (const PendingPull& pp : t->pending_pulls) bytes += pp.len;
        if (t->pending_pulls.size() >= static_cast<size_t>(m4d::pull_batch()) || bytes >= m4d::pull_batch_bytes() ||
            t->inflight_launches == 0)
            flush_pulls(t);
    }
    for (size_t i = before; i < t->done.size(); ++i)
        if (t->done[i].req_id == req_id) {
            *now = t->done[i];
            t->done.erase(t->done.begin() + static_cast<long>(i));
            break;
        }
    return M4D_OK;
}

m4d_status m4d_transport_post_many(m4d_transport* t, int is_send, uint32_t channel, int peer, uint32_t tag,
                                   void* const* ptrs, const uint64_t* lens, int count, int domain, int on_device,
                                   const uint64_t* req_ids, m4d_completion* now, int* posted) {
    *posted = 0;
    for (int i = 0; i < count; ++i) {
        const m4d_status st = is_send ? m4d_transport_post_send(t, channel, peer, tag, ptrs[i], lens[i], domain,
                                                                on_device, req_ids[i], &now[i])
                                      : m4d_transport_post_recv(t, channel, peer, tag, ptrs[i], lens[i], domain,
                                                                on_device, req_ids[i], &now[i]);
        if (st != M4D_OK) return st;
        *posted = i + 1;
    }
    return M4D_OK;
}

int m4d_transport_progress(m4d_transport* t, m4d_completion* out, int max) {
    map_missing_peers(t);
    // Copies first: a finished pull must send its FIN in this same call, or a
    // sender whose peer stops polling would wait forever.
    if (t->inflight_launches) poll_copies(t);
    if (!t->eager_copies.empty()) poll_eager_copies(t);
    if (!t->proxy_sends.empty()) poll_proxy_sends(t);
    for (int q = 0; q < t->world; ++q)
        if (q != t->rank) {
            drain_peer(t, q);
            flush_peer(t, q);
        }
    flush_pulls(t);
    if (!t->reqs.empty()) check_liveness(t);
    int n = 0;
    const int avail = static_cast<int>(t->done.size());
    n = avail < max ? avail : max;
    if (n > 0) {
        memcpy(out, t->done.data(), sizeof(m4d_completion) * n);
        t->done.erase(t->done.begin(), t->done.begin() + n);
    }
    return n;
}

int m4d_transport_pending_completions(const m4d_transport* t) { return static_cast<int>(t->done.size()); }

m4d_status m4d_transport_cancel(m4d_transport* t, uint64_t req_id, int* cancelled) {
    *cancelled = 0;
    Req* r = find_req(t, req_id);
    if (!r) return M4D_OK;  // already finished
    Peer& p = t->peers[r->peer];
    if (r->kind == kRecv && r->in_posted) {
        auto q = p.posted.find(ckey(r->channel, r->tag));
        if (q != p.posted.end()) {
            for (auto it = q->second.begin(); it != q->second.end(); ++it)
                if (*it == r) {
                    q->second.erase(it);
                    break;
                }
            if (q->second.empty()) p.posted.erase(q);
        }
    } else if (r->kind == kSend && r->in_outq && !r->started) {
        for (auto it = p.outq.begin(); it != p.outq.end(); ++it)
            if (*it == r) {
                p.outq.erase(it);
                break;
            }
    } else {
        return M4D_OK;  // matched or partly on the wire: no longer retractable
    }
    *cancelled = 1;
    const uint64_t id = r->id;
    t->reqs.erase(id);  // the caller records the cancellation itself
    return M4D_OK;
}

m4d_status m4d_transport_purge_channel(m4d_transport* t, uint32_t channel) {
    for (int q = 0; q < t->world; ++q) {
        if (q == t->rank) continue;
        Peer& p = t->peers[q];
        drain_peer(t, q);
        flush_pulls(t);
        for (auto it = p.unexpected.begin(); it != p.unexpected.end();) {
            if ((it->first >> 32) == channel) {
                for (auto& u : it->second) {
                    if (u->rts) queue_fin(t, q, u->rec.send_id, M4D_ERR_CANCELLED, 0);
                    if (u->eager_dev) dev_release(t, q, u->dev_pos);
                }
                if (p.inbound.active && p.inbound.buf) {
                    for (auto& u : it->second)
                        if (u == p.inbound.buf) p.inbound.buf.reset();
                }
                it = p.unexpected.erase(it);
            } else {
                ++it;
            }
        }
        for (auto it = p.posted.begin(); it != p.posted.end();) {
            if ((it->first >> 32) == channel) {
                for (Req* r : it->second) {
                    fail(M4D_ERR_CANCELLED, "transfer cancelled");
                    complete(t, r, M4D_ERR_CANCELLED, 0);
                }
                it = p.posted.erase(it);
            } else {
                ++it;
            }
        }
        flush_fins(t, p);
    }
    return M4D_OK;
}

m4d_status m4d_transport_wait_ready(m4d_transport* t, double timeout) {
    const double deadline = now_s() + timeout;
    for (;;) {
        int missing = -1;
        for (int q = 0; q < t->world && missing < 0; ++q) {
            if (q == t->rank || t->peers[q].seg) continue;
            int st = try_map_peer(t, q);
            if (st) return st;
            if (!t->peers[q].seg) missing = q;
        }
        if (missing < 0) return M4D_OK;
        if (now_s() > deadline) return fail(M4D_ERR_STARTUP, "rank %d unreachable during startup", missing);
        usleep(500);
    }
}

int m4d_transport_mesh_ready(const m4d_transport* t) {
    for (int q = 0; q < t->world; ++q)
        if (q != t->rank && !t->peers[q].seg) return 0;
    return 1;
}

m4d_status m4d_transport_set_pull_engine(m4d_transport* t, int copy_engine) {
    t->use_ce = copy_engine != 0;
    return M4D_OK;
}

m4d_status m4d_transport_set_pull_ctas(m4d_transport* t, int max_ctas) {
    if (max_ctas < 1) return fail(M4D_ERR_USAGE, "pull grid cap must be positive");
    t->pull_ctas = max_ctas;
    return M4D_OK;
}

int m4d_transport_peer_alive(const m4d_transport* t, int peer) {
    if (peer < 0 || peer >= t->world || peer == t->rank) return 0;
    return t->peers[peer].dead ? 0 : 1;
}

m4d_status m4d_transport_stats_get(const m4d_transport* t, m4d_transport_stats* out) {
    *out = t->stats;
    return M4D_OK;
}

uint64_t m4d_transport_eager_device_max(const m4d_transport* t) {
    return t && t->dev_ring ? eager_device_max() : 0;
}

int m4d_transport_take_loan(m4d_transport* t, uint64_t req_id, uint64_t* ptr, uint64_t* token) {
    auto it = t->loans.find(req_id);
    if (it == t->loans.end()) return 0;
    *ptr = it->second.first;
    *token = it->second.second;
    t->loans.erase(it);
    return 1;
}

m4d_status m4d_transport_release_loan(m4d_transport* t, uint64_t token) {
    if (token & kPoolToken) {
        recv_slot_put(t, reinterpret_cast<uint8_t*>(token & ~kPoolToken));
        return M4D_OK;
    }
    const int peer = static_cast<int>(token >> 48);
    if (peer < 0 || peer >= t->world || peer == t->rank) return fail(M4D_ERR_USAGE, "invalid loan token");
    dev_release(t, peer, token & ((uint64_t(1) << 48) - 1));
    return M4D_OK;
}

m4d_status m4d_transport_close(m4d_transport* t) {
    if (!t) return M4D_OK;
    // Say goodbye through every ring that has room, then mark the segment closed.
    for (int q = 0; q < t->world; ++q) {
        if (q == t->rank || !t->peers[q].seg) continue;
        Peer& p = t->peers[q];
        flush_peer(t, q);
        uint8_t* w = p.out.reserve(sizeof(RecHdr) + 8);
        if (w) {
            RecHdr* h = reinterpret_cast<RecHdr*>(w);
            h->bytes = 16;
            h->kind = kBye;
            h->flags = 0;
            p.out.commit(16);
        }
    }
    if (t->me) t->me->state.store(kStateClosed, std::memory_order_release);
    if (!t->pull_streams.empty()) {
        for (cudaStream_t st : t->pull_streams) cudaStreamSynchronize(st);
        for (auto& q : t->inflight)
            for (Launch& l : q) t->spare_events.push_back(l.ev);
        for (cudaEvent_t e : t->spare_events) cudaEventDestroy(e);
        for (cudaStream_t st : t->pull_streams) cudaStreamDestroy(st);
    }
    if (t->proxy_stream) {  // the kernel idles out (M4D_EAGER_PROXY_IDLE_US) before the rings go
        cudaStreamSynchronize(t->proxy_stream);
        cudaStreamDestroy(t->proxy_stream);
    }
    for (auto& kv : t->ipc_maps) cudaIpcCloseMemHandle(kv.second.base);
    drop_holds(t, -1);
    if (t->eager_stream) {
        cudaStreamSynchronize(t->eager_stream);
        for (EagerCopy& c : t->eager_copies) cudaEventDestroy(c.ev);
        for (auto& kv : t->reqs)
            if (kv.second->dev_ev) cudaEventDestroy(kv.second->dev_ev);
        cudaStreamDestroy(t->eager_stream);
    }
    if (t->dev_ring) cudaFree(t->dev_ring);
    for (void* slab : t->recv_slabs) cudaFree(slab);
    for (auto& kv : t->recv_big) cudaFree(kv.second);
    if (t->pq) cudaFreeHost(t->pq);
    if (t->proxy_state) cudaFree(t->proxy_state);
    if (t->me_registered) cudaHostUnregister(t->me);
    for (Peer& p : t->peers)
        if (p.seg) munmap(p.seg, p.seg_len);
    if (t->me) {
        munmap(t->me, t->me_len);
        shm_unlink(t->seg_name.c_str());
    }
    delete t;
    return M4D_OK;
}

}  // extern "C"
