/*
 * m4d.h — C ABI of libm4d.so, the B200-native data path behind the
 * `commshim` drop-in package (paper_2101_08878_b200).
 *
 * Plain pointers, sizes and integer status codes only: no torch types cross
 * this boundary.  Every function returns an `m4d_status` (0 = success); the
 * message of the most recent failure on the calling thread is available from
 * m4d_last_error().  Status codes map 1:1 onto the reference exception
 * hierarchy (pkg/src/commshim/errors.py:6-89); see M4D_ERR_* below.
 *
 * Sections
 *   1. status codes / library info
 *   2. device helpers (streams, events, memory, IPC export/import)
 *   3. transport (replaces pkg/src/commshim/transport/base.py:199-306
 *      Transport.post_send/post_recv/test/progress/cancel/purge_channel,
 *      selected by transport_init(kind="nvlink"), transport/__init__.py:42-76)
 *   4. transpose_sum kernels
 *   5. key_merge kernels
 *
 * Threading: a context (m4d_ctx) belongs to one executor thread
 * (reference base.py:9-11); the library starts no host threads.
 */
#ifndef M4D_H
#define M4D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* 1. status codes                                                          */
/* ------------------------------------------------------------------------ */

typedef int m4d_status;

enum {
    M4D_OK = 0,
    M4D_ERR_CONFIGURATION = 1,  /* errors.ConfigurationError            */
    M4D_ERR_STARTUP = 2,        /* errors.StartupError(rank)            */
    M4D_ERR_USAGE = 3,          /* errors.UsageError                    */
    M4D_ERR_CHANNEL = 4,        /* errors.ChannelError                  */
    M4D_ERR_COUNT_OVERFLOW = 5, /* errors.CountOverflowError            */
    M4D_ERR_TRANSFER = 6,       /* errors.TransferError(bytes_moved)    */
    M4D_ERR_TRUNCATION = 7,     /* errors.TruncationError               */
    M4D_ERR_CANCELLED = 8,      /* errors.CancelledTransferError        */
    M4D_ERR_PROTOCOL = 9,       /* errors.ProtocolError                 */
    M4D_ERR_CLOSED = 10,        /* errors.CommClosedError               */
    M4D_ERR_BUSY = 11,          /* errors.BusyError                     */
    M4D_ERR_CUDA = 12,          /* CUDA runtime failure (TransferError) */
    M4D_ERR_NOMEM = 13,         /* host allocation failure              */
    M4D_ERR_CAPACITY = 14       /* output buffer too small; retry with the reported size */
};

/* Copies the last failure message of this thread (NUL-terminated). */
size_t m4d_last_error(char* buf, size_t n);
/* Library ABI version: (major << 16) | minor. */
int m4d_version(void);
/* Number of visible CUDA devices (0 on a host without a driver; never fails). */
int m4d_device_count(void);
/* Device that owns device (or managed) memory `ptr`; *device = -1 for host memory. */
m4d_status m4d_pointer_device(const void* ptr, int* device);
/* cudaMemGetInfo of `device` (bytes free / total). */
m4d_status m4d_mem_get_info(int device, uint64_t* free_bytes, uint64_t* total_bytes);

/* ------------------------------------------------------------------------ */
/* 2. device helpers                                                        */
/* ------------------------------------------------------------------------ */

m4d_status m4d_set_device(int device);
m4d_status m4d_stream_create(int device, void** stream_out);  /* non-blocking stream */
m4d_status m4d_stream_destroy(void* stream);
m4d_status m4d_stream_sync(void* stream);
m4d_status m4d_device_sync(int device);
/* Event timing on a given stream (the stream the kernel is launched on). */
m4d_status m4d_event_create(void** ev_out);
m4d_status m4d_event_destroy(void* ev);
m4d_status m4d_event_record(void* ev, void* stream);
m4d_status m4d_event_sync(void* ev);
m4d_status m4d_stream_wait_event(void* stream, void* ev);  /* later work on stream waits for ev */
m4d_status m4d_event_elapsed_ms(void* start, void* stop, float* ms_out);
m4d_status m4d_malloc(int device, size_t nbytes, void** ptr_out);
m4d_status m4d_free(void* ptr);
m4d_status m4d_host_alloc(size_t nbytes, void** ptr_out);   /* pinned */
m4d_status m4d_host_free(void* ptr);
m4d_status m4d_memcpy(void* dst, const void* src, size_t nbytes, void* stream); /* async, any direction */
m4d_status m4d_memset(void* dst, int value, size_t nbytes, void* stream);
/* Legacy CUDA IPC: 64-byte handle of the allocation containing `ptr`;
 * `offset_out` is ptr - allocation base. */
m4d_status m4d_ipc_export(const void* ptr, uint8_t handle_out[64], uint64_t* offset_out);
m4d_status m4d_ipc_import(int device, const uint8_t handle[64], void** base_out);
m4d_status m4d_ipc_close(void* base);
/* Enables peer access between two devices in this process (same-process multi-rank mode). */
m4d_status m4d_enable_peer(int device, int peer_device);

/* ------------------------------------------------------------------------ */
/* 3. transport                                                             */
/* ------------------------------------------------------------------------ */
/* Replaces the reference Transport contract (pkg/src/commshim/transport/
 * base.py:199-306): exact (channel, peer, tag) FIFO matching, non-blocking
 * posts, cooperative progress.  One context per rank; all ranks of a world
 * share `session` and live on one node (shared-memory rings carry control
 * and host payloads, CUDA-IPC rendezvous carries device payloads over
 * NVLink).  Python binding: paper_2101_08878_b200/transport/nvlink.py. */

typedef struct m4d_transport m4d_transport;

typedef struct m4d_transport_config {
    int32_t world;            /* world size (transport_init world_size)            */
    int32_t rank;             /* this rank (transport_init self_rank)              */
    int32_t device;           /* CUDA ordinal, or -1 for a host-only context       */
    int32_t reserved;
    uint64_t ring_bytes;      /* per ordered pair ring, multiple of 4096, >= 64 KiB */
    double connect_timeout;   /* seconds to wait for every peer (StartupError)     */
    const char* session;      /* shared-memory namespace of the world              */
} m4d_transport_config;

/* A finished request.  status: M4D_OK, or the M4D_ERR_* code of the
 * failure (TRUNCATION, CANCELLED, TRANSFER, CLOSED, CUDA); status -1 in an
 * immediate-completion slot means "still pending". */
typedef struct m4d_completion {
    uint64_t req_id;
    int32_t status;
    int32_t kind;             /* 0 send, 1 recv */
    uint64_t bytes;           /* bytes moved (TransferRequest.bytes_moved) */
} m4d_completion;

typedef struct m4d_transport_stats {
    uint64_t sends_completed, recvs_completed, bytes_sent, bytes_received;
    uint64_t eager_bytes;       /* host payload bytes written into rings         */
    uint64_t nvlink_bytes;      /* device payload bytes received peer-to-peer    */
    uint64_t rendezvous_pulls;
    uint64_t unexpected_messages;
    uint64_t pull_kernel_launches; /* SM copy kernels issued for rendezvous pulls  */
    uint64_t eager_device_sends;   /* device payloads sent by the eager protocol    */
    uint64_t eager_device_loans;   /* eager device messages received by loan        */
    uint64_t eager_proxy_copies;   /* eager device sends copied by the proxy kernel */
    uint64_t eager_proxy_launches; /* proxy kernel launches (it exits when idle)     */
} m4d_transport_stats;

/* transport_init: publishes this rank and maps the peers that are already up
 * (the rest are mapped lazily by progress, like the reference socket mesh,
 * tcp.py:173-254).  ConfigurationError for a rank collision or disagreeing
 * settings. */
m4d_status m4d_transport_open(const m4d_transport_config* cfg, m4d_transport** out);
/* SocketTransport.wait_ready (tcp.py:163-171): block until every peer is
 * mapped; StartupError naming the first unreachable rank after `timeout` s. */
m4d_status m4d_transport_wait_ready(m4d_transport* t, double timeout);
int m4d_transport_mesh_ready(const m4d_transport* t);
/* Transport.post_send (base.py:267-269).  `on_device` bit 0: ptr is device
 * memory (rendezvous over NVLink); host payloads are sent eagerly.  Bit 1
 * (device sends only): eager allowed -- a payload of at most
 * m4d_transport_eager_device_max() bytes is copied by the sender into its
 * region of the receiver's device ring and completes once that copy is done,
 * without waiting for the receiver; larger ones, or any that find the ring
 * full, take the rendezvous.  For post_recv, bit 1 lets an eager device message
 * complete the receive by LOAN: no copy, the bytes stay in the ring
 * (m4d_transport_take_loan) until m4d_transport_release_loan.  Bit 2 (device
 * receives): loan only -- ptr may be NULL, `len` is the largest message
 * accepted; a message that arrives by rendezvous is pulled into a transport
 * receive slot that is lent the same way.  When the
 * request finishes inside the call, *now receives its completion (status
 * != -1) and it is not reported again by m4d_transport_progress. */
m4d_status m4d_transport_post_send(m4d_transport* t, uint32_t channel, int peer, uint32_t tag,
                                   const void* ptr, uint64_t len, int domain, int on_device,
                                   uint64_t req_id, m4d_completion* now);
/* Transport.post_recv (base.py:271-273); same conventions. */
m4d_status m4d_transport_post_recv(m4d_transport* t, uint32_t channel, int peer, uint32_t tag,
                                   void* ptr, uint64_t cap, int domain, int on_device,
                                   uint64_t req_id, m4d_completion* now);
/* Vectored post_send / post_recv: `count` posts to one (channel, peer, tag) in
 * one call (osu_bw's window, a frame's chunks), ptrs[i] / lens[i] with id
 * req_ids[i]; now[i] as for a single post.  Stops at the first post that fails
 * and returns its status; *posted = posts made before it. */
m4d_status m4d_transport_post_many(m4d_transport* t, int is_send, uint32_t channel, int peer, uint32_t tag,
                                   void* const* ptrs, const uint64_t* lens, int count, int domain, int on_device,
                                   const uint64_t* req_ids, m4d_completion* now, int* posted);
/* Eager device protocol: its size threshold (0: no device ring), and the loans
 * of receives posted with on_device bit 1: 1 and (*ptr, *token) when receive
 * req_id was completed by a loan of ring bytes at device address *ptr (valid
 * until released, at most until the transport closes), else 0. */
uint64_t m4d_transport_eager_device_max(const m4d_transport* t);
int m4d_transport_take_loan(m4d_transport* t, uint64_t req_id, uint64_t* ptr, uint64_t* token);
m4d_status m4d_transport_release_loan(m4d_transport* t, uint64_t token);
/* Transport.progress (sim.py:144-159, tcp.py:334-344): drains rings, flushes
 * queued sends, polls device copies; writes up to `max` completions and
 * returns how many. */
int m4d_transport_progress(m4d_transport* t, m4d_completion* out, int max);
int m4d_transport_pending_completions(const m4d_transport* t);
/* Transport.cancel: *cancelled = 1 when the request was still unmatched. */
m4d_status m4d_transport_cancel(m4d_transport* t, uint64_t req_id, int* cancelled);
/* Transport.purge_channel (sim.py:171-180): drop unmatched state of a channel id. */
m4d_status m4d_transport_purge_channel(m4d_transport* t, uint32_t channel);
int m4d_transport_peer_alive(const m4d_transport* t, int peer);
/* Cap on the CTAs of one pull-kernel launch (default 296 = 2 per SM, which one
 * in-flight message needs to reach the NVLink peak).  Lower it while pulls run
 * beside compute kernels (the key_merge shuffle uses 64). */
m4d_status m4d_transport_set_pull_ctas(m4d_transport* t, int max_ctas);
/* copy_engine != 0: rendezvous pulls use the copy engines only (no SM
 * kernels), leaving every SM to compute kernels running beside the transfer
 * (the key_merge shuffle: N=2 9.7 -> 8.4 ms per step); 0 restores SM pulls. */
m4d_status m4d_transport_set_pull_engine(m4d_transport* t, int copy_engine);
m4d_status m4d_transport_stats_get(const m4d_transport* t, m4d_transport_stats* out);
m4d_status m4d_transport_close(m4d_transport* t);

/* ------------------------------------------------------------------------ */
/* 4. transpose_sum (K3/K4)                                                 */
/* ------------------------------------------------------------------------ */

/* x[r, c] = (splitmix64(seed ^ (r * n + c)) >> 11) * 2^-53 for the b x b block
 * whose top-left global element is (row0, col0); dst is row-major b*b. */
m4d_status m4d_fill_block_f64(double* dst, int64_t n, int64_t row0, int64_t col0,
                              int64_t b, uint64_t seed, void* stream);

/* One output block y(i,j) = x(i,j) + x(j,i)^T of a chunked square array.
 *   a  : x(i,j), local, row-major b*b
 *   bt : x(j,i), local OR a peer-mapped pointer (read over NVLink, no staging)
 *   y  : y(i,j) output, local
 *   y2 : y(j,i) output when it is also owned here (pairs the two outputs so
 *        x is read once), else NULL.  For a diagonal block (i == j) pass
 *        a == bt, y2 == NULL and diag = 1.
 * slot_y / slot_y2 index the per-block sum array handed to m4d_ts_run. */
typedef struct m4d_ts_task {
    const double* a;
    const double* bt;
    double* y;
    double* y2;
    int32_t slot_y;
    int32_t slot_y2;
    int32_t diag;
    int32_t remote;   /* 0 when bt is local; otherwise a group id (e.g. 1 + the
                         peer's rank) of the GPU bt is read from over NVLink.
                         The plan runs one item stream per group plus the local
                         one concurrently, so every peer is read at once and
                         NVLink and HBM traffic overlap */
} m4d_ts_task;

typedef struct m4d_ts_plan m4d_ts_plan;

m4d_status m4d_ts_plan_create(int device, const m4d_ts_task* tasks, int ntasks,
                              int64_t block, int nslots, m4d_ts_plan** plan_out);
/* Launches the fused transpose-add-reduce kernel (plus a tiny fold launch on
 * the TMA path; see m4d_ts_launches_per_run).  Writes
 * block_sums[nslots] (device, fp64, deterministic fixed-order reduction of
 * each output block) and *total (device, sequential sum of block_sums in slot
 * order; may be NULL). */
m4d_status m4d_ts_run(m4d_ts_plan* plan, double* block_sums, double* total, void* stream);
m4d_status m4d_ts_plan_destroy(m4d_ts_plan* plan);
/* 1 when the plan runs the TMA-fed persistent kernel, 0 for the LDG fallback. */
int m4d_ts_plan_uses_tma(const m4d_ts_plan* plan);
/* Number of kernel launches one m4d_ts_run of this plan issues (gpu_launches accounting). */
int m4d_ts_launches_per_run(const m4d_ts_plan* plan);

/* ------------------------------------------------------------------------ */
/* 5. key_merge (K5 partition, K7 join, K8 digest)                          */
/* ------------------------------------------------------------------------ */

enum {
    M4D_PART_LOCAL = 0,  /* bucket = (h & 0xffffffff) >> (32 - log2 buckets), h = splitmix64(key) */
    M4D_PART_RANK = 1,   /* bucket = owner rank = (uint32(h >> 32) * buckets) >> 32               */
    M4D_PART_OWNER_COARSE = 2  /* bucket = owner rank * C + the top log2 C bits of the LOCAL id
                                  (m4d_partition_owner_coarse only) */
};

/* Largest power of two C with world * C <= 256 (the owner+coarse fan-out). */
int m4d_owner_coarse_count(int world);
/* One pass that both routes rows to their owner rank (as M4D_PART_RANK with
 * `world` buckets) and performs the owner's first local pass: bucket = owner *
 * coarse + the top log2(coarse) bits of the LOCAL partition id (coarse a power
 * of two, world * coarse <= 256).  bounds[] gets world * coarse + 1 entries;
 * scratch as m4d_partition_scratch_bytes(n, world * coarse). */
m4d_status m4d_partition_owner_coarse(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                      int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes,
                                      void* stream);

/* The same owner+coarse partition split in two calls so the shuffle can be
 * fused into the scatter (replaces the shuffle of the reference's merge,
 * "hash-shuffles rows to their owner").
 * m4d_partition_owner_plan: histogram + offsets (kept in `scratch`) and
 * bounds[world * coarse + 1] (device), exactly as m4d_partition_owner_coarse.
 * m4d_partition_owner_push: the scatter of that plan (same keys, vals, n,
 * scratch), writing owner d's rows -- its `coarse` runs back to back, the
 * layout m4d_partition_owner_coarse gives segment d -- to the device address
 * seg_dest[d] (host array of `world` addresses, world <= 64): a peer B200's
 * receive buffer mapped through CUDA IPC, so the rows cross NVLink as the
 * kernel's own stores and no separate exchange step exists. */
m4d_status m4d_partition_owner_plan(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                    int64_t* bounds, void* scratch, size_t scratch_bytes, void* stream);
m4d_status m4d_partition_owner_push(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                    const uint64_t* seg_dest, void* scratch, size_t scratch_bytes, void* stream);

/* Table generator: keys[i] = band + splitmix64(seed + row0 + i) % total,
 * vals[i] = row0 + i (the global row index). */
m4d_status m4d_merge_generate(int64_t* keys, int64_t* vals, int64_t row0, int64_t count,
                              uint64_t total, uint64_t seed, uint64_t band, void* stream);
/* Device scratch m4d_partition needs for n rows and `buckets` buckets. */
size_t m4d_partition_scratch_bytes(int64_t n, int buckets);
/* Hash partition of one table into `buckets` buckets, written bucket-major as
 * 16-byte (key, payload) pairs to out_pairs[2n]; bounds[buckets + 1] (device)
 * receives the bucket start rows.  Input: SoA columns (keys, vals), or pairs
 * (keys = pairs, vals = NULL).  n < 2^32.  The hash shuffle of SPEC.md:425.
 * LOCAL with more than 256 buckets (power of two, <= 65536) runs as two
 * L2-friendly scatter passes; up to 8192 buckets the first pass needs no
 * histogram pass (fixed per-CTA regions, exact on-device fallback when one
 * overflows; M4D_PASS1=hist disables it).  RANK allows up to 16384 buckets. */
m4d_status m4d_partition(const int64_t* keys, const int64_t* vals, int64_t n, int mode, int buckets,
                         int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes,
                         void* stream);
/* Counted receiver split (the push shuffle): each sender counts its rows per
 * (owner, local partition) -- out_counts[world][buckets] (32-bit), buckets a power
 * of two, world * buckets * 2 <= m4d_fine_count_smem_limit() -- and hands owner d
 * its row d; the owner's m4d_partition_runs_counted then splits the received
 * runs with those counts (fine_in[sources][buckets]) instead of counting them
 * again.  Same output as m4d_partition_runs. */
size_t m4d_fine_count_smem_limit(void);
m4d_status m4d_partition_fine_counts(const int64_t* keys, const int64_t* vals, int64_t n, int world, int buckets,
                                     uint32_t* out_counts, void* stream);
/* The push scatter (m4d_partition_owner_push) counting its rows per (owner,
 * local partition) in the same pass: out_counts[world][parts] (32-bit, zeroed
 * by the call; the buffer holds world * parts + 1 words, the last one the
 * kernel's completion counter) is what m4d_partition_fine_counts returns,
 * without another read of the keys; count_dest (may be NULL): for each owner d
 * the address (e.g. in its IPC-mapped receive buffer) that receives row d,
 * written by the kernel's last CTA.  parts a power of two, world * parts * 2 <=
 * m4d_push_fine_smem_limit(); run tables as for m4d_partition_owner_push. */
size_t m4d_push_fine_smem_limit(void);
m4d_status m4d_partition_owner_push_fine(const int64_t* keys, const int64_t* vals, int64_t n, int world, int coarse,
                                         const uint64_t* seg_dest, int parts, uint32_t* out_counts,
                                         const uint64_t* count_dest, void* scratch, size_t scratch_bytes,
                                         void* stream);
m4d_status m4d_partition_runs_counted(const int64_t* in_pairs, int64_t n, const int64_t* runs_host, int coarse,
                                      int sources, int buckets, const uint32_t* fine_in, int64_t* out_pairs,
                                      int64_t* bounds, void* scratch, size_t scratch_bytes, void* stream);
/* Receiver side of an M4D_PART_OWNER_COARSE exchange: in_pairs holds `sources`
 * segments, each made of `coarse` runs in coarse-bucket order; runs_host (host
 * memory, int64[coarse][sources][2]) gives each run's [start, end) row in
 * in_pairs.  Writes the rows split into `buckets` LOCAL partitions (power of
 * two <= 32768, coarse dividing it) to out_pairs and bounds[buckets + 1]
 * (device); within a partition rows keep source order.  Launches 4
 * kernels. */
m4d_status m4d_partition_runs(const int64_t* in_pairs, int64_t n, const int64_t* runs_host, int coarse, int sources,
                              int buckets, int64_t* out_pairs, int64_t* bounds, void* scratch, size_t scratch_bytes,
                              void* stream);
size_t m4d_partition_runs_scratch_bytes(int sources, int buckets, int coarse);
/* Target rows per local partition for the hash join's shared-memory tables (the
 * harness sizes its partition count from it). */
int m4d_join_partition_rows(void);
/* Kernel launches (plus memsets) one m4d_partition call issues for that bucket count. */
int m4d_partition_launches(int buckets);
/* Inner join of partitioned build (left) and probe (right) pair arrays,
 * partition by partition (bounds from m4d_partition, same bucket count).  Writes at most
 * `capacity` rows (key, lval, rval) and result[4] (device) =
 * {rows produced, rows, sum of row hashes, sum of keys} (mod 2^64); a row
 * count above `capacity` means the output was cut: retry with a larger
 * buffer. */
m4d_status m4d_hash_join(const int64_t* lpairs, const int64_t* lbounds, const int64_t* rpairs,
                         const int64_t* rbounds, int parts, int64_t* out_keys, int64_t* out_lvals,
                         int64_t* out_rvals, int64_t capacity, unsigned long long* result, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* M4D_H */
