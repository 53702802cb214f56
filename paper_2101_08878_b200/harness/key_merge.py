"""``key_merge``: inner merge of two int64-key dataframes across B200s.

Operator definition: SPEC.md:422-430 (each worker generates its partitions of
the left and right tables with a match-fraction overlap band, hash-shuffles
rows to their owner, joins locally, reports the global row count), PAPER.md
:387-389 and :438 (cuDF merge, chunk 1e8, ``Shuffle: True``, fraction 0.3).

Generator: ``total`` rows per side over all workers (weak
scaling: ``rows_per_rank * world``), worker ``r`` owns global rows
``[r*n, (r+1)*n)``; left key = ``splitmix64(seed_l + g) % total``, right key
= ``floor((1-f)*total) + splitmix64(seed_r + g) % total``; payload = ``g``.

B200 pipeline per rank (one CUDA stream, SoA device columns):

1. world > 1, shuffle ``push`` (default): one owner+coarse pass plans both
   sides (histogram, offsets), the run tables are all-gathered as eager host
   messages, and the scatter kernel itself writes every owner's rows into
   that owner's receive buffer (CUDA-IPC mapped, so peer rows cross NVLink as
   the kernel's stores: partitioning and shuffle are one kernel,
   ``m4d_partition_owner_push``); a one-byte "side written" exchange then
   lets each owner split what it received.  Shuffle ``pull``
   (``M4D_MERGE_SHUFFLE=pull``, also the fallback when a receive buffer is
   too small): the owner pass writes a local send buffer and every owner
   pulls its segments over NVLink as device-frame rendezvous messages of the
   transport, the two sides pipelined;
2. hash-partition the rows this rank owns into ``parts`` local partitions
   of ~1.5K rows (mode LOCAL), small enough for a shared-memory hash table;
3. ``m4d_hash_join``: one CTA per partition builds and probes, writes the
   (key, lval, rval) rows and an order-independent digest (count, sum of
   row hashes, sum of keys, mod 2^64).

The global result is the digest summed over ranks: identical for every
worker count, and equal to the oracle's (tests/test_key_merge_gpu.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import struct

from .. import native
from ..errors import CommShimError, UsageError
from ..messaging import await_request
from .collectives import allgather
from ..transport import MemoryDomain

SEED_LEFT = 0x4C454654
SEED_RIGHT = 0x52494748
EXCHANGE_TAG = 900
DATA_TAG = 910
_SHUFFLE = os.environ.get("M4D_MERGE_SHUFFLE", "push")
_MASK64 = (1 << 64) - 1


def merge_band(total: int, fraction: float) -> int:
    """floor((1 - f) * total) in IEEE double (the overlap band start)."""
    return int(math.floor((1.0 - fraction) * float(total)))


def choose_parts(rows: int) -> int:
    """Power-of-two partition count with about m4d_join_partition_rows() rows per
    partition (~12K: one 1024-thread join CTA per SM with a 16384-head table), at most
    65536."""
    per = native.lib().m4d_join_partition_rows()
    parts = 1
    while parts < 65536 and rows / parts > per:
        parts *= 2
    return parts


class _Columns:
    """keys + vals device columns of one table (capacity rows): the user-facing SoA layout."""

    def __init__(self, device: int, capacity: int):
        self.capacity = max(1, int(capacity))
        self.keys = native.DeviceBuffer(device, self.capacity * 8)
        self.vals = native.DeviceBuffer(device, self.capacity * 8)


class _Pairs:
    """(key, payload) 16-byte pairs: the internal layout of partitioned / shuffled rows."""

    def __init__(self, device: int, capacity: int, extra_bytes: int = 0):
        self.capacity = max(1, int(capacity))
        self.buf = native.DeviceBuffer(device, self.capacity * 16 + extra_bytes)  # extra: after the rows
        self.ptr = self.buf.ptr


class _RawBytes:
    """``__cuda_array_interface__`` of a raw device byte range (a torch view, no copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _torch_bytes(ptr: int, nbytes: int, device: int):
    import torch

    return torch.as_tensor(_RawBytes(ptr, nbytes), device=torch.device("cuda", device))


class KeyMerge:
    """One rank's share of a distributed inner merge on an int64 key."""

    def __init__(self, rows_per_rank: int, fraction: float = 0.3, *, rank: int = 0, world: int = 1,
                 device: int = 0, transport=None, seed_l: int = SEED_LEFT, seed_r: int = SEED_RIGHT,
                 parts: int | None = None, stream: native.Stream | None = None, shuffle: str | None = None):
        if rows_per_rank < 0 or not 0.0 <= fraction <= 1.0:
            raise UsageError("rows per rank must be >= 0 and fraction in [0, 1]")
        if world > 1 and transport is None:
            raise UsageError("a multi-worker key_merge needs a transport")
        self.n = int(rows_per_rank)
        self.fraction = fraction
        self.rank, self.world, self.device = rank, world, device
        self.transport = transport
        self.total = self.n * world
        self.band = merge_band(self.total, fraction) if self.total else 0
        self.seeds = (seed_l, seed_r)
        native.set_device(device)
        self.stream = stream or native.Stream(device)
        self.parts = parts or choose_parts(self.n)
        slack = self.n + int(6 * math.sqrt(max(self.n, 1))) + 4096
        self.inputs = [_Columns(device, self.n), _Columns(device, self.n)]
        self.sendbuf = [_Pairs(device, self.n), _Pairs(device, self.n)] if world > 1 else None
        # M4D_MERGE_FINE=1 (default, push shuffle): senders count side 1's rows per (owner,
        # partition) beside push 0 and hand each owner its counts after its rows in the
        # receive buffer, so side 1's receiver split needs no histogram pass
        lib = native.lib()
        self.fine = (world > 1 and (shuffle or _SHUFFLE) == "push" and os.environ.get("M4D_MERGE_FINE", "1") != "0"
                     and self.parts > 1 and world * self.parts * 2 <= lib.m4d_fine_count_smem_limit())
        # M4D_MERGE_FINE_FUSED (default: where the 16-bit counters take <= 32 KB, P = 2 at 8192
        # partitions): the push scatter itself counts both sides' rows per (owner, partition)
        # -- no separate count pass, and both receiver splits are counted.  N=2 6.05 -> 5.84 ms;
        # at N=4 the push CTAs' count flush (4 x 8192 global adds each) ate the gain (7.22-7.28
        # vs 7.17-7.23 ms, profiles/r2_push_fine.txt), so =1 forces it wherever the counters fit.
        fused = os.environ.get("M4D_MERGE_FINE_FUSED", "")
        limit = lib.m4d_push_fine_smem_limit() if fused == "1" else min(lib.m4d_push_fine_smem_limit(), 32768)
        self.fine_fused = self.fine and fused != "0" and world * self.parts * 2 <= limit
        fine_bytes = world * self.parts * 4 if self.fine else 0
        # bytes after each receive buffer's rows: the senders' counts (kept when a buffer grows)
        self._recv_extra = [fine_bytes if self.fine_fused else 0, fine_bytes]
        self.recv = [_Pairs(device, slack, self._recv_extra[0]), _Pairs(device, slack, self._recv_extra[1])] if world > 1 else None
        if self.fine:
            self.fine_out = native.DeviceBuffer(device, fine_bytes + 256)  # + the push's completion counter
            self.fine_done = native.Event()
        self.parted = [_Pairs(device, slack), _Pairs(device, slack)]
        self.bounds = [native.DeviceBuffer(device, (max(self.parts, world) + 1) * 8) for _ in range(2)]
        lib = native.lib()
        # owner + coarse buckets of the sender pass (SoA input -> P * C runs; C | parts)
        self.coarse = min(lib.m4d_owner_coarse_count(world), self.parts) if world > 1 else 1
        self.rank_bounds = [native.DeviceBuffer(device, (world * self.coarse + 1) * 8) for _ in range(2)]
        scratch = max(lib.m4d_partition_scratch_bytes(slack, self.parts),
                      lib.m4d_partition_scratch_bytes(self.n, max(world, 1) * self.coarse),
                      lib.m4d_partition_runs_scratch_bytes(max(world, 1), self.parts, self.coarse))
        self.scratch = native.DeviceBuffer(device, scratch)
        self.scratch_bytes = scratch
        # side 1's receiver split may run beside side 0's: its own (small) scratch
        runs_bytes = lib.m4d_partition_runs_scratch_bytes(max(world, 1), self.parts, self.coarse) if world > 1 else 0
        self.split_scratch1 = (native.DeviceBuffer(device, max(1, runs_bytes)), runs_bytes) if world > 1 else None
        self.shuffle = (shuffle or _SHUFFLE) if world > 1 else "local"
        if self.shuffle not in ("push", "pull", "nccl", "local"):
            raise UsageError(f"unknown shuffle {self.shuffle!r} (push | pull | nccl)")
        if self.shuffle == "nccl":
            # owner pass per side on its own stream, NCCL all-to-all (torch.distributed, the
            # default NCCL group) enqueued on that stream, receiver split on a split stream
            self.nccl_streams = [self.stream, native.Stream(device)]
            self.nccl_scratch1 = native.DeviceBuffer(device, scratch)
            self.a2a_done = [native.Event(), native.Event()]
            self.split_streams = [native.Stream(device), native.Stream(device)]
            self.split_done = [native.Event(), native.Event()]
        if self.shuffle == "push":  # per-side plan scratch (both plans live until their push)
            # Coarse runs per owner of the push scatter (M4D_PUSH_BUCKETS = owners x runs,
            # default 256).  Fewer make each tile's run per bucket longer, so NVLink
            # stores are more efficient (tools/probes/write_probe.cu: 8-row runs 395
            # GB/s, 64-row runs 638 GB/s), but the receiver's split fans out wider;
            # measured N=2 / N=4: 64 -> 8.10 / 9.68 ms, 128 -> 7.81 / 9.40, 256 -> 7.72 / 9.29.
            target = int(os.environ.get("M4D_PUSH_BUCKETS", "256"))
            c = 1
            while world * c * 2 <= target and c * 2 <= self.coarse:
                c *= 2
            self.coarse_push = c
            nb = lib.m4d_partition_scratch_bytes(self.n, world * self.coarse)
            self.push_scratch = [native.DeviceBuffer(device, nb) for _ in range(2)]
            self.push_scratch_bytes = nb
            self.pushed = [native.Event(), native.Event()]
            self.plan_stream = native.Stream(device)
            # M4D_MERGE_OVERLAP=1 (default): the receiver splits run on a second stream, so
            # side 0's split (HBM-bound) overlaps side 1's push (NVLink-bound)
            self.overlap = os.environ.get("M4D_MERGE_OVERLAP", "1") != "0"
            # one split stream per side: side 1's split may start while side 0's finishes
            self.split_streams = ([native.Stream(device), native.Stream(device)] if self.overlap
                                  else [self.stream, self.stream])
            self.split_stream = self.split_streams[0]
            self.split_done = [native.Event(), native.Event()]
        # world == 1: side 1 partitions on its own stream (M4D_MERGE_SIDES=serial: one stream)
        self.side_stream = self.side_scratch = None
        if world == 1 and os.environ.get("M4D_MERGE_SIDES", "concurrent") != "serial":
            self.side_stream = native.Stream(device)
            self.side_scratch = native.DeviceBuffer(device, scratch)
            self.side_ready, self.side_done = native.Event(), native.Event()
        self._peer_recv: list[list[int]] | None = None  # [side][rank] receive-buffer address (mapped)
        self._imported: list[int] = []
        self.out_capacity = int(fraction * self.n * 1.25) + 65536
        self.out = [native.DeviceBuffer(device, self.out_capacity * 8) for _ in range(3)]
        self.result = native.DeviceBuffer(device, 4 * 8)
        self.received = [0, 0]
        self.launches = 0
        self.profile = False  # diagnostics: synchronise and stamp each phase (never in timed runs)
        self.tracing = False  # diagnostics: CUDA-event trace points without synchronisation
        self._trace_points: list = []
        self.trace: dict[str, float] = {}
        # CUDA-event kernel timing inside timed runs (no synchronisation added): partition
        # kernels (local or plan + push) and the join, summed over steps in kernel_ms
        self.timing = False
        self.kernel_ms = {"partition": 0.0, "join": 0.0}
        self._ev = [native.Event() for _ in range(4)]
        self.phases: dict[str, float] = {}

    # -- data -------------------------------------------------------------------------------

    def generate(self) -> None:
        native.set_device(self.device)  # (several ranks may share a process: tests, profiling)
        lib = native.lib()
        row0 = self.rank * self.n
        for side, (cols, seed, band) in enumerate(zip(self.inputs, self.seeds, (0, self.band))):
            if self.n:
                native.check(lib.m4d_merge_generate(cols.keys.ptr, cols.vals.ptr, row0, self.n, self.total, seed,
                                                    band, self.stream.handle))
        self.stream.synchronize()

    # -- pipeline ---------------------------------------------------------------------------

    def _partition(self, src, n: int, mode: int, buckets: int, dst: _Pairs, bounds, stream=None,
                   scratch=None) -> None:
        keys, vals = (src.keys.ptr, src.vals.ptr) if isinstance(src, _Columns) else (src.ptr, None)
        native.set_device(self.device)  # ranks of one process may sit on different GPUs
        native.check(native.lib().m4d_partition(keys, vals, n, mode, buckets, dst.ptr, bounds.ptr,
                                                (scratch or self.scratch).ptr, self.scratch_bytes,
                                                (stream or self.stream).handle))
        self.launches += native.lib().m4d_partition_launches(buckets)

    def _tp(self, name: str, stream=None) -> None:
        """Trace point (diagnostics, ``self.tracing``): a CUDA event on `stream`; after the
        step, ``self.trace`` maps each name to its time in ms since the step began.
        Unlike ``profile`` this adds no synchronisation, so overlap stays visible."""
        if self.tracing:
            ev = native.Event()
            ev.record(stream or self.stream)
            self._trace_points.append((name, ev))

    def _mark(self, name: str) -> None:
        if self.profile:
            import time

            self.stream.synchronize()
            for st in getattr(self, "split_streams", []):
                st.synchronize()
            now = time.perf_counter()
            self.phases[name] = (now - self._t_last) * 1e3
            self._t_last = now

    def _read_bounds(self, buf, count: int, stream=None) -> list[int]:
        raw = native.to_host(buf.ptr, (count + 1) * 8, stream or self.stream)
        return list(struct.unpack(f"<{count + 1}q", raw))

    def _owner_split(self, side: int) -> list[int]:
        """One pass over one side's columns: rows grouped by (owner rank, top bits of their
        local partition), i.e. routed to their owner and already through the owner's first
        local pass.  Returns the P * C + 1 bucket bounds (synchronises)."""
        P, C = self.world, self.coarse
        native.set_device(self.device)  # ranks of one process may sit on different GPUs
        native.check(native.lib().m4d_partition_owner_coarse(
            self.inputs[side].keys.ptr, self.inputs[side].vals.ptr, self.n, P, C, self.sendbuf[side].ptr,
            self.rank_bounds[side].ptr, self.scratch.ptr, self.scratch_bytes, self.stream.handle))
        self.launches += native.lib().m4d_partition_launches(P * C)
        return self._read_bounds(self.rank_bounds[side], P * C)

    def _post_side(self, side: int, sends: list[int], incoming: list[int]) -> list:
        """Post one side's exchange: pulls of every peer's segment (device frames over NVLink)
        into the source-major receive buffer, and this rank's segments for the peers."""
        from ..transport.base import DeviceView

        t, P, me = self.transport, self.world, self.rank
        total = sum(incoming)
        if total > self.recv[side].capacity:
            self.recv[side] = _Pairs(self.device, int(total * 1.1) + 4096, self._recv_extra[side])
        if total > self.parted[side].capacity:
            self.parted[side] = _Pairs(self.device, int(total * 1.1) + 4096)
        reqs, at = [], 0
        for src in range(P):  # receive layout: source-major, each source's rows contiguous
            rows = incoming[src]
            dst = self.recv[side].ptr + at * 16
            if src == me:
                native.memcpy(dst, self.sendbuf[side].ptr + sends[me] * 16, rows * 16, self.stream)
            elif rows:
                reqs.append(t.post_recv(0, src, DATA_TAG + side, DeviceView(dst, rows * 16, self.device),
                                        MemoryDomain.DEVICE))
            at += rows
        for dst_rank in range(P):
            rows = sends[dst_rank + 1] - sends[dst_rank]
            if dst_rank != me and rows:
                view = DeviceView(self.sendbuf[side].ptr + sends[dst_rank] * 16, rows * 16, self.device)
                reqs.append(t.post_send(0, dst_rank, DATA_TAG + side, view, MemoryDomain.DEVICE))
        t.progress()  # match what already arrived: the pulls start now, on the transport's streams
        return reqs

    async def _exchange_side(self, side: int):
        """Owner pass, run-table exchange and posting of one side's transfers."""
        t, P, me, C = self.transport, self.world, self.rank, self.coarse
        b = self._owner_split(side)  # synchronises: the send buffer is complete before peers pull
        rel = [b[d * C + c] - b[d * C] for d in range(P) for c in range(C + 1)]
        table = [struct.unpack(f"<{P * (C + 1)}q", blob)
                 for blob in await allgather(t, struct.pack(f"<{P * (C + 1)}q", *rel), EXCHANGE_TAG + 2 + side)]
        runs_in = [table[src][me * (C + 1):(me + 1) * (C + 1)] for src in range(P)]  # my runs in each source
        incoming = [r[C] for r in runs_in]
        sends = [b[d * C] for d in range(P)] + [b[P * C]]
        return self._post_side(side, sends, incoming), runs_in

    def _finish_side(self, side: int, runs_in: list, coarse: int | None = None, stream=None,
                     counted: bool = False) -> int:
        """Split the received source segments (each C coarse runs) into the local partitions.
        ``counted``: the senders' per-partition counts follow the rows in the receive
        buffer (push shuffle, side 1), so no histogram pass over the rows."""
        P, C = self.world, coarse or self.coarse
        runs, total = runs_in if isinstance(runs_in, tuple) else self._runs_table(runs_in, C)
        native.set_device(self.device)  # ranks of one process may sit on different GPUs
        scratch, nbytes = (self.scratch, self.scratch_bytes) if side == 0 else self.split_scratch1
        if counted:  # the senders' counts, after the rows
            fine_in = self.recv[side].ptr + self.recv[side].capacity * 16
            native.check(native.lib().m4d_partition_runs_counted(
                self.recv[side].ptr, total, runs.ctypes.data, C, P, self.parts, fine_in, self.parted[side].ptr,
                self.bounds[side].ptr, scratch.ptr, nbytes, (stream or self.stream).handle))
            self.launches += 3
            return total
        native.check(native.lib().m4d_partition_runs(self.recv[side].ptr, total, runs.ctypes.data, C, P, self.parts,
                                                     self.parted[side].ptr, self.bounds[side].ptr, scratch.ptr,
                                                     nbytes, (stream or self.stream).handle))
        self.launches += 4
        return total

    def _runs_table(self, runs_in: list, C: int):
        """(C x P x 2 run bounds, total rows) of the received source segments: source src's
        coarse run c is rows [start_src + r[c], start_src + r[c + 1]) of the receive buffer."""
        import numpy as np

        r = np.asarray(runs_in, dtype=np.int64)  # [P][C + 1], relative to each source's segment
        starts = np.concatenate(([0], np.cumsum(r[:, C])))[:-1]
        runs = np.empty((C, self.world, 2), dtype=np.int64)
        runs[:, :, 0] = (starts[:, None] + r[:, :C]).T
        runs[:, :, 1] = (starts[:, None] + r[:, 1:]).T
        return np.ascontiguousarray(runs), int(r[:, C].sum())

    async def _shuffle_and_partition(self) -> list[int]:
        """Owner pass, NVLink exchange and local partition of both sides, pipelined: side 1's
        owner pass runs while side 0's rows are pulled, and side 0's local partition while
        side 1's rows are pulled."""
        t = self.transport
        engine = getattr(t, "pull_copy_engine", None)
        if engine is not None:
            t.set_pull_engine(True)  # copy-engine pulls: every SM stays on the partition kernels
        reqs0, runs0 = await self._exchange_side(0)
        reqs1, runs1 = await self._exchange_side(1)
        self._mark("owner_partition_and_post_ms")
        for r in reqs0:
            await await_request(t, r)
        self._mark("side0_exchange_wait_ms")
        n0 = self._finish_side(0, runs0)
        for r in reqs1:
            await await_request(t, r)
        self._mark("side1_exchange_wait_ms")
        n1 = self._finish_side(1, runs1)
        if engine is not None:
            t.set_pull_engine(engine)
        return [n0, n1]

    async def _connect_push(self) -> None:
        """Swap CUDA-IPC handles of both receive buffers (once): every rank's scatter
        kernel then writes straight into its peers' buffers."""
        me = self.rank
        blob = b""
        for side in range(2):
            handle, off = native.ipc_export(self.recv[side].ptr)
            blob += struct.pack("<iQQQ", os.getpid(), self.recv[side].ptr, off, self.recv[side].capacity) + handle
        peer = [[0] * self.world for _ in range(2)]
        self._peer_cap = [[0] * self.world for _ in range(2)]
        size = struct.calcsize("<iQQQ") + 64
        for src, item in enumerate(await allgather(self.transport, blob, EXCHANGE_TAG + 4)):
            for side in range(2):
                rec = item[side * size:(side + 1) * size]
                pid, ptr, off, cap = struct.unpack_from("<iQQQ", rec)
                self._peer_cap[side][src] = cap
                if src == me or pid == os.getpid():  # same process (multi-rank tests): plain pointer
                    peer[side][src] = ptr
                else:
                    base = native.ipc_import(self.device, rec[28:92])
                    self._imported.append(base)
                    peer[side][src] = base + off
        self._peer_recv = peer

    async def _push_shuffle_and_partition(self) -> list[int] | None:
        """Fused owner scatter + NVLink shuffle of both sides (``m4d_partition_owner_push``),
        then the local split of what arrived.  None: a receive buffer is too small for this
        step's rows (every rank sees the same run tables and falls back together)."""
        t, P, me, C, lib = self.transport, self.world, self.rank, self.coarse_push, native.lib()
        if self._peer_recv is None:
            await self._connect_push()
        # Side 0's plan runs alone, so its push starts as early as possible; side 1's plan
        # runs on the plan stream beside that push (the push leaves SMs free, M4D_PUSH_SMS),
        # and its run tables are exchanged while side 0's rows move.
        plan_streams = [self.stream, self.plan_stream]
        width = P * (C + 1)
        runs_in = [None, None]
        for side in range(2):
            native.set_device(self.device)  # ranks of one process may sit on different GPUs
            native.check(lib.m4d_partition_owner_plan(
                self.inputs[side].keys.ptr, self.inputs[side].vals.ptr, self.n, P, C, self.rank_bounds[side].ptr,
                self.push_scratch[side].ptr, self.push_scratch_bytes, plan_streams[side].handle))
            self.launches += 5
            b = self._read_bounds(self.rank_bounds[side], P * C, plan_streams[side])
            self._tp(f"plan{side}_done", plan_streams[side])
            if side == 1 and self.fine and not self.fine_fused:
                # my side-1 rows per (owner, partition), into each owner's receive buffer after
                # its rows (queued after the plan's read-back, so the run-table exchange below
                # does not wait for it; it runs beside push 0)
                parts, stream = self.parts, plan_streams[1]
                native.check(lib.m4d_partition_fine_counts(self.inputs[1].keys.ptr, self.inputs[1].vals.ptr, self.n, P,
                                                           parts, self.fine_out.ptr, stream.handle))
                for d in range(P):
                    dst = self._peer_recv[1][d] + self._peer_cap[1][d] * 16 + me * parts * 4
                    native.memcpy(dst, self.fine_out.ptr + d * parts * 4, parts * 4, stream)
                self.fine_done.record(stream)
                self.launches += 1
            # my rows per (owner, coarse run), relative to each owner's segment
            blob = struct.pack(f"<{width}q", *[b[d * C + c] - b[d * C] for d in range(P) for c in range(C + 1)])
            tables = [struct.unpack(f"<{width}q", x) for x in await allgather(t, blob, EXCHANGE_TAG + 2 + 7 * side)]
            runs_in[side] = self._runs_table([tables[src][me * (C + 1):(me + 1) * (C + 1)] for src in range(P)], C)
            if any(sum(tables[src][d * (C + 1) + C] for src in range(P)) > self._peer_cap[side][d] for d in range(P)):
                # a receive buffer is too small: every rank sees the same tables and falls back
                # together, once side 0's pushes (if any) have landed everywhere
                if side == 1:
                    self.pushed[0].synchronize()
                    await allgather(t, b"\x00", EXCHANGE_TAG + 10)
                return None
            dest = (ctypes.c_uint64 * P)()
            for d in range(P):  # my segment in owner d's buffer: after the rows of lower sources
                before = sum(tables[src][d * (C + 1) + C] for src in range(me))
                dest[d] = self._peer_recv[side][d] + before * 16
            self._tp(f"push{side}_start")
            native.set_device(self.device)
            if self.fine_fused:  # the push counts my rows per (owner, partition) as it moves them
                parts = self.parts
                # owner d's row of counts goes after the rows of its receive buffer (written by
                # the kernel's last CTA)
                cdst = (ctypes.c_uint64 * P)(*[self._peer_recv[side][d] + self._peer_cap[side][d] * 16 + me * parts * 4
                                               for d in range(P)])
                native.check(lib.m4d_partition_owner_push_fine(
                    self.inputs[side].keys.ptr, self.inputs[side].vals.ptr, self.n, P, C, dest, parts,
                    self.fine_out.ptr, cdst, self.push_scratch[side].ptr, self.push_scratch_bytes, self.stream.handle))
            else:
                native.check(lib.m4d_partition_owner_push(
                    self.inputs[side].keys.ptr, self.inputs[side].vals.ptr, self.n, P, C, dest,
                    self.push_scratch[side].ptr, self.push_scratch_bytes, self.stream.handle))
            self.pushed[side].record(self.stream)
            self._tp(f"push{side}_end")
        self._mark("owner_plan_push_ms")
        self.launches += 2
        out = []
        for side in range(2):
            self.pushed[side].synchronize()  # my rows for side `side` are in every owner's buffer
            if side == 1 and self.fine and not self.fine_fused:
                self.fine_done.synchronize()  # ... and so are my side-1 counts
            await allgather(t, b"\x01", EXCHANGE_TAG + 6 + side)  # ... and every peer's rows in mine
            self._mark(f"side{side}_push_ms")
            self._tp(f"split{side}_start", self.split_streams[side])
            out.append(self._finish_side(side, runs_in[side], C, self.split_streams[side],
                                         counted=self.fine_fused or (side == 1 and self.fine)))
            self._tp(f"split{side}_end", self.split_streams[side])
        for side in range(2):  # the join waits for both splits
            if self.split_streams[side] is not self.stream:
                self.split_done[side].record(self.split_streams[side])
                self.split_done[side].wait_on(self.stream)
        return out

    async def _nccl_shuffle_and_partition(self) -> list[int]:
        """Owner pass of each side into a local send buffer, then one NCCL all-to-all per
        side (NVLink, ``torch.distributed.all_to_all_single`` on the raw buffers) enqueued
        on that side's stream -- side 1's owner pass runs while side 0's bytes move --
        and the receiver split of each side once its all-to-all is done.  The rows land
        source-major, as in the pull shuffle."""
        import numpy as np
        import torch
        import torch.distributed as dist

        t, P, me, C, lib = self.transport, self.world, self.rank, self.coarse, native.lib()
        out = []
        runs = []
        for side in range(2):
            st = self.nccl_streams[side]
            scratch = self.scratch if side == 0 else self.nccl_scratch1
            native.set_device(self.device)  # ranks of one process may sit on different GPUs
            native.check(lib.m4d_partition_owner_coarse(
                self.inputs[side].keys.ptr, self.inputs[side].vals.ptr, self.n, P, C, self.sendbuf[side].ptr,
                self.rank_bounds[side].ptr, scratch.ptr, self.scratch_bytes, st.handle))
            self.launches += lib.m4d_partition_launches(P * C)
            b = self._read_bounds(self.rank_bounds[side], P * C, st)  # the send buffer is complete
            self._tp(f"owner{side}_done", st)
            rel = [b[d * C + c] - b[d * C] for d in range(P) for c in range(C + 1)]
            table = [struct.unpack(f"<{P * (C + 1)}q", blob) for blob in
                     await allgather(t, struct.pack(f"<{P * (C + 1)}q", *rel), EXCHANGE_TAG + 2 + side)]
            runs_in = [table[src][me * (C + 1):(me + 1) * (C + 1)] for src in range(P)]
            incoming = [r[C] for r in runs_in]
            total = sum(incoming)
            if total > self.recv[side].capacity:
                self.recv[side] = _Pairs(self.device, int(total * 1.1) + 4096, self._recv_extra[side])
            if total > self.parted[side].capacity:
                self.parted[side] = _Pairs(self.device, int(total * 1.1) + 4096)
            send_t = _torch_bytes(self.sendbuf[side].ptr, max(1, b[P * C] * 16), self.device)
            recv_t = _torch_bytes(self.recv[side].ptr, max(1, total * 16), self.device)
            with torch.cuda.stream(torch.cuda.ExternalStream(st.handle, device=torch.device("cuda", self.device))):
                dist.all_to_all_single(recv_t, send_t, [r * 16 for r in incoming],
                                       [(b[(d + 1) * C] - b[d * C]) * 16 for d in range(P)])
            self.a2a_done[side].record(st)
            self._tp(f"a2a{side}_end", st)
            runs.append(runs_in)
        for side in range(2):
            self.a2a_done[side].wait_on(self.split_streams[side])
            self._tp(f"split{side}_start", self.split_streams[side])
            out.append(self._finish_side(side, runs[side], C, self.split_streams[side]))
            self._tp(f"split{side}_end", self.split_streams[side])
            self.split_done[side].record(self.split_streams[side])
            self.split_done[side].wait_on(self.stream)
        return out

    def close(self) -> None:
        """Unmap the peers' receive buffers (push shuffle)."""
        for base in self._imported:
            native.ipc_close(base)
        self._imported = []
        self._peer_recv = None

    async def run(self) -> tuple[int, int, int]:
        """One full step (partition [+ shuffle] + join).  Returns this rank's digest."""
        native.set_device(self.device)
        if self.profile:
            import time

            self.stream.synchronize()
            self._t_last = time.perf_counter()
            self.phases = {}
        if self.timing:
            self._ev[0].record(self.stream)
        self._trace_points = []
        self._tp("step_start")
        if self.world > 1:
            if self.shuffle == "nccl":
                got = await self._nccl_shuffle_and_partition()
            else:
                got = await self._push_shuffle_and_partition() if self.shuffle == "push" else None
                if got is None and self.shuffle == "push":
                    self.close()  # the pull path may grow the receive buffers: map them again next step
            self.received = got if got is not None else await self._shuffle_and_partition()
        else:
            # The two sides partition concurrently on two streams: each pass is
            # latency-bound with one or two CTAs per SM, so CTAs of the other side's
            # kernels fill the rest of the SM.
            self.received = [self.n, self.n]
            if self.side_stream is not None:
                self.side_ready.record(self.stream)
                self.side_ready.wait_on(self.side_stream)
            self._partition(self.inputs[0], self.n, 0, self.parts, self.parted[0], self.bounds[0])
            self._partition(self.inputs[1], self.n, 0, self.parts, self.parted[1], self.bounds[1],
                            self.side_stream, self.side_scratch)
            if self.side_stream is not None:
                self.side_done.record(self.side_stream)
                self.side_done.wait_on(self.stream)
        self._mark("local_partition_ms")
        if self.timing:
            self._ev[1].record(self.stream)
        self._tp("join_start")
        while True:
            native.set_device(self.device)  # ranks of one process may sit on different GPUs
            native.check(native.lib().m4d_hash_join(
                self.parted[0].ptr, self.bounds[0].ptr, self.parted[1].ptr, self.bounds[1].ptr, self.parts,
                self.out[0].ptr, self.out[1].ptr, self.out[2].ptr, self.out_capacity, self.result.ptr,
                self.stream.handle))
            self.launches += 2
            if self.timing:
                self._ev[2].record(self.stream)
            self._tp("join_end")
            raw = native.to_host(self.result.ptr, 32, self.stream)
            if self.tracing:  # the read-back synchronised the stream
                t0 = self._trace_points[0][1]
                self.trace = {name: round(t0.elapsed_ms(ev), 3) for name, ev in self._trace_points}
            if self.timing:  # the read-back synchronised the stream
                self.kernel_ms["partition"] += self._ev[0].elapsed_ms(self._ev[1])
                self.kernel_ms["join"] += self._ev[1].elapsed_ms(self._ev[2])
            self._mark("join_ms")
            produced, count, hsum, ksum = struct.unpack("<4Q", raw)
            if count <= self.out_capacity:
                self.rows_out = count
                return count, hsum, ksum
            # output cut short: grow and re-join (rare: skewed keys)
            self.out_capacity = int(count * 1.1) + 65536
            self.out = [native.DeviceBuffer(self.device, self.out_capacity * 8) for _ in range(3)]

    async def run_global(self) -> tuple[int, int, int]:
        """run() plus the digest summed over all ranks (the global row count of SPEC.md:426)."""
        mine = await self.run()
        if self.world == 1:
            return mine
        parts = await allgather(self.transport, struct.pack("<5Q", *mine, *self.received), tag=EXCHANGE_TAG + 1)
        total = [0, 0, 0]
        received = [0, 0]
        for blob in parts:
            vals = struct.unpack("<5Q", blob)
            for k in range(3):
                total[k] = (total[k] + vals[k]) & _MASK64
            received[0] += vals[3]
            received[1] += vals[4]
        # row conservation: every generated row reached exactly one owner
        if received != [self.total, self.total]:
            raise CommShimError(f"row conservation violated: owners received {received} rows per side, "
                                f"{self.total} generated")
        self.conserved = True
        return tuple(total)

    def output_rows(self, limit: int | None = None):
        """The materialised (key, lval, rval) rows of this rank (host copy, for tests)."""
        import numpy as np

        n = self.rows_out if limit is None else min(limit, self.rows_out)
        cols = [np.frombuffer(native.to_host(b.ptr, n * 8, self.stream), dtype=np.int64) for b in self.out]
        return cols

    def algorithmic_bytes(self) -> dict:
        """read both input tables once (16 B/row/side), write the
        output once (24 B/row); NVLink: the rows that change owner (16 B/row/side)."""
        moved = 0
        if self.world > 1:
            moved = 2 * self.n * 16 * (self.world - 1) // self.world
        return {"hbm": 2 * self.n * 16 + getattr(self, "rows_out", 0) * 24, "nvlink": moved}
