"""Small-frame storm: many concurrent endpoints per worker pair.

Workload: ``total`` frames with sizes log-uniform in [1 B, 8 KiB] (seed
``0x5EED``) spread over every ordered worker pair, ``conns`` endpoints per
ordered pair (``Endpoint`` is single-writer / single-reader,
``endpoints.py:144-145, :161-162`` of the reference), one writer and one reader
task per endpoint, all on one cooperative executor per worker.  Reported:
wall time (first writer start to last reader finish, over all workers),
frames/s, and the per-frame latency distribution (send call to read return).

The harness is written against the reference's public API (``Node``,
``Endpoint``, ``CommTable.duplicate``, ``Message``/``Frame``, ``TaskLoop``),
passed in as a namespace, so the same code drives this package on the nvlink
transport and the reference package on its socket transport (the bench's
reference arm).  Endpoints are created pairwise from agreed duplicate-channel
generations instead of listen/connect: the reference's listener cannot run on a
rank that also connects (defect D2), and connection setup is outside
the timed region anyway.  Stream ``c`` from the low rank to the high rank of a
pair uses generation ``2c+1``, the reverse direction ``2c+2``.

Payload bytes are deterministic per frame id and checked bit-exactly after
the timed region.

``device=d`` (this package only): the frames are device frames on cuda:d --
windows of one pool uploaded before the timed region -- so every frame moves
GPU to GPU by the transport's eager device protocol (sender proxy-kernel copy
into the receiver's device ring, received by loan).
"""

from __future__ import annotations

import random
import struct
import time
from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np

STORM_SEED = 0x5EED
MAX_FRAME = 8192


def frame_sizes(total: int, seed: int = STORM_SEED, max_frame: int = MAX_FRAME) -> list[int]:
    """Log-uniform sizes in [1, max_frame] (one per global frame id)."""
    rng = random.Random(seed)
    top = float(np.log2(max_frame))
    return [min(max_frame, max(1, int(2.0 ** rng.uniform(0.0, top)))) for _ in range(total)]


def payload(frame_id: int, size: int) -> bytes:
    return ((np.arange(size, dtype=np.uint32) * 7 + frame_id * 31) & 0xFF).astype(np.uint8).tobytes()


def streams(world: int, conns: int) -> list[tuple[int, int, int]]:
    """Every (src, dst, c) stream, in a fixed global order."""
    return [(s, d, c) for s in range(world) for d in range(world) if s != d for c in range(conns)]


def generation(src: int, dst: int, c: int) -> int:
    return 2 * c + 1 if src < dst else 2 * c + 2


def assign(total: int, world: int, conns: int) -> dict:
    """Frame ids per stream: frame k goes to stream k mod S (round-robin)."""
    ss = streams(world, conns)
    out = {s: [] for s in ss}
    for k in range(total):
        out[ss[k % len(ss)]].append(k)
    return out


def namespace_of(package) -> SimpleNamespace:
    """The API surface the storm uses, taken from ``package`` (this one or the reference)."""
    import importlib

    name = package if isinstance(package, str) else package.__name__
    ep = importlib.import_module(name + ".endpoints")
    msg = importlib.import_module(name + ".messaging")
    ch = importlib.import_module(name + ".channels")
    lp = importlib.import_module(name + ".loop")
    ns = SimpleNamespace(Node=ep.Node, Endpoint=ep.Endpoint, build_comm_table=ch.build_comm_table,
                         Message=msg.Message, Frame=msg.Frame, make_frame=msg.make_frame,
                         send_payload=msg.send_payload, recv_payload=msg.recv_payload, TaskLoop=lp.TaskLoop,
                         MonotonicClock=lp.MonotonicClock, gather=lp.gather, device_frames=None)
    if name == __name__.rsplit(".", 2)[0]:
        ns.device_frames = _device_frames
    return ns


def _device_frames(blobs: list[bytes], device: int) -> list:
    """Device frames holding ``blobs``: 256-byte aligned windows of one cuda:device pool
    (one allocation, one upload)."""
    from ..messaging import Frame
    from ..transport import MemoryDomain
    from ..transport.nvlink import CudaRegion

    offs, at = [], 0
    for b in blobs:
        offs.append(at)
        at += (len(b) + 255) & ~255
    host = bytearray(max(at, 1))
    for o, b in zip(offs, blobs):
        host[o:o + len(b)] = b
    pool = CudaRegion(bytes(host), device)
    return [Frame(CudaRegion(len(b), device, ptr=pool.ptr + o, owner=pool), len(b), MemoryDomain.DEVICE)
            for o, b in zip(offs, blobs)]


@dataclass
class StormResult:
    frames: int
    bytes: int
    wall_s: float
    frames_per_s: float
    p50_us: float
    p99_us: float
    max_us: float
    verified: int


class StormWorker:
    """One worker's side of the storm: writers for its outgoing streams, readers for its incoming ones."""

    def __init__(self, ns: SimpleNamespace, transport, *, conns: int = 8, total: int = 100_000,
                 seed: int = STORM_SEED, device: int | None = None):
        self.ns, self.t = ns, transport
        self.rank, self.world = transport.rank, transport.world_size
        self.conns, self.total = conns, total
        self.sizes = frame_sizes(total, seed)
        self.plan = assign(total, self.world, conns)
        self.node = ns.Node(transport, ns.build_comm_table(transport))
        self.out, self.inc = {}, {}
        for (s, d, c), ids in self.plan.items():
            if s == self.rank or d == self.rank:
                peer = d if s == self.rank else s
                chan = self.node.table.duplicate(peer, generation=generation(s, d, c))
                origin = "connector" if s == self.rank else "listener"
                ep = ns.Endpoint(self.node, chan, peer, origin, (s << 20) | (d << 10) | c)
                (self.out if s == self.rank else self.inc)[(s, d, c)] = (ep, ids)
        ids_out = [k for _, ids in self.out.values() for k in ids]
        if device is None:
            self.frames_out = {k: ns.Frame(payload(k, self.sizes[k]), self.sizes[k]) for k in ids_out}
        else:
            if ns.device_frames is None:
                raise ValueError("device frames need this package's namespace")
            frames = ns.device_frames([payload(k, self.sizes[k]) for k in ids_out], device)
            self.frames_out = dict(zip(ids_out, frames))
        self.sent_ns: dict[int, int] = {}
        self.recv_ns: dict[int, int] = {}
        self.received: dict[int, object] = {}
        self.rounds: list[tuple] = []  # (t_start, t_end, sent, recv) per timed round

    async def _writer(self, ep, ids) -> None:
        Message, frames, stamp = self.ns.Message, self.frames_out, self.sent_ns
        for k in ids:
            stamp[k] = time.monotonic_ns()
            await ep.write(Message([frames[k]]))

    async def _reader(self, ep, ids) -> None:
        stamp, got = self.recv_ns, self.received
        for k in ids:
            msg = await ep.read()
            stamp[k] = time.monotonic_ns()
            got[k] = msg.frames[0]

    async def run(self, timed: bool = True) -> None:
        """One round (the timed region): every writer and reader of this worker, concurrently."""
        self.sent_ns, self.recv_ns = {}, {}
        tasks = [self._writer(ep, ids) for ep, ids in self.out.values()]
        tasks += [self._reader(ep, ids) for ep, ids in self.inc.values()]
        t_start = time.monotonic_ns()
        await self.ns.gather(*tasks)
        t_end = time.monotonic_ns()
        if timed:
            self.rounds.append((t_start, t_end, self.sent_ns, self.recv_ns))

    async def close(self) -> None:
        await self.ns.gather(*[ep.close() for ep, _ in list(self.out.values()) + list(self.inc.values())])

    def verify(self) -> int:
        """Bit-exact check of the last round's received frames; returns how many were checked."""
        bad = [k for k, f in self.received.items() if f.to_bytes() != payload(k, self.sizes[k])]
        if bad:
            raise AssertionError(f"storm: {len(bad)} frames corrupted (first id {bad[0]})")
        return len(self.received)

    def report(self) -> bytes:
        """This worker's timed rounds for the cross-worker summary (see :func:`summarise`)."""
        out = [struct.pack("<q", len(self.rounds))]
        for t_start, t_end, sent_ns, recv_ns in self.rounds:
            sent = np.array(sorted(sent_ns.items()), dtype=np.int64).reshape(-1, 2)
            recv = np.array(sorted(recv_ns.items()), dtype=np.int64).reshape(-1, 2)
            out += [struct.pack("<qqqq", t_start, t_end, len(sent), len(recv)), sent.tobytes(), recv.tobytes()]
        return b"".join(out)


def summarise(reports: list[bytes], sizes: list[int], verified: int) -> StormResult:
    """Combine every worker's report (same-host CLOCK_MONOTONIC, so stamps compare across
    processes).  Wall time per round = last reader finish - first writer start over all
    workers; rounds add up."""
    per_round: dict[int, list] = {}
    for blob in reports:
        (nrounds,) = struct.unpack_from("<q", blob)
        off = 8
        for r in range(nrounds):
            a, b, ns_, nr = struct.unpack_from("<qqqq", blob, off)
            off += 32
            arr = np.frombuffer(blob, dtype=np.int64, count=2 * (ns_ + nr), offset=off)
            off += 16 * (ns_ + nr)
            per_round.setdefault(r, []).append((a, b, arr[: 2 * ns_].reshape(-1, 2), arr[2 * ns_:].reshape(-1, 2)))
    wall, lats, frames = 0.0, [], 0
    for r, parts in sorted(per_round.items()):
        sent = {int(k): int(v) for _, _, s, _ in parts for k, v in s}
        recv = {int(k): int(v) for _, _, _, q in parts for k, v in q}
        if len(recv) != len(sizes) or set(recv) != set(sent):
            raise AssertionError(f"storm round {r}: {len(recv)} of {len(sizes)} frames accounted for")
        ids = sorted(recv)
        lats.append((np.array([recv[k] for k in ids]) - np.array([sent[k] for k in ids])) / 1e3)
        wall += (max(p[1] for p in parts) - min(p[0] for p in parts)) / 1e9
        frames += len(ids)
    lat = np.concatenate(lats) if lats else np.zeros(1)
    return StormResult(frames=frames, bytes=int(sum(sizes)) * len(per_round), wall_s=wall,
                       frames_per_s=frames / wall if wall else 0.0,
                       p50_us=float(np.percentile(lat, 50)), p99_us=float(np.percentile(lat, 99)),
                       max_us=float(lat.max()), verified=verified)


def run_worker(ns: SimpleNamespace, transport, sync, *, conns: int = 8, total: int = 100_000,
               seed: int = STORM_SEED, rounds: int = 1, warmup: int = 0, verify: bool = True,
               device: int | None = None) -> StormResult:
    """One worker process: set up, then per round a barrier and the timed storm;
    close, verify, gather.  ``sync(bytes) -> list[bytes]`` is an all-gather over
    the workers (any control plane: torch.distributed gloo, or the transport
    itself).  Returns the :class:`StormResult` on every worker."""
    w = StormWorker(ns, transport, conns=conns, total=total, seed=seed, device=device)
    loop = ns.TaskLoop(ns.MonotonicClock())
    for r in range(warmup + rounds):
        w.received = {}  # (device frames: received frames hold ring slots until dropped)
        sync(b"go")
        loop.run_until_complete(w.run(timed=r >= warmup))
    loop.run_until_complete(w.close())
    checked = w.verify() if verify else 0
    reports = sync(w.report() + struct.pack("<q", checked))
    verified = sum(struct.unpack("<q", r[-8:])[0] for r in reports)
    return summarise([r[:-8] for r in reports], w.sizes, verified)


def run_local(ns: SimpleNamespace, transports, *, conns: int = 8, total: int = 100_000,
              seed: int = STORM_SEED, rounds: int = 1, device: int | None = None) -> StormResult:
    """Every worker in this process on one executor (tests; in-process worlds)."""
    workers = [StormWorker(ns, t, conns=conns, total=total, seed=seed, device=device) for t in transports]
    loop = ns.TaskLoop(ns.MonotonicClock())

    async def all_runs():
        for _ in range(rounds):
            await ns.gather(*[w.run() for w in workers])
        await ns.gather(*[w.close() for w in workers])

    loop.run_until_complete(all_runs())
    verified = sum(w.verify() for w in workers)
    return summarise([w.report() for w in workers], workers[0].sizes, verified)


def transport_sync(transport, tag: int = 950):
    """An all-gather of variable-length blobs over the transport's world channel
    (works with this package's transports and the reference's)."""
    from .collectives import allgather_sync

    def sync(blob: bytes) -> list[bytes]:
        lens = [struct.unpack("<q", b)[0] for b in allgather_sync(transport, struct.pack("<q", len(blob)), tag)]
        padded = allgather_sync(transport, blob + bytes(max(lens) - len(blob)), tag + 1)
        return [p[:n] for p, n in zip(padded, lens)]

    return sync
