"""``transpose_sum``: sum(x + x.T) over a chunked fp64 array on B200s.

Operator definition: SPEC.md:413-421 (block (i,j) of y needs x(i,j) and
x(j,i); deterministic checksum of y; result identical for any worker count),
ownership round-robin over workers in row-major block order,
PAPER.md:380-383 (``y = x + x.T; y.persist(); wait(y)``).

B200 layout.  Each rank keeps the blocks it owns in one dedicated
``cudaMalloc`` pool (``x`` pool and ``y`` pool, block-major, every block
row-major ``b*b`` fp64), so one CUDA-IPC handle exports a rank's whole ``x``.
A block whose transpose partner lives on another GPU is computed by reading
the partner tile straight out of that peer's pool over NVLink inside the
fused kernel: no staging copy, no separate exchange step.  Pairs whose two
blocks are both local are computed together so ``x`` is read exactly once
(16 B of HBM per output element).

The scalar is the fixed-order per-block sums (device) combined with
``math.fsum`` in global row-major block order, so it is bit-identical for
every worker count.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
from dataclasses import dataclass

from .. import native
from ..errors import UsageError

DEFAULT_SEED = 0x210108878


def owner_of(i: int, j: int, nb: int, world: int) -> int:
    """Round-robin row-major block placement."""
    return (i * nb + j) % world


@dataclass
class TransposeSumResult:
    checksum: float
    block_sums: dict  # global block id -> fp64 sum of that y block


class TransposeSum:
    """One rank's share of a distributed ``y = x + x.T`` with a deterministic checksum.

    ``exchange(payload: bytes) -> list[bytes]`` is an all-gather over the world
    (only needed when ``world > 1``); the harness uses it once at setup to swap
    IPC handles of the ``x`` pools, and once per step to gather block sums.
    """

    def __init__(self, n: int, b: int, *, rank: int = 0, world: int = 1, device: int = 0,
                 seed: int = DEFAULT_SEED, exchange=None, stream: native.Stream | None = None):
        if b <= 0 or n <= 0 or n % b:
            raise UsageError(f"dims {n} not divisible by block {b}")
        if not 0 <= rank < world:
            raise UsageError(f"rank {rank} outside world {world}")
        if world > 1 and exchange is None:
            raise UsageError("a multi-worker transpose_sum needs an exchange function")
        self.n, self.b, self.nb = n, b, n // b
        self.rank, self.world, self.device, self.seed = rank, world, device, seed
        self.exchange = exchange
        native.set_device(device)
        self.stream = stream or native.Stream(device)
        nb = self.nb
        self.owned = [g for g in range(nb * nb) if g % world == rank]  # row-major ids
        self.slot_of = {g: s for s, g in enumerate(self.owned)}
        self.block_bytes = b * b * 8
        pool_bytes = max(1, len(self.owned)) * self.block_bytes
        self.x = native.DeviceBuffer(device, pool_bytes)
        self.y = native.DeviceBuffer(device, pool_bytes)
        self.sums = native.DeviceBuffer(device, max(1, len(self.owned)) * 8 + 8)
        self._peer_bases: dict[int, int] = {}
        self._imported: list[int] = []
        self._plan = None
        self.tasks_single = 0
        self.tasks_paired = 0
        self.tasks_diag = 0

    # -- layout -------------------------------------------------------------------------------

    def x_ptr(self, g: int) -> int:
        return self.x.ptr + self.slot_of[g] * self.block_bytes

    def y_ptr(self, g: int) -> int:
        return self.y.ptr + self.slot_of[g] * self.block_bytes

    def remote_x_ptr(self, g: int) -> int:
        owner = g % self.world
        slot = g // self.world  # position of g among its owner's row-major blocks
        return self._peer_bases[owner] + slot * self.block_bytes

    def generate(self) -> None:
        """Fill this rank's x blocks with the deterministic generator."""
        lib = native.lib()
        native.set_device(self.device)
        for g in self.owned:
            i, j = divmod(g, self.nb)
            native.check(lib.m4d_fill_block_f64(self.x_ptr(g), self.n, i * self.b, j * self.b, self.b,
                                                self.seed, self.stream.handle))
        self.stream.synchronize()

    # -- setup ---------------------------------------------------------------------------------

    def connect_peers(self) -> None:
        """Swap CUDA-IPC handles of the x pools so partner tiles can be read over NVLink."""
        if self.world == 1:
            return
        handle, offset = native.ipc_export(self.x.ptr)
        blob = struct.pack("<iQQ", os.getpid(), self.x.ptr, offset) + handle
        gathered = self.exchange(blob)
        for peer, item in enumerate(gathered):
            if peer == self.rank:
                continue
            pid, ptr, off = struct.unpack_from("<iQQ", item)
            if pid == os.getpid():  # same process (multi-rank test mode): plain peer pointer
                self._peer_bases[peer] = ptr
            else:
                base = native.ipc_import(self.device, item[20:84])
                self._imported.append(base)
                self._peer_bases[peer] = base + off

    def build_plan(self) -> None:
        nb, world, rank = self.nb, self.world, self.rank
        tasks = []
        for g in self.owned:
            i, j = divmod(g, nb)
            t = native.TsTask()
            t.slot_y = self.slot_of[g]
            t.slot_y2 = -1
            t.a = self.x_ptr(g)
            t.y = self.y_ptr(g)
            if i == j:
                t.bt = t.a
                t.diag = 1
                self.tasks_diag += 1
            else:
                partner = j * nb + i
                if partner % world == rank:
                    if i > j:
                        continue  # covered by the pair task of (j, i)
                    t.bt = self.x_ptr(partner)
                    t.y2 = self.y_ptr(partner)
                    t.slot_y2 = self.slot_of[partner]
                    self.tasks_paired += 1
                else:
                    t.bt = self.remote_x_ptr(partner)
                    t.remote = 1 + partner % world  # item stream of the peer the tile is read from
                    self.tasks_single += 1
            tasks.append(t)
        arr = (native.TsTask * max(1, len(tasks)))(*tasks)
        plan = ctypes.c_void_p()
        native.check(native.lib().m4d_ts_plan_create(self.device, arr, len(tasks), self.b,
                                                     len(self.owned), ctypes.byref(plan)))
        self._plan = plan.value

    def setup(self, generate: bool = True) -> "TransposeSum":
        if generate:
            self.generate()
        self.connect_peers()
        self.build_plan()
        return self

    # -- step ------------------------------------------------------------------------------------

    def launch(self) -> None:
        """Enqueue the fused kernel on ``self.stream``."""
        native.check(native.lib().m4d_ts_run(self._plan, self.sums.ptr,
                                             self.sums.ptr + len(self.owned) * 8, self.stream.handle))

    def read_block_sums(self) -> dict:
        native.set_device(self.device)
        raw = native.to_host(self.sums.ptr, len(self.owned) * 8, self.stream)
        values = struct.unpack(f"<{len(self.owned)}d", raw)
        return dict(zip(self.owned, values))

    def combine(self, local_sums: dict) -> TransposeSumResult:
        """Gather every rank's block sums and fsum them in global row-major order."""
        if self.world > 1:
            blob = struct.pack(f"<{2 * len(local_sums)}d",
                               *[v for g in sorted(local_sums) for v in (float(g), local_sums[g])])
            merged = {}
            for item in self.exchange(blob):
                vals = struct.unpack(f"<{len(item) // 8}d", item)
                for k in range(0, len(vals), 2):
                    merged[int(vals[k])] = vals[k + 1]
        else:
            merged = dict(local_sums)
        ordered = [merged[g] for g in sorted(merged)]
        return TransposeSumResult(math.fsum(ordered), merged)

    def step(self) -> TransposeSumResult:
        self.launch()
        return self.combine(self.read_block_sums())

    def load_x(self, host_ptr: int, stream: native.Stream | None = None) -> None:
        """Upload this rank's x pool (block-major, the layout of ``self.x``) from host
        memory for the next step, then fence: peers read partner tiles straight out of
        this pool over NVLink, so no rank may launch before every rank's upload has
        landed.  (The reverse hazard -- overwriting a pool a peer's previous kernel is
        still reading -- is excluded by step(): its block-sum exchange completes only
        after every rank's kernel finished.)"""
        s = stream or self.stream
        native.memcpy(self.x.ptr, host_ptr, len(self.owned) * self.block_bytes, s)
        if self.world > 1:
            s.synchronize()
            self.exchange(b"\x01")  # input-ready barrier
        elif s is not self.stream:
            s.synchronize()

    def read_y_block(self, g: int) -> bytes:
        native.set_device(self.device)
        return native.to_host(self.y_ptr(g), self.block_bytes, self.stream)

    def close(self) -> None:
        if self._plan:
            native.lib().m4d_ts_plan_destroy(self._plan)
            self._plan = None
        for base in self._imported:
            try:
                native.ipc_close(base)
            except Exception:
                pass
        self._imported.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def local_world(cls, n: int, b: int, world: int, *, devices=None, seed: int = DEFAULT_SEED):
        """All ``world`` ranks in this process (test mode): peers are wired with
        plain device pointers (peer access enabled across distinct devices)."""
        devices = list(devices) if devices is not None else [0] * world
        ranks = [cls(n, b, rank=r, world=world, device=devices[r], seed=seed, exchange=lambda _b: [])
                 for r in range(world)]
        for r in ranks:
            r.generate()
        for r in ranks:
            for peer in ranks:
                if peer is not r:
                    native.check(native.lib().m4d_enable_peer(r.device, peer.device))
                    r._peer_bases[peer.rank] = peer.x.ptr
            r.build_plan()
        return ranks

    # -- roofline bookkeeping -----------------------------------------------------------------

    def algorithmic_bytes(self) -> dict:
        """HBM and NVLink bytes one step must move on this rank:
        8 B read of x + 8 B write of y per output element, plus 8 B over NVLink per
        element whose transpose partner is remote."""
        elems = self.b * self.b
        owned = len(self.owned)
        remote = self.tasks_single
        return {
            "hbm": owned * elems * 16,
            "nvlink": remote * elems * 8,
        }
