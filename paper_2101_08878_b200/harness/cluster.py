"""Mini cluster bootstrap and heartbeat accounting.

Roles follow the paper's dask-mpi convention (§IV-A): rank 0 is the
scheduler, rank 1 the client, ranks >= 2 are workers; ``world_size == 2`` is
a configuration error (no workers), 1 is a solo run.  Everything below is
control plane: registration, heartbeats and shutdown travel as small utf-8
frames over :class:`~paper_2101_08878_b200.endpoints.Endpoint`s on the same
transport (and executor) as the bulk data, which is the paper's control /
data isolation claim (Fig. 2's dotted control connections) made testable.

* ``bootstrap()`` — the scheduler listens on ``mpi://0``; the client and
  every worker connect and register; once all have, the scheduler answers
  each with the worker set.
* ``heartbeat_loop()`` (workers) — one beat per interval on the worker's
  control endpoint until the scheduler says stop.
* the scheduler counts beats per worker and marks a worker *suspect* when
  more than ``suspect_after`` (3) intervals pass without one -- a report, no
  eviction.
* ``stop_all()`` (client) — the scheduler relays stop to every worker and
  collects their last beats; ``report()`` gives beats and suspects.

Intervals are in the loop clock's units: ticks on the simulated transport
(deterministic tests), seconds on real transports.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ..endpoints import Endpoint, Node, connect, listen
from ..errors import CommShimError, ConfigurationError, EndOfStream
from ..loop import current_loop, sleep, spawn
from ..messaging import Message, make_frame

SCHEDULER, CLIENT, WORKER, SOLO = "scheduler", "client", "worker", "solo"


def role_of(rank: int, world: int) -> str:
    """Rank 0 scheduler, 1 client, >= 2 workers."""
    if world == 1:
        return SOLO
    if world == 2:
        raise ConfigurationError("cluster mode needs world_size >= 3 (ranks 0 and 1 are scheduler and client)")
    return SCHEDULER if rank == 0 else CLIENT if rank == 1 else WORKER


@dataclass
class Role:
    kind: str
    rank: int
    world: int
    workers: list[int] = field(default_factory=list)


@dataclass
class HeartbeatReport:
    beats: dict[int, int]
    suspects: list[tuple[object, int]]  # (clock time of the report, worker rank)
    closed: list[int]                   # workers whose control endpoint ended without a goodbye


def _msg(*parts) -> Message:
    return Message([make_frame("|".join(str(p) for p in parts), 1)])


def _parts(msg: Message) -> list[str]:
    return msg.frames[0].decode().split("|")


class Cluster:
    """One rank of the mini cluster."""

    def __init__(self, node: Node, *, heartbeat_interval, suspect_after: int = 3):
        self.node = node
        self.rank = node.rank
        self.world = node.transport.world_size
        self.kind = role_of(self.rank, self.world)
        self.interval = heartbeat_interval
        self.suspect_after = suspect_after
        self.workers: list[int] = []
        self._ep: Endpoint | None = None           # client / worker: control endpoint to the scheduler
        self._eps: dict[int, Endpoint] = {}        # scheduler: rank -> control endpoint
        self._kinds: dict[int, str] = {}
        self._registered = None
        self._stop = False
        self.beats: dict[int, int] = {}
        self._last: dict[int, object] = {}
        self._suspects: list[tuple[object, int]] = []
        self._closed: list[int] = []
        self._byes = 0
        self._stop_requested = None
        self._listener = None

    # -- bootstrap --------------------------------------------------------------------------

    async def bootstrap(self) -> Role:
        if self.kind == SOLO:
            return Role(SOLO, 0, 1)
        loop = current_loop()
        if self.kind == SCHEDULER:
            self._registered = loop.create_future()
            self._stop_requested = loop.create_future()
            self._listener = listen(self.node, "mpi://0", self._on_connection)
            await self._listener.start()
            await self._registered
            self.workers = sorted(r for r, k in self._kinds.items() if k == WORKER)
            for r, ep in sorted(self._eps.items()):
                await ep.write(_msg("ready", ",".join(map(str, self.workers))))
            now = self.node.transport.clock.now()
            for r in self.workers:
                self.beats[r] = 0
                self._last[r] = now
                spawn(self._read_worker(r), name=f"beats-{r}")
            spawn(self._monitor(), name="suspects")
        else:
            self._ep = await connect(self.node, "mpi://0")
            await self._ep.write(_msg("register", self.kind, self.rank))
            kind, workers = _parts(await self._ep.read())
            if kind != "ready":
                raise CommShimError(f"unexpected bootstrap reply {kind!r}")
            self.workers = [int(w) for w in workers.split(",") if w]
        return Role(self.kind, self.rank, self.world, list(self.workers))

    async def _on_connection(self, ep: Endpoint) -> None:
        kind, kind_name, rank = _parts(await ep.read())
        if kind != "register":
            raise CommShimError(f"expected a registration, got {kind!r}")
        self._eps[int(rank)] = ep
        self._kinds[int(rank)] = kind_name
        if len(self._eps) == self.world - 1 and not self._registered.done():
            self._listener.stop()
            self._registered.set_result(None)
        if kind_name == CLIENT:  # the client's only request: stop the workers
            msg = await ep.read()
            if _parts(msg)[0] == "stop" and not self._stop_requested.done():
                self._stop_requested.set_result(None)

    # -- heartbeats -------------------------------------------------------------------------

    async def heartbeat_loop(self) -> int:
        """Worker: beat every interval until the scheduler says stop.  Returns beats sent."""
        if self.kind != WORKER:
            raise CommShimError("only workers send heartbeats")

        async def watch():
            try:
                if _parts(await self._ep.read())[0] == "stop":
                    self._stop = True
            except (EndOfStream, CommShimError):
                self._stop = True

        spawn(watch(), name="stop-watch")
        seq = 0
        while not self._stop:
            await self._ep.write(_msg("beat", self.rank, seq))
            seq += 1
            await sleep(self.interval)
        await self._ep.write(_msg("bye", self.rank, seq))
        return seq

    async def _read_worker(self, r: int) -> None:
        ep = self._eps[r]
        clock = self.node.transport.clock
        while True:
            try:
                kind = _parts(await ep.read())[0]
            except (EndOfStream, CommShimError):
                self._closed.append(r)
                self._byes += 1
                return
            if kind == "beat":
                self.beats[r] += 1
                self._last[r] = clock.now()
            elif kind == "bye":
                self._byes += 1
                self._last.pop(r, None)
                return

    async def _monitor(self) -> None:
        clock = self.node.transport.clock
        flagged: set[int] = set()
        while self._byes < len(self.workers):
            await sleep(self.interval)
            now = clock.now()
            for r, last in list(self._last.items()):
                if r not in flagged and now - last > self.suspect_after * self.interval:
                    flagged.add(r)
                    self._suspects.append((now, r))

    # -- shutdown ---------------------------------------------------------------------------

    async def stop_all(self) -> None:
        """Client: ask the scheduler to stop every worker's heartbeat loop."""
        if self.kind != CLIENT:
            raise CommShimError("stop_all is the client's request")
        await self._ep.write(_msg("stop"))

    async def serve(self) -> HeartbeatReport:
        """Scheduler: wait for the client's stop, relay it, collect the last beats."""
        if self.kind != SCHEDULER:
            raise CommShimError("serve runs on the scheduler")
        await self._stop_requested
        for r in self.workers:
            try:
                await self._eps[r].write(_msg("stop"))
            except CommShimError:
                pass  # a dead worker: its reader already recorded the close
        while self._byes < len(self.workers):
            await sleep(self.interval)
        return self.report()

    def report(self) -> HeartbeatReport:
        return HeartbeatReport(dict(self.beats), list(self._suspects), list(self._closed))

    async def close(self) -> None:
        for ep in ([self._ep] if self._ep else []) + list(self._eps.values()):
            try:
                await ep.close()
            except CommShimError:
                pass
