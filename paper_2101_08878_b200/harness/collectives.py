"""Small host-side collectives over the comm transport (control plane of the operators).

The operators' bulk bytes move as device frames (NVLink); these helpers only
carry metadata — IPC handles, row counts, per-block sums — as eager host
messages on the world channel (tags >= 900 are reserved for the harness).
"""

from __future__ import annotations

import time

from ..errors import CommShimError
from ..messaging import await_request

_SYNC_TIMEOUT = 120.0


def _post_exchange(transport, payload: bytes, tag: int):
    world, me = transport.world_size, transport.rank
    bufs = {p: bytearray(len(payload)) for p in range(world) if p != me}
    reqs = [transport.post_recv(0, p, tag, bufs[p]) for p in bufs]
    reqs += [transport.post_send(0, p, tag, payload) for p in bufs]
    return bufs, reqs


def _collect(world: int, me: int, payload: bytes, bufs: dict) -> list[bytes]:
    out = [b""] * world
    out[me] = payload
    for p, b in bufs.items():
        out[p] = bytes(b)
    return out


async def allgather(transport, payload: bytes, tag: int) -> list[bytes]:
    """Every rank's equally sized ``payload``, in rank order (coroutine)."""
    if transport is None or transport.world_size == 1:
        return [payload]
    bufs, reqs = _post_exchange(transport, payload, tag)
    for r in reqs:
        await await_request(transport, r)
    return _collect(transport.world_size, transport.rank, payload, bufs)


def allgather_sync(transport, payload: bytes, tag: int) -> list[bytes]:
    """Blocking variant for code outside an event loop (drives progress itself)."""
    if transport is None or transport.world_size == 1:
        return [payload]
    bufs, reqs = _post_exchange(transport, payload, tag)
    deadline = time.monotonic() + _SYNC_TIMEOUT
    for r in reqs:
        while r.pending:
            transport.progress()
            if time.monotonic() > deadline:
                raise CommShimError(f"allgather timed out waiting for {r}")
        if r.failed:
            raise r.error
    return _collect(transport.world_size, transport.rank, payload, bufs)


def barrier_sync(transport, tag: int) -> None:
    allgather_sync(transport, b"\x00", tag)
