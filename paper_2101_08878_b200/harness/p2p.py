"""Point-to-point micro-benchmarks of the paper's §V-A (Fig. 6) on the nvlink transport.

Methodology (reference pattern
``pkg/tests/test_messaging.py:301-333``):

* ``pingpong``   — rank 0 sends a frame with ``send_payload`` and awaits the
  echo from rank 1 (``recv_payload``); latency = RTT / 2, throughput =
  2 * size / RTT.  This is the full comm path: transfer header + payload
  chunks, cooperative polling on the executor.
* ``osu_bw``     — transport layer: rank 0 posts a window of back-to-back
  ``post_send``s, rank 1 a window of ``post_recv``s, then a 4-byte ack;
  GB/s = size * window * iters / time (osu_bw style).
* ``osu_latency``— transport layer ping-pong with raw posts (no framing).

Device frames live in B200 memory (CudaRegion) and move GPU-to-GPU over
NVLink by CUDA-IPC rendezvous; host frames move through the shared-memory
rings.  Every payload is checked bit-exactly once per size outside the
timed loop.
"""

from __future__ import annotations

import time
from types import SimpleNamespace

from ..channels import build_comm_table
from ..loop import MonotonicClock, TaskLoop
from ..messaging import Frame, make_frame, recv_payload, send_payload
from ..transport import MemoryDomain, Transport

ACK_TAG = 1001
DATA_TAG = 1002
PP_TAG = 1003
CHECK_TAG = 1004


def pattern(n: int, salt: int = 0) -> bytes:
    block = bytes((k * 131 + salt * 17 + 7) & 0xFF for k in range(4096))
    return (block * (n // 4096 + 1))[:n]


def _wait(transport: Transport, *reqs, timeout: float = 60.0) -> None:
    deadline = time.monotonic() + timeout
    for r in reqs:
        while r.pending:
            transport.progress()
            if time.monotonic() > deadline:
                raise TimeoutError(f"request stuck: {r}")
        if r.failed:
            raise r.error


def _region(transport: Transport, data: bytes, device: bool):
    if device:
        from ..transport.nvlink import CudaRegion

        return CudaRegion(data, transport.device)
    return bytearray(data)


def _window(buf, device: bool, n: int):
    return buf.window(0, n) if device else memoryview(buf)[:n]


def verify_once(transport: Transport, peer: int, n: int, device: bool) -> None:
    """Bit-exact check of one transfer of size n (outside timing)."""
    me = transport.rank
    dom = MemoryDomain.DEVICE if device else MemoryDomain.HOST
    if me == 0:
        src = _region(transport, pattern(n, 1), device)
        _wait(transport, transport.post_send(0, peer, CHECK_TAG, _window(src, device, n), dom))
    else:
        dst = _region(transport, bytes(n), device)
        _wait(transport, transport.post_recv(0, peer, CHECK_TAG, _window(dst, device, n), dom))
        got = dst.to_bytes() if device else bytes(dst)
        if got != pattern(n, 1):
            raise AssertionError(f"p2p payload of {n} bytes differs")


def _blank(transport: Transport, nbytes: int, device: bool):
    if device:
        from .. import native
        from ..transport.nvlink import CudaRegion

        region = CudaRegion(max(1, nbytes), transport.device)
        native.check(native.lib().m4d_memset(region.ptr, 0x5A, max(1, nbytes), None))
        native.check(native.lib().m4d_stream_sync(None))
        return region
    return bytearray(nbytes)


def _slot(buf, device: bool, k: int, n: int):
    return buf.window(k * n, n) if device else memoryview(buf)[k * n:(k + 1) * n]


def osu_bw(transport: Transport, peer: int, n: int, window: int, iters: int, device: bool,
           vectored: bool | None = None) -> float:
    """Transport-layer bandwidth in GB/s (measured on rank 0; rank 1 mirrors).

    Every message of a window has its own source and destination region (the
    OSU benchmark reuses one buffer, which lets concurrent pulls of identical
    lines be served once and reports more than the link can carry).
    ``vectored``: post each device window with one ``post_many`` call instead
    of the MPI_Isend / MPI_Irecv loop (same posts, same order).  Off by
    default: measured slower at 1-16 MiB (4 MiB: 584-635 vs 691-697 GB/s,
    ``profiles/r2_post_many_p2p.txt``) -- the whole window's pulls launch at
    once and crowd the four pull streams, where the posting loop staggers them."""
    me = transport.rank
    dom = MemoryDomain.DEVICE if device else MemoryDomain.HOST
    buf = _blank(transport, n * window, device)
    views = [_slot(buf, device, k, n) for k in range(window)]
    many = getattr(transport, "post_many", None) if (device and vectored) else None
    ack = bytearray(4)
    start = None
    for it in range(iters + 1):  # iteration 0 is warm-up
        if it == 1:
            start = time.perf_counter()
        if me == 0:
            reqs = (many("send", 0, peer, DATA_TAG, views, dom) if many
                    else [transport.post_send(0, peer, DATA_TAG, v, dom) for v in views])
            _wait(transport, *reqs)
            _wait(transport, transport.post_recv(0, peer, ACK_TAG, ack))
        else:
            reqs = (many("recv", 0, peer, DATA_TAG, views, dom) if many
                    else [transport.post_recv(0, peer, DATA_TAG, v, dom) for v in views])
            _wait(transport, *reqs)
            _wait(transport, transport.post_send(0, peer, ACK_TAG, b"done"))
    elapsed = time.perf_counter() - start
    return n * window * iters / elapsed / 1e9


def osu_latency(transport: Transport, peer: int, n: int, iters: int, device: bool, eager: bool = False) -> float:
    """Transport-layer one-way latency in microseconds (raw posts, RTT / 2).  ``eager``
    (device frames): eager sends and loanable receives (the protocol the messaging layer
    uses for small device frames) instead of plain posts (rendezvous)."""
    me = transport.rank
    dom = MemoryDomain.DEVICE if device else MemoryDomain.HOST
    sbuf = _region(transport, pattern(n), device)
    rbuf = _region(transport, bytes(n), device)
    sv, rv = _window(sbuf, device, n), _window(rbuf, device, n)
    send = transport.post_send_eager if eager else transport.post_send
    recv = transport.post_recv_loanable if eager else transport.post_recv

    def receive():
        req = recv(0, peer, PP_TAG, rv, dom)
        _wait(transport, req)
        if eager:
            transport.take_loan(req)  # dropped at once: the ring slot goes back

    warm = max(10, iters // 10)
    start = None
    for it in range(iters + warm):
        if it == warm:
            start = time.perf_counter()
        if me == 0:
            _wait(transport, send(0, peer, PP_TAG, sv, dom))
            receive()
        else:
            receive()
            _wait(transport, send(0, peer, PP_TAG, sv, dom))
    return (time.perf_counter() - start) / iters / 2 * 1e6


def pingpong(transport: Transport, peer: int, n: int, iters: int, device: bool, ns=None) -> dict:
    """Comm-path ping-pong through send_payload/recv_payload on the TaskLoop.

    ``ns`` (see ``storm.namespace_of``) selects whose comm stack runs: this
    package by default, or the reference package for the bench's reference arm."""
    if ns is None:
        ns = SimpleNamespace(TaskLoop=TaskLoop, MonotonicClock=MonotonicClock, build_comm_table=build_comm_table,
                             send_payload=send_payload, recv_payload=recv_payload, make_frame=make_frame)
    send_payload_, recv_payload_ = ns.send_payload, ns.recv_payload
    loop = ns.TaskLoop(ns.MonotonicClock())
    table = ns.build_comm_table(transport)
    channel = table.lookup(peer)
    if device:
        from ..transport.nvlink import CudaRegion

        frame = Frame(CudaRegion(pattern(n), transport.device), n, MemoryDomain.DEVICE)
    else:
        frame = ns.make_frame(pattern(n))
    warm = max(5, iters // 10)
    samples = []

    async def leader():
        for it in range(iters + warm):
            t0 = time.perf_counter()
            await send_payload_(transport, channel, 50, frame)
            echo = await recv_payload_(transport, channel, 51)
            if it >= warm:
                samples.append((time.perf_counter() - t0) / 2)
            if it == 0 and echo.to_bytes() != pattern(n):
                raise AssertionError("ping-pong echo differs")

    async def echo():
        for _ in range(iters + warm):
            got = await recv_payload_(transport, channel, 50)
            await send_payload_(transport, channel, 51, got)

    loop.run_until_complete(leader() if transport.rank == 0 else echo())
    if not samples:
        return {}
    samples.sort()
    mean = sum(samples) / len(samples)
    return {"mean_s": mean, "median_s": samples[len(samples) // 2], "p99_s": samples[int(len(samples) * 0.99) - 1],
            "throughput_Bps": 2 * n / (2 * mean)}
