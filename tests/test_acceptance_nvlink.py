"""SPEC.md acceptance criteria (lines 526-536 of the reference) exercised on the
B200 transport: end-to-end identity across chunk sizes, domains and progress
modes; isolation soak with many endpoints per pair and identical tags;
deadlock freedom of a 16-task symmetric exchange; heartbeat liveness during a
bulk chunked transfer (control/data isolation); and
socket wire interop with the unmodified reference (N4)."""

import os
import random
import socket
import subprocess
import sys
import textwrap
import time

import pytest

from nvlink_fixtures import close_all, nvlink_nodes, nvlink_transports, nvlink_world
from paper_2101_08878_b200.endpoints import Endpoint
from paper_2101_08878_b200.harness import storm
from paper_2101_08878_b200.loop import gather, sleep
from paper_2101_08878_b200.messaging import (
    Frame,
    Message,
    ProgressMode,
    make_frame,
    read_message,
    recv_payload,
    send_payload,
    set_progress_mode,
    write_message,
)
from paper_2101_08878_b200.transport import MemoryDomain

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
DEVICES = [pytest.param(-1, id="host"), pytest.param(0, id="cuda", marks=pytest.mark.gpu)]


def _frame(payload: bytes, device: int, k: int) -> Frame:
    if device >= 0 and k % 2:
        from paper_2101_08878_b200.transport.nvlink import CudaRegion

        return Frame(CudaRegion(payload, device), len(payload), MemoryDomain.DEVICE)
    return make_frame(payload)


def _corpus(seed: int, max_size: int, device: int) -> list[Message]:
    rng = random.Random(seed)
    out = []
    for i in range(10):
        frames = []
        for k in range(rng.randrange(0, 9)):  # 0-8 frames per message
            size = min(max_size, int(2 ** rng.uniform(0, 22)) if rng.random() < 0.9 else 0)
            frames.append(_frame(rng.randbytes(size), device, i + k))
        out.append(Message(frames))
    return out


@pytest.mark.parametrize("device", DEVICES)
@pytest.mark.parametrize("max_chunk,max_size", [(17, 3000), (64 * 1024, 1 << 20), (1 << 20, 4 << 20)])
@pytest.mark.parametrize("mode", ["cooperative", "periodic"])
def test_end_to_end_identity(device, max_chunk, max_size, mode):
    """Randomised corpus (0-8 frames, 0 B - 4 MiB, both domains) survives write/read
    byte-identically for every chunk size and progress mode."""
    corpus = _corpus(max_chunk ^ max_size, max_size, device)
    loop, ts, tables = nvlink_world(2, device)
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
    got = []

    async def main():
        if mode == "periodic":
            for t in ts:
                set_progress_mode(t, ProgressMode.periodic(0.0002))

        async def writer():
            for m in corpus:
                await write_message(ts[0], ch0, m, max_chunk=max_chunk)

        async def reader():
            for _ in corpus:
                got.append(await read_message(ts[1], ch1, max_chunk=max_chunk))

        await gather(writer(), reader())
        for t in ts:
            set_progress_mode(t, ProgressMode.cooperative())

    try:
        loop.run_until_complete(main())
    finally:
        close_all(ts)
    for want, have in zip(corpus, got):
        assert [f.to_bytes() for f in have.frames] == [f.to_bytes() for f in want.frames]
        assert [f.domain for f in have.frames] == [f.domain for f in want.frames]


def test_isolation_soak_four_ranks_eight_endpoints_per_pair():
    """4 ranks, 8 endpoints per ordered pair, identical tags on every endpoint,
    interleaved writers/readers: zero cross-talk, zero loss."""
    ts = nvlink_transports(4)
    try:
        r = storm.run_local(storm.namespace_of("paper_2101_08878_b200"), ts, conns=8, total=6000, rounds=2)
    finally:
        close_all(ts)
    assert r.frames == 12000 and r.verified == 6000


def test_sixteen_task_symmetric_exchange_completes():
    """16 concurrent tasks on one executor exchanging symmetric payloads, cooperative
    mode: no busy-wait deadlock (the §IV-B scenario negated)."""
    loop, ts, tables = nvlink_world(4)

    async def pair(a, b, tag):
        ca, cb = tables[a].lookup(b), tables[b].lookup(a)
        got = await gather(send_payload(ts[a], ca, tag, make_frame(bytes([a]) * 3000)),
                           recv_payload(ts[a], ca, tag + 1),
                           send_payload(ts[b], cb, tag + 1, make_frame(bytes([b]) * 3000)),
                           recv_payload(ts[b], cb, tag))
        return got[1].to_bytes()[:1] + got[3].to_bytes()[:1]

    async def main():
        jobs = [pair(a, b, 100 + 2 * k) for k, (a, b) in enumerate([(0, 1), (2, 3), (0, 2), (1, 3)])]
        return await gather(*jobs)  # 4 pairs x 4 operations = 16 tasks

    try:
        out = loop.run_until_complete(main())
    finally:
        close_all(ts)
    assert out == [bytes([1, 0]), bytes([3, 2]), bytes([2, 0]), bytes([3, 1])]


@pytest.mark.parametrize("device", DEVICES)
def test_heartbeat_stays_live_during_bulk_chunked_transfer(device):
    """A heartbeat endpoint keeps beating (no gap > 3 intervals) while a 64 MiB frame
    moves in 64 KiB chunks on another channel of the same pair."""
    loop, nodes = nvlink_nodes(2, device, max_chunk=64 * 1024)
    ts = [n.transport for n in nodes]
    chan = [nodes[0].table.duplicate(1, generation=1), nodes[1].table.duplicate(0, generation=1)]
    beat_tx = Endpoint(nodes[0], chan[0], 1, "connector", 1)
    beat_rx = Endpoint(nodes[1], chan[1], 0, "listener", 1)
    bulk = os.urandom(64 << 20)
    if device >= 0:
        from paper_2101_08878_b200.transport.nvlink import CudaRegion

        frame = Frame(CudaRegion(bulk, device), len(bulk), MemoryDomain.DEVICE)
    else:
        frame = make_frame(bulk)
    interval = 0.002
    state = {"done": False, "gaps": [], "beats": 0}

    async def bulk_tx():
        await send_payload(ts[0], nodes[0].table.lookup(1), 500, frame, max_chunk=64 * 1024)

    async def bulk_rx():
        got = await recv_payload(ts[1], nodes[1].table.lookup(0), 500, max_chunk=64 * 1024)
        state["done"] = True
        return got

    async def beater():
        k = 0
        while not state["done"]:
            await beat_tx.write(Message([make_frame(k.to_bytes(8, "little"))]))
            k += 1
            until = time.monotonic() + interval
            while time.monotonic() < until:
                await sleep(0)
        await beat_tx.write(Message([make_frame((2**64 - 1).to_bytes(8, "little"))]))

    async def monitor():
        last = time.monotonic()
        while True:
            msg = await beat_rx.read()
            now = time.monotonic()
            state["gaps"].append(now - last)
            last = now
            if int.from_bytes(msg.frames[0].to_bytes(), "little") == 2**64 - 1:
                return
            state["beats"] += 1

    async def main():
        out = await gather(bulk_tx(), bulk_rx(), beater(), monitor())
        return out[1]

    try:
        got = loop.run_until_complete(main())
    finally:
        close_all(ts)
    assert got.to_bytes() == bulk
    assert state["beats"] >= 1
    missed = [g for g in state["gaps"] if g > 3 * interval + 0.05]  # 50 ms slack for a loaded CI host
    assert not missed, f"heartbeat gaps {missed[:5]}"


INTEROP = textwrap.dedent('''
    import sys
    impl, root, ref, rank, p0, p1 = sys.argv[1:7]
    rank = int(rank)
    if impl == "ref":
        sys.path.insert(0, ref)
        import commshim
        assert commshim.__file__.startswith(ref), commshim.__file__
        pkg = "commshim"
    else:
        sys.path.insert(0, root)
        pkg = "paper_2101_08878_b200"
    import importlib
    tr = importlib.import_module(pkg + ".transport")
    ch = importlib.import_module(pkg + ".channels")
    msg = importlib.import_module(pkg + ".messaging")
    lp = importlib.import_module(pkg + ".loop")
    rm = {0: ("127.0.0.1", int(p0)), 1: ("127.0.0.1", int(p1))}
    t = tr.transport_init(2, rank, tr.TransportConfig(kind="socket", rank_map=rm, connect_timeout=30.0))
    t.wait_ready(30.0)
    table = ch.build_comm_table(t)
    c = table.lookup(1 - rank)
    loop = lp.TaskLoop(lp.MonotonicClock())
    sizes = [0, 1, 17, 4096, 100000, 3 << 20]
    async def main():
        for i, n in enumerate(sizes):
            body = bytes((i * 31 + k) & 255 for k in range(min(n, 4096))) * (n // 4096 + 1)
            body = body[:n]
            if rank == 0:
                await msg.write_message(t, c, msg.Message([msg.make_frame(body), msg.make_frame("x%d" % i, 1)]),
                                        max_chunk=65536)
                echo = await msg.read_message(t, c, max_chunk=65536)
                assert echo.frames[0].to_bytes() == body and echo.decode()[1] == "x%d" % i, i
            else:
                m = await msg.read_message(t, c, max_chunk=65536)
                assert m.frames[0].to_bytes() == body, i
                await msg.write_message(t, c, m, max_chunk=65536)
    loop.run_until_complete(main())
    import time
    time.sleep(0.2)
    t.close()
    print("OK", impl, rank)
''')


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("impls", [("ours", "ref"), ("ref", "ours")], ids=["ours-rank0", "ref-rank0"])
def test_socket_wire_interop_with_the_reference(impls):
    """This package's socket transport and the unmodified reference's talk to each
    other: same M4D1 frames, hello, message headers and chunking."""
    if not os.path.isdir(os.path.join(REF, "commshim")):
        pytest.skip("baseline/_ref not installed")
    ports = [str(_free_port()), str(_free_port())]
    procs = [subprocess.Popen([sys.executable, "-c", INTEROP, impls[r], ROOT, REF, str(r), *ports],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    for p in procs:
        try:
            out, _ = p.communicate(timeout=120)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        assert p.returncode == 0 and "OK" in out, out[-3000:]
