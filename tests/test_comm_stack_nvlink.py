"""The comm stack (messaging framing, endpoints, progress modes, asyncio bridge)
running on the nvlink transport: host-only contexts in the CPU suite, cuda:0
(device frames moved device-to-device) in the gpu suite."""

import asyncio
import os
import random
import subprocess
import sys
import textwrap

import pytest

from paper_2101_08878_b200.endpoints import connect, listen
from paper_2101_08878_b200.errors import EndOfStream
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

from nvlink_fixtures import close_all, new_session, nvlink_nodes, nvlink_world

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEVICES = [pytest.param(-1, id="host"), pytest.param(0, id="cuda", marks=pytest.mark.gpu)]


def device_frame(payload: bytes, device: int) -> Frame:
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    region = CudaRegion(payload, device)
    return Frame(region, len(payload), MemoryDomain.DEVICE)


@pytest.mark.parametrize("device", DEVICES)
def test_symmetric_payload_exchange(device):
    loop, ts, tables = nvlink_world(2, device)
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)

    async def side(t, ch, payload):
        _, frame = await gather(send_payload(t, ch, 40, make_frame(payload)), recv_payload(t, ch, 40))
        return frame.to_bytes()

    async def main():
        return await gather(side(ts[0], ch0, b"from-zero"), side(ts[1], ch1, b"from-one!"))

    try:
        assert loop.run_until_complete(main()) == [b"from-one!", b"from-zero"]
    finally:
        close_all(ts)


@pytest.mark.parametrize("device", DEVICES)
def test_messages_with_chunking_serializers_and_order(device):
    loop, ts, tables = nvlink_world(2, device)
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
    rng = random.Random(99)
    msgs = []
    for i in range(12):
        frames = [make_frame(rng.randbytes(rng.randrange(0, 5000))) for _ in range(rng.randrange(0, 4))]
        frames.append(make_frame(f"msg {i} héllo", 1))
        frames.append(make_frame([1.5 * i, -2.25], 2))
        msgs.append(Message(frames))

    async def main():
        got = []

        async def writer():
            for m in msgs:
                await write_message(ts[0], ch0, m, max_chunk=777)

        async def reader():
            for _ in msgs:
                got.append(await read_message(ts[1], ch1, max_chunk=777))

        await gather(writer(), reader())
        return got

    try:
        got = loop.run_until_complete(main())
        for want, have in zip(msgs, got):
            assert [f.to_bytes() for f in have.frames] == [f.to_bytes() for f in want.frames]
            assert have.decode()[-2] == want.decode()[-2]
    finally:
        close_all(ts)


@pytest.mark.parametrize("device", DEVICES)
def test_cooperative_and_periodic_modes_deliver_identical_bytes(device):
    rng = random.Random(7)
    corpus = [Message([make_frame(rng.randbytes(rng.randrange(0, 3000))) for _ in range(rng.randrange(0, 4))])
              for _ in range(5)]

    def run(mode):
        loop, ts, tables = nvlink_world(2, device)
        ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
        got = []

        async def main():
            set_progress_mode(ts[0], mode)
            set_progress_mode(ts[1], mode)

            async def writer():
                for m in corpus:
                    await write_message(ts[0], ch0, m, max_chunk=500)

            async def reader():
                for _ in corpus:
                    got.append(await read_message(ts[1], ch1, max_chunk=500))

            await gather(writer(), reader())
            set_progress_mode(ts[0], ProgressMode.cooperative())
            set_progress_mode(ts[1], ProgressMode.cooperative())

        try:
            loop.run_until_complete(main())
        finally:
            close_all(ts)
        return [[f.to_bytes() for f in m.frames] for m in got]

    assert run(ProgressMode.cooperative()) == run(ProgressMode.periodic(0.0005))


@pytest.mark.parametrize("device", DEVICES)
def test_endpoints_handshake_agreement_all_pairs(device):
    n = 4
    loop, nodes = nvlink_nodes(n, device)
    server_side = {}

    def handler_for(rank):
        async def handler(ep):
            server_side[(rank, ep.connection_id)] = ep
        return handler

    async def main():
        for node in nodes:
            await listen(node, f"mpi://{node.rank}", handler_for(node.rank)).start()
        dials = [(c, l) for c in range(n) for l in range(n) if c != l]
        random.Random(n * 1771).shuffle(dials)
        client = []
        for c, l in dials:
            client.append((l, await connect(nodes[c], f"mpi://{l}")))
        for _ in range(20):
            await sleep(0)
        for l, ep in client:
            assert server_side[(l, ep.connection_id)].channel.id == ep.channel.id
        assert len({ep.channel.id for _, ep in client}) == len(client)

    try:
        loop.run_until_complete(main())
    finally:
        close_all([nd.transport for nd in nodes])


@pytest.mark.parametrize("device", DEVICES)
def test_endpoint_streams_isolated_and_closed_cleanly(device):
    loop, nodes = nvlink_nodes(2, device)
    rng = random.Random(4242)
    streams, per_stream = 4, 12
    server_data = {}

    async def handler(ep):
        got = []
        try:
            while True:
                got.append((await ep.read()).frames[0].to_bytes())
        except EndOfStream:
            server_data[ep.connection_id] = got
            await ep.close()

    async def main():
        await listen(nodes[0], "mpi://0", handler).start()
        eps = [await connect(nodes[1], "mpi://0") for _ in range(streams)]

        async def writer(index, ep):
            for seq in range(per_stream):
                await ep.write(Message([make_frame(bytes([seq]) + bytes([index]) * rng.randrange(1, 600))]))
            await ep.close()

        await gather(*(writer(i, ep) for i, ep in enumerate(eps)))
        for _ in range(100000):
            if len(server_data) == streams and all(ep._released for ep in eps):
                break
            await sleep(0)
        assert len(server_data) == streams
        for index, ep in enumerate(eps):
            blobs = server_data[ep.connection_id]
            assert [b[0] for b in blobs] == list(range(per_stream))
            assert all(set(b[1:]) == {index} for b in blobs)
        assert all(ep._released for ep in eps)

    try:
        loop.run_until_complete(main())
    finally:
        close_all([nd.transport for nd in nodes])


def test_asyncio_bridge_runs_the_same_coroutines():
    """north_star: Comm.write/Comm.read as coroutines on asyncio."""
    from nvlink_fixtures import nvlink_transports
    from paper_2101_08878_b200.channels import build_comm_table

    ts = nvlink_transports(2, -1)
    tables = [build_comm_table(t) for t in ts]

    async def main():
        ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
        msg = Message([make_frame(b"over asyncio"), make_frame("ok", 1)])
        _, got = await asyncio.gather(write_message(ts[0], ch0, msg), read_message(ts[1], ch1))
        return got.decode()

    try:
        assert asyncio.run(main()) == [b"over asyncio", "ok"]
    finally:
        close_all(ts)


@pytest.mark.gpu
def test_device_frames_move_device_to_device_without_staging():
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    loop, ts, tables = nvlink_world(2, 0)
    ch0, ch1 = tables[0].lookup(1), tables[1].lookup(0)
    payloads = [os.urandom(n) for n in (1, 1000, 1 << 20, (8 << 20) + 3)]

    async def main():
        got = []
        for p in payloads:
            _, frame = await gather(send_payload(ts[0], ch0, 42, device_frame(p, 0)), recv_payload(ts[1], ch1, 42))
            got.append(frame)
        return got

    try:
        frames = loop.run_until_complete(main())
        for p, f in zip(payloads, frames):
            assert f.domain == MemoryDomain.DEVICE and isinstance(f.data, CudaRegion)
            assert f.to_bytes() == p
        for t in ts:
            assert t.metrics.staged_bytes == 0 and t.metrics.staging_copies == 0
        assert ts[1].native_stats()["nvlink_bytes"] == sum(len(p) for p in payloads)
    finally:
        close_all(ts)


@pytest.mark.gpu
def test_device_truncation_fails_both_sides():
    from nvlink_fixtures import nvlink_transports, pump
    from paper_2101_08878_b200.errors import TruncationError
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    ts = nvlink_transports(2, 0)
    try:
        src = CudaRegion(b"x" * 64, 0)
        dst = CudaRegion(16, 0)
        s = ts[0].post_send(0, 1, 5, src.window(), MemoryDomain.DEVICE)
        r = ts[1].post_recv(0, 0, 5, dst.window(), MemoryDomain.DEVICE)
        pump(ts, s, r)
        assert isinstance(r.error, TruncationError) and isinstance(s.error, TruncationError)
    finally:
        close_all(ts)


@pytest.mark.gpu
def test_mixed_domains_device_to_host_and_host_to_device():
    from nvlink_fixtures import nvlink_transports, pump
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    ts = nvlink_transports(2, 0)
    try:
        p = os.urandom(300000)
        host = bytearray(len(p))
        s = ts[0].post_send(0, 1, 6, CudaRegion(p, 0).window(), MemoryDomain.DEVICE)
        r = ts[1].post_recv(0, 0, 6, host)
        pump(ts, s, r)
        assert bytes(host) == p
        dev = CudaRegion(len(p), 0)
        s = ts[1].post_send(0, 0, 7, p)
        r = ts[0].post_recv(0, 1, 7, dev.window(), MemoryDomain.DEVICE)
        pump(ts, s, r)
        assert dev.to_bytes() == p
    finally:
        close_all(ts)


WORKER = textwrap.dedent('''
    import os, sys, random
    sys.path.insert(0, sys.argv[1])
    from paper_2101_08878_b200.channels import build_comm_table
    from paper_2101_08878_b200.endpoints import Node, connect, listen
    from paper_2101_08878_b200.errors import EndOfStream
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop
    from paper_2101_08878_b200.messaging import Frame, Message, make_frame
    from paper_2101_08878_b200.transport import MemoryDomain, TransportConfig, transport_init
    rank, session, device = int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
    t = transport_init(2, rank, TransportConfig(kind="nvlink", session=session, device=device, connect_timeout=20))
    t.wait_ready()
    node = Node(t, build_comm_table(t))
    loop = TaskLoop(MonotonicClock())
    rng = random.Random(1234)
    sizes = [int(2 ** rng.uniform(0, 22)) for _ in range(60)]
    def frame_for(i, n):
        body = bytes([(i * 7 + k) % 251 for k in range(min(n, 4096))]) * (n // 4096 + 1)
        body = body[:n]
        if device >= 0 and i % 2:
            from paper_2101_08878_b200.transport.nvlink import CudaRegion
            return Frame(CudaRegion(body, device), n, MemoryDomain.DEVICE)
        return make_frame(body)
    async def main():
        if rank == 0:
            done = []
            async def handler(ep):
                for i, n in enumerate(sizes):
                    msg = await ep.read()
                    assert msg.frames[0].to_bytes() == frame_for(i, n).to_bytes(), i
                    await ep.write(Message([make_frame(str(i), 1)]))
                try:
                    await ep.read()
                except EndOfStream:
                    done.append(True)
                await ep.close()
            await listen(node, "mpi://0", handler).start()
            from paper_2101_08878_b200.loop import sleep
            while not done:
                await sleep(0)
        else:
            ep = await connect(node, "mpi://0")
            for i, n in enumerate(sizes):
                await ep.write(Message([frame_for(i, n)]))
                assert (await ep.read()).decode() == [str(i)]
            await ep.close()
            from paper_2101_08878_b200.loop import sleep
            while not ep._released:
                await sleep(0)
    loop.run_until_complete(main())
    print("rank", rank, "ok", t.native_stats())
    t.close()
''')


def run_two_processes(device):
    session = new_session()
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, ROOT, str(r), session, str(device)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=180)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append((p.returncode, out))
    for rc, out in outs:
        assert rc == 0, out[-3000:]
    return outs


def test_two_processes_endpoint_ping_pong_host():
    run_two_processes(-1)


@pytest.mark.gpu
def test_two_processes_endpoint_ping_pong_device_frames_cuda_ipc():
    outs = run_two_processes(0)
    assert any("'rendezvous_pulls': 0" not in out for _, out in outs)
