"""One rank of a multi-process GPU parity test (test infrastructure; run as a script).

    python tests/mp_worker.py MODE RANK WORLD SESSION DEVMODE

MODE     ts        transpose_sum, 2048^2 fp64 / 256 blocks, peers' x pools mapped through
                   CUDA IPC (harness/transpose_sum.py connect_peers), checked against the oracle
         ts_fence  the same with x re-uploaded from host memory before every step through
                   TransposeSum.load_x, alternating two different arrays
         km_push   key_merge with the fused owner-scatter push shuffle (peers' receive buffers
                   mapped through CUDA IPC), digest checked against the oracle
         km_pull   key_merge with the rendezvous pull shuffle (device frames of the transport)
         frames    device frames of many sizes both ways through the transport, bit-exact
         churn     150 freshly allocated device frames sent and freed: no exporter memory leak
         torch     torch tensors through Endpoint.write/read as zero-copy device array frames
DEVMODE  same      every rank on cuda:0 (one B200: still separate processes, so IPC)
         own       rank r on cuda:r (NVLink between B200s)

Prints one JSON line ``{"rank": r, "ok": true, ...}``; exits non-zero on any mismatch.
"""

import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2101_08878_b200 import native  # noqa: E402
from paper_2101_08878_b200.harness.collectives import allgather_sync  # noqa: E402
from paper_2101_08878_b200.transport import TransportConfig, transport_init  # noqa: E402


def transport(rank, world, session, device):
    t = transport_init(world, rank, TransportConfig(kind="nvlink", session=session, device=device,
                                                    connect_timeout=60))
    t.wait_ready(60.0)
    return t


def run_ts(t, rank, world, device, fenced):
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    tags = iter(range(920, 10**9))
    n, b = 2048, 256
    ts = TransposeSum(n, b, rank=rank, world=world, device=device,
                      exchange=lambda blob: allgather_sync(t, blob, next(tags))).setup()
    _, want = oracle.transpose_sum_checksum(n, b, threads=4)
    res = ts.step()
    assert res.checksum == want or abs(res.checksum - want) <= 1e-12 * abs(want), (res.checksum, want)
    assert ts.tasks_single > 0  # some partner tiles are read out of a peer's pool
    nb = n // b
    for g in ts.owned[:: max(1, len(ts.owned) // 6)]:
        i, j = divmod(g, nb)
        y = np.frombuffer(ts.read_y_block(g), dtype=np.float64).reshape(b, b)
        a = oracle.gen_block_c(n, i * b, j * b, b)
        bt = oracle.gen_block_c(n, j * b, i * b, b)
        assert np.array_equal(y, oracle.transpose_block_c(a, bt)), g
    out = {"checksum": res.checksum, "remote_tasks": ts.tasks_single}
    if fenced:
        # two host copies of this rank's pool: x (seed A) and x' (seed B), alternated
        pool = len(ts.owned) * ts.block_bytes
        hosts = []
        sums = []
        for seed in (oracle.SEED_X, oracle.SEED_X + 1):
            ts.seed = seed
            ts.generate()
            h = native.PinnedHostBuffer(pool)
            native.memcpy(h.ptr, ts.x.ptr, pool, ts.stream)
            ts.stream.synchronize()
            hosts.append(h)
            sums.append(oracle.transpose_sum_checksum(n, b, seed=seed, threads=4)[1])
        for step in range(6):
            k = step % 2
            ts.load_x(hosts[k].ptr)
            got = ts.step().checksum
            assert abs(got - sums[k]) <= 1e-12 * abs(sums[k]), (step, got, sums[k])
        out["fenced_steps"] = 6
        for h in hosts:
            h.free()
    ts.close()
    return out


def run_km(t, rank, world, device, shuffle):
    from paper_2101_08878_b200.harness.key_merge import KeyMerge
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop

    rows = 200_000
    km = KeyMerge(rows, 0.3, rank=rank, world=world, device=device, transport=t, shuffle=shuffle)
    km.generate()
    loop = TaskLoop(MonotonicClock())
    want = oracle.key_merge_c(rows, world, 0.3)
    got = None
    for _ in range(3):  # repeated steps reuse the mapped buffers
        got = loop.run_until_complete(km.run_global())
        assert got == want, (got, want)
    assert getattr(km, "conserved", False)
    out = {"digest": list(got), "received": km.received, "mapped_peers": len(km._imported)}
    km.close()
    return out


def run_frames(t, rank, world, device):
    from paper_2101_08878_b200.transport import MemoryDomain
    from paper_2101_08878_b200.transport.base import DeviceView

    assert world == 2
    peer = 1 - rank
    sizes = [1, 7, 4096, 65536, 1 << 20, (4 << 20) + 3, 16 << 20]
    cap = max(sizes)
    send = native.DeviceBuffer(device, cap)
    recv = native.DeviceBuffer(device, cap)
    for i, n in enumerate(sizes):
        pattern = ((np.arange(n, dtype=np.uint64) * (2 * i + 3 + rank)) % 251).astype(np.uint8)
        native.memcpy(send.ptr, pattern.ctypes.data, n)
        native.check(native.lib().m4d_device_sync(device))
        rq = t.post_recv(0, peer, 500 + i, DeviceView(recv.ptr, n, device), MemoryDomain.DEVICE)
        sq = t.post_send(0, peer, 500 + i, DeviceView(send.ptr, n, device), MemoryDomain.DEVICE)
        while rq.pending or sq.pending:
            t.progress()
        assert not rq.failed and not sq.failed, (rq.error, sq.error)
        got = np.frombuffer(native.to_host(recv.ptr, n), dtype=np.uint8)
        want = ((np.arange(n, dtype=np.uint64) * (2 * i + 3 + peer)) % 251).astype(np.uint8)
        assert np.array_equal(got, want), n
    stats = t.native_stats()
    return {"sizes": len(sizes), "staged": t.metrics.staging_copies, "pulls": stats["rendezvous_pulls"]}


def run_churn(t, rank, world, device):
    """Rank 0 sends 150 freshly allocated 8 MiB device frames (freed after each send),
    rank 1 receives them; rank 0's free device memory must come back (the receiver closes
    each CUDA-IPC mapping before the exporter's cudaFree, transport.cpp release_exported)."""
    from paper_2101_08878_b200.transport import MemoryDomain
    from paper_2101_08878_b200.transport.base import DeviceView
    from paper_2101_08878_b200.transport.nvlink import CudaRegion

    n, frames = 8 << 20, 150
    recv = native.DeviceBuffer(device, n)
    allgather_sync(t, b"\x00", 980)
    before = native.mem_get_info(device)[0]
    for i in range(frames):
        if rank == 0:
            region = CudaRegion(n, device)
            native.check(native.lib().m4d_memset(region.ptr, i % 251, n, None))
            req = t.post_send(0, 1, 600, region.window(), MemoryDomain.DEVICE)
        else:
            req = t.post_recv(0, 0, 600, DeviceView(recv.ptr, n, device), MemoryDomain.DEVICE)
        while req.pending:
            t.progress()
        assert not req.failed, req.error
        if rank == 0:
            del region, req
        else:
            assert native.to_host(recv.ptr + n - 1, 1)[0] == i % 251
    allgather_sync(t, b"\x00", 981)  # drives both sides' progress: unmaps and their answers
    for _ in range(100):
        t.progress()
    allgather_sync(t, b"\x00", 982)
    after = native.mem_get_info(device)[0]
    return {"frames": frames, "leak_mib": (before - after) / 2**20}


def run_torch(t, rank, world, device):
    """Torch tensors (caching-allocator memory, several sharing one allocator segment)
    written by rank 0 through Endpoint.write as array_frames (zero-copy device frames,
    serializer tag 3) and read by rank 1 as CUDA arrays on its own device."""
    import torch

    from paper_2101_08878_b200.channels import build_comm_table
    from paper_2101_08878_b200.endpoints import Node, connect, listen
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop, sleep
    from paper_2101_08878_b200.messaging import Message, array_frames, frames_to_array

    torch.cuda.set_device(device)
    specs = [(torch.float32, (1,)), (torch.int64, (1000,)), (torch.float32, (250_000,)), (torch.float64, (3, 1_000_000)),
             (torch.int16, (7, 5))]
    node = Node(t, build_comm_table(t))
    loop = TaskLoop(MonotonicClock())
    got = []

    def expect(i, dtype, shape):
        n = 1
        for d in shape:
            n *= d
        return (torch.arange(n, device=f"cuda:{device}", dtype=torch.int64) * (i + 3) % 997).to(dtype).reshape(shape)

    async def main():
        if rank == 0:
            ep = await connect(node, "mpi://1")
            tensors = [expect(i, dt, sh) for i, (dt, sh) in enumerate(specs)]  # caching-allocator blocks
            for x in tensors:
                await ep.write(Message(array_frames(x)))
            await ep.read()  # the reader's "done"
            await ep.close()
        else:
            done = []

            async def handler(ep):
                for i, (dt, sh) in enumerate(specs):
                    msg = await ep.read()
                    arr = frames_to_array(msg.frames)
                    y = arr.to_torch()
                    assert y.device.index == device and y.dtype == dt and tuple(y.shape) == sh, (y.device, y.dtype, y.shape)
                    assert y.data_ptr() == arr.region.ptr  # zero copy: the tensor is the received region
                    assert torch.equal(y, expect(i, dt, sh)), i
                    got.append(tuple(sh))
                from paper_2101_08878_b200.messaging import make_frame
                await ep.write(Message([make_frame("done", 1)]))
                done.append(True)

            await listen(node, "mpi://1", handler).start()
            while not done:
                await sleep(0)

    loop.run_until_complete(main())
    return {"tensors": len(specs) if rank == 0 else len(got), "staged": t.metrics.staging_copies}


def main() -> int:
    mode, rank, world, session, devmode = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    device = rank if devmode == "own" else 0
    native.set_device(device)
    t = transport(rank, world, session, device)
    if mode in ("ts", "ts_fence"):
        out = run_ts(t, rank, world, device, mode == "ts_fence")
    elif mode in ("km_push", "km_pull"):
        out = run_km(t, rank, world, device, mode[3:])
    elif mode == "frames":
        out = run_frames(t, rank, world, device)
    elif mode == "churn":
        out = run_churn(t, rank, world, device)
    elif mode == "torch":
        out = run_torch(t, rank, world, device)
    else:
        raise SystemExit(f"unknown mode {mode}")
    allgather_sync(t, b"\x00", 990)  # nobody closes while a peer still reads its memory
    t.close()
    print(json.dumps({"rank": rank, "ok": True, **out}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
