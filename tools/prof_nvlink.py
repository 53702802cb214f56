"""Profiling driver for ncu NVLink counters: the kernels that move bytes between two B200s,
run with both ranks in ONE process on cuda:0 and cuda:1 (peer access enabled, so ncu
sees a single process; kernels run serialised under ncu).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
nvltx__bytes.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
        python tools/prof_nvlink.py [km|ts|p2p]

km : key_merge, 1e8 rows/side/GPU, push shuffle (m4d_partition_owner_push writes peer HBM)
ts : transpose_sum 40000^2 / 2000, 2 ranks (ts_kernel_tma reads partner tiles over NVLink)
p2p: 8 x 4 MiB device frames cuda:0 -> cuda:1 through the transport (pull kernel)
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2101_08878_b200 import native  # noqa: E402


def enable_peers():
    native.check(native.lib().m4d_enable_peer(0, 1))
    native.check(native.lib().m4d_enable_peer(1, 0))


def km(rows=100_000_000):
    from paper_2101_08878_b200.harness.key_merge import KeyMerge
    from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop, gather
    from paper_2101_08878_b200.transport import TransportConfig, transport_init
    import uuid

    session = "pn" + uuid.uuid4().hex[:8]
    ts = [transport_init(2, r, TransportConfig(kind="nvlink", session=session, device=r)) for r in range(2)]
    for t in ts:
        t.wait_ready(10)
    ranks = [KeyMerge(rows, 0.3, rank=r, world=2, device=r, transport=ts[r]) for r in range(2)]
    for k in ranks:
        k.generate()
    loop = TaskLoop(MonotonicClock())
    for _ in range(2):
        print(loop.run_until_complete(gather(*(k.run_global() for k in ranks))))
    for k in ranks:
        k.close()
    for t in ts:
        t.close()


def ts():
    from paper_2101_08878_b200.harness.transpose_sum import TransposeSum

    ranks = TransposeSum.local_world(40000, 2000, 2, devices=[0, 1])
    for _ in range(2):
        for r in ranks:
            r.launch()
        for r in ranks:
            r.stream.synchronize()
    print("ts ok", sum(r.tasks_single for r in ranks))


def p2p(n=4 << 20, window=8):
    import uuid

    from paper_2101_08878_b200.transport import MemoryDomain, TransportConfig, transport_init
    from paper_2101_08878_b200.transport.base import DeviceView

    session = "pp" + uuid.uuid4().hex[:8]
    ts_ = [transport_init(2, r, TransportConfig(kind="nvlink", session=session, device=r)) for r in range(2)]
    for t in ts_:
        t.wait_ready(10)
    src = native.DeviceBuffer(0, n * window)
    dst = native.DeviceBuffer(1, n * window)
    for _ in range(2):
        rq = [ts_[1].post_recv(0, 0, 7, DeviceView(dst.ptr + k * n, n, 1), MemoryDomain.DEVICE) for k in range(window)]
        sq = [ts_[0].post_send(0, 1, 7, DeviceView(src.ptr + k * n, n, 0), MemoryDomain.DEVICE) for k in range(window)]
        while any(r.pending for r in rq + sq):
            for t in ts_:
                t.progress()
    print("p2p ok", ts_[1].native_stats()["pull_kernel_launches"])
    for t in ts_:
        t.close()


if __name__ == "__main__":
    if native.device_count() < 2:
        raise SystemExit("needs two GPUs")
    enable_peers()
    {"km": km, "ts": ts, "p2p": p2p}[sys.argv[1] if len(sys.argv) > 1 else "km"]()
