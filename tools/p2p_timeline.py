"""Where a 4 MiB osu_bw window goes: sender post loop vs. transfer vs. completion (2 ranks, torchrun)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness import p2p  # noqa: E402
from paper_2101_08878_b200.transport import MemoryDomain, TransportConfig, transport_init  # noqa: E402
from paper_2101_08878_b200.transport.nvlink import CudaRegion  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
t = transport_init(2, rank, TransportConfig(kind="nvlink", device=rank, connect_timeout=60))
t.wait_ready()
n, window = int(sys.argv[1]) if len(sys.argv) > 1 else 4 << 20, 64
buf = CudaRegion(n * window, rank)  # distinct region per message of the window
views = [buf.window(k * n, n) for k in range(window)]
ack = bytearray(4)
for it in range(6):
    t0 = time.perf_counter()
    if rank == 0:
        reqs = [t.post_send(0, 1, 77, v, MemoryDomain.DEVICE) for v in views]
        t1 = time.perf_counter()
        p2p._wait(t, *reqs)
        t2 = time.perf_counter()
        p2p._wait(t, t.post_recv(0, 1, 78, ack))
        t3 = time.perf_counter()
    else:
        reqs = [t.post_recv(0, 0, 77, v, MemoryDomain.DEVICE) for v in views]
        t1 = time.perf_counter()
        p2p._wait(t, *reqs)
        t2 = time.perf_counter()
        p2p._wait(t, t.post_send(0, 0, 78, b"done"))
        t3 = time.perf_counter()
    if it >= 2:
        print(f"rank {rank} post {1e6*(t1-t0):7.1f} us  complete {1e6*(t2-t1):7.1f} us  ack {1e6*(t3-t2):6.1f} us"
              f"  -> {n*window/(t3-t0)/1e9:6.1f} GB/s", flush=True)
t.close()
