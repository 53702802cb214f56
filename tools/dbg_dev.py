import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from nvlink_fixtures import nvlink_transports
from paper_2101_08878_b200.transport import MemoryDomain
from paper_2101_08878_b200.transport.nvlink import CudaRegion
ts = nvlink_transports(2, 0)
for n in (1, 1000, 1 << 20):
    src = CudaRegion(os.urandom(n), 0)
    dst = CudaRegion(n, 0)
    s = ts[0].post_send(0, 1, 5, src.window(), MemoryDomain.DEVICE)
    print("posted send", s, flush=True)
    r = ts[1].post_recv(0, 0, 5, dst.window(), MemoryDomain.DEVICE)
    print("posted recv", r, flush=True)
    t0 = time.time()
    while (s.pending or r.pending) and time.time() - t0 < 5:
        ts[0].progress(); ts[1].progress()
    print(n, s, r, ts[0].native_stats(), ts[1].native_stats(), flush=True)
    print("equal", dst.to_bytes() == src.to_bytes(), flush=True)
