"""Where does the receiver's time go in a 4 MB osu_bw window?  (2 processes, 2 GPUs)"""
import os, sys, time, uuid, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(rank, session, n, window, iters):
    from paper_2101_08878_b200.transport import TransportConfig, transport_init, MemoryDomain
    from paper_2101_08878_b200.transport.nvlink import CudaRegion
    from paper_2101_08878_b200.harness.p2p import _wait
    t = transport_init(2, rank, TransportConfig(kind="nvlink", session=session, device=rank, connect_timeout=30))
    t.wait_ready()
    buf = CudaRegion(n, rank)
    view = buf.window(0, n)
    ack = bytearray(4)
    rows = []
    for it in range(iters):
        t0 = time.perf_counter()
        if rank == 0:
            reqs = [t.post_send(0, 1, 7, view, MemoryDomain.DEVICE) for _ in range(window)]
            t1 = time.perf_counter()
            _wait(t, *reqs)
            _wait(t, t.post_recv(0, 1, 8, ack))
        else:
            reqs = [t.post_recv(0, 0, 7, view, MemoryDomain.DEVICE) for _ in range(window)]
            t1 = time.perf_counter()
            _wait(t, *reqs)
            _wait(t, t.post_send(0, 0, 8, b"done"))
        t2 = time.perf_counter()
        rows.append((t1 - t0, t2 - t0))
    post = sum(r[0] for r in rows[1:]) / (iters - 1)
    tot = sum(r[1] for r in rows[1:]) / (iters - 1)
    print(f"rank {rank} n={n} window={window}: post loop {post*1e6/window:.2f} us/msg, total {tot*1e6/window:.2f} us/msg, "
          f"{n*window/tot/1e9:.1f} GB/s", flush=True)
    # raw ctypes call cost
    if rank == 1:
        import ctypes
        from paper_2101_08878_b200 import native
        lib = native.lib()
        t0 = time.perf_counter()
        for _ in range(10000):
            lib.m4d_transport_mesh_ready(t._h)
        print(f"ctypes null call {(time.perf_counter()-t0)/10000*1e6:.2f} us", flush=True)
        from paper_2101_08878_b200.transport import TransferRequest
        t0 = time.perf_counter()
        for _ in range(10000):
            TransferRequest(t, "recv", 0, 0, 7, view, MemoryDomain.DEVICE)
        print(f"TransferRequest() {(time.perf_counter()-t0)/10000*1e6:.2f} us", flush=True)
        t0 = time.perf_counter()
        for _ in range(10000):
            t.progress()
        print(f"idle progress() {(time.perf_counter()-t0)/10000*1e6:.2f} us", flush=True)
    t.close()


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
    else:
        for n in (1 << 20, 4 << 20, 16 << 20):
            s = "pr" + uuid.uuid4().hex[:8]
            ps = [subprocess.Popen([sys.executable, __file__, str(r), s, str(n), "64", "10"]) for r in range(2)]
            for p in ps:
                p.wait()
