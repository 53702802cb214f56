#!/usr/bin/env python3
"""2-rank p2p sweep (osu_latency / osu_bw / comm-path ping-pong) on the nvlink transport.

    python tools/p2p_sweep.py [--device-frames] [--max-size 67108864]

Spawns two processes (rank r on GPU r when two GPUs are visible, else both on
GPU 0) and prints one JSON line per size from rank 0."""
import argparse
import json
import os
import subprocess
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank: int, session: str, args) -> None:
    from paper_2101_08878_b200 import native
    from paper_2101_08878_b200.harness import p2p
    from paper_2101_08878_b200.transport import TransportConfig, transport_init

    ngpu = native.device_count()
    device = (rank % ngpu) if (ngpu and not args.host) else -1
    t = transport_init(2, rank, TransportConfig(kind="nvlink", session=session, device=device, connect_timeout=30))
    t.wait_ready()
    dev = device >= 0
    peer = 1 - rank
    n = 1
    while n <= args.max_size:
        p2p.verify_once(t, peer, n, dev)
        lat_iters = 2000 if n <= 65536 else (300 if n <= (4 << 20) else 50)
        lat = p2p.osu_latency(t, peer, n, lat_iters, dev)
        bw = p2p.osu_bw(t, peer, n, 64, 20 if n <= (1 << 20) else 5, dev)
        pp = p2p.pingpong(t, peer, n, min(lat_iters, 1000), dev)
        if rank == 0:
            print(json.dumps({"size": n, "device": dev, "osu_latency_us": lat, "osu_bw_GBps": bw,
                              "pingpong_latency_us": pp["mean_s"] * 1e6, "pingpong_p99_us": pp["p99_s"] * 1e6,
                              "pingpong_GBps": pp["throughput_Bps"] / 1e9}), flush=True)
        n *= args.step
    if rank == 0:
        print(json.dumps({"stats": t.native_stats()}), flush=True)
    t.close()


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-size", type=int, default=64 << 20)
    ap.add_argument("--step", type=int, default=4)
    ap.add_argument("--host", action="store_true", help="host frames only (no GPU)")
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--session", default=None)
    args = ap.parse_args()
    if args.rank is not None:
        worker(args.rank, args.session, args)
        return 0
    session = "p2p" + uuid.uuid4().hex[:8]
    base = [sys.executable, os.path.abspath(__file__), "--max-size", str(args.max_size), "--step", str(args.step),
            "--session", session] + (["--host"] if args.host else [])
    procs = [subprocess.Popen(base + ["--rank", str(r)]) for r in range(2)]
    rcs = [p.wait() for p in procs]
    return max(rcs)


if __name__ == "__main__":
    sys.exit(main())
