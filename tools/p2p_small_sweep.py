"""Device-frame osu_latency (and osu_bw from 64 KiB) at 1 B - 1 MiB under the current M4D_SMALL_PULL (2 ranks, torchrun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness import p2p  # noqa: E402
from paper_2101_08878_b200.transport import TransportConfig, transport_init  # noqa: E402

rank = int(os.environ["RANK"])
t = transport_init(2, rank, TransportConfig(kind="nvlink", device=rank, connect_timeout=60))
t.wait_ready()
out = []
for n in (1, 16384, 65536, 262144, 1048576, 4194304):
    p2p.verify_once(t, 1 - rank, n, True)
    lat = p2p.osu_latency(t, 1 - rank, n, 1000 if n < (1 << 20) else 100, True)
    bw = p2p.osu_bw(t, 1 - rank, n, 64, 10, True) if n >= 65536 else 0.0
    out.append(f"{n}B {lat:6.2f}us {bw:6.1f}GB/s")
t.close()
if rank == 0:
    print(f"lone_ce_max={os.environ.get("M4D_LONE_CE_MAX", "default")} | " + " ".join(out), flush=True)
