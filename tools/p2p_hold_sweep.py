"""osu_bw (window 64, distinct buffers) at 4 / 8 / 16 MiB under the current M4D_PULL_BATCH (2 ranks, torchrun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness import p2p  # noqa: E402
from paper_2101_08878_b200.transport import TransportConfig, transport_init  # noqa: E402

rank = int(os.environ["RANK"])
t = transport_init(2, rank, TransportConfig(kind="nvlink", device=rank, connect_timeout=60))
t.wait_ready()
out = []
for n in (4 << 20, 8 << 20, 16 << 20):
    p2p.verify_once(t, 1 - rank, n, True)
    bws = [p2p.osu_bw(t, 1 - rank, n, 64, 4, True) for _ in range(5)]
    out.append(f"{n >> 20}MiB " + " ".join(f"{b:6.1f}" for b in bws))
launches = t.native_stats()["pull_kernel_launches"]
t.close()
if rank == 0:
    print(f"batch={os.environ.get('M4D_PULL_BATCH', '8')} launches(rank0)={launches} | " + " | ".join(out), flush=True)
