"""Profiling driver: one key_merge step of an in-process world of W ranks on one GPU (for
ncu: the shuffle kernels at their multi-GPU sizes, peer writes landing in local HBM)."""
import argparse, os, sys, uuid
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness.key_merge import KeyMerge  # noqa: E402
from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop, gather  # noqa: E402
from paper_2101_08878_b200.transport import TransportConfig, transport_init  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=100_000_000)
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
session = "p" + uuid.uuid4().hex[:10]
ts = [transport_init(a.world, r, TransportConfig(kind="nvlink", session=session, device=0)) for r in range(a.world)]
for t in ts:
    t.wait_ready(10.0)
ranks = [KeyMerge(a.rows, 0.3, rank=r, world=a.world, device=0, transport=ts[r]) for r in range(a.world)]
for km in ranks:
    km.generate()
loop = TaskLoop(MonotonicClock())


async def main():
    return await gather(*(km.run_global() for km in ranks))


for _ in range(a.steps):
    print(loop.run_until_complete(main())[0])
for km in ranks:
    km.close()
for t in ts:
    t.close()
