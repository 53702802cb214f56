"""key_merge N=1 timing without the bench's parity gate (diagnostic variants may change
the digest): per-step ms and partition / join kernel ms (CUDA events), median of steps.

    python tools/km_time.py [--rows N] [--fraction F] [--steps K]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness.key_merge import KeyMerge  # noqa: E402
from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=100_000_000)
ap.add_argument("--fraction", type=float, default=0.3)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--tag", default="")
a = ap.parse_args()
km = KeyMerge(a.rows, a.fraction)
km.generate()
loop = TaskLoop(MonotonicClock())
for _ in range(3):
    digest = loop.run_until_complete(km.run())
km.timing = True
steps, parts, joins = [], [], []
for _ in range(a.steps):
    km.kernel_ms = {"partition": 0.0, "join": 0.0}
    t0 = time.perf_counter()
    loop.run_until_complete(km.run())
    steps.append((time.perf_counter() - t0) * 1e3)
    parts.append(km.kernel_ms["partition"])
    joins.append(km.kernel_ms["join"])
print(a.tag, "step_ms", round(statistics.median(steps), 3), "partition_ms", round(statistics.median(parts), 3),
      "join_ms", round(statistics.median(joins), 3), "digest", digest)
