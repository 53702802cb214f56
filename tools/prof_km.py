"""Profiling driver: one key_merge step on one GPU (for ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness.key_merge import KeyMerge  # noqa: E402
from paper_2101_08878_b200.loop import MonotonicClock, TaskLoop  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=100_000_000)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
km = KeyMerge(a.rows, 0.3)
km.generate()
loop = TaskLoop(MonotonicClock())
for _ in range(a.steps):
    print(loop.run_until_complete(km.run()))
