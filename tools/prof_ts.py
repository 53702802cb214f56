"""Profiling driver: set up transpose_sum and launch the fused kernel a few times (for ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2101_08878_b200 import native  # noqa: E402
from paper_2101_08878_b200.harness.transpose_sum import TransposeSum  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=40000)
ap.add_argument("--block", type=int, default=2000)
ap.add_argument("--launches", type=int, default=3)
a = ap.parse_args()
ts = TransposeSum(a.n, a.block).setup()
for _ in range(a.launches):
    ts.launch()
ts.stream.synchronize()
print("checksum", ts.combine(ts.read_block_sums()).checksum)
