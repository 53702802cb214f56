#!/bin/bash
# Join grid: one CTA per partition (default) vs a persistent grid claiming partitions from a counter (M4D_JOIN_PERSIST=2).
exec > gpurun_out/r2_join_dyn.log 2>&1
M4D_JOIN_PERSIST=2 timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "per-partition"
  M4D_JOIN_PERSIST=2 timeout 300 python tools/km_time.py --tag "persistent dynamic"
  M4D_JOIN_PERSIST=2 M4D_JOIN_PF=0 timeout 300 python tools/km_time.py --tag "persistent dynamic pf=0"
done
