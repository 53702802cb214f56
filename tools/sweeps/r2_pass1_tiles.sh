#!/bin/bash
# Tile-sorted pass 1 + gathering pass 2 (M4D_PASS1=tiles) vs histogram + scatter: parity tests, N=1 timing.
exec > gpurun_out/r2_pass1_tiles.log 2>&1
M4D_PASS1=tiles timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -3
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "scatter"
  M4D_PASS1=tiles timeout 300 python tools/km_time.py --tag "tiles"
done
