#!/bin/bash
# L2 prefetch of the next chunk: tile scatter (M4D_TILE_PF) and the other streaming passes (M4D_STREAM_PF).
exec > gpurun_out/r2_stream_pf.log 2>&1
for rep in 1 2; do
for c in "1 1" "1 0" "0 0" "0 1"; do set -- $c
  M4D_TILE_PF=$1 M4D_STREAM_PF=$2 timeout 300 python tools/km_time.py --tag "tile=$1,stream=$2"
done; done
