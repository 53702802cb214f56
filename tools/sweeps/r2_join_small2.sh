#!/bin/bash
# Small join (two 512-thread CTAs per SM, 16384 partitions) vs big, after the L2 prefetch and the kept second match.
exec > gpurun_out/r2_join_small2.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "big"
  M4D_JOIN=small timeout 300 python tools/km_time.py --tag "small"
done
