#!/bin/bash
# Persistent join grid (one wave walking partitions, next partition prefetched) vs one CTA per partition.
exec > gpurun_out/r2_join_persist.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "default"
  M4D_JOIN_PERSIST=1 timeout 300 python tools/km_time.py --tag "persist pf=3"
  M4D_JOIN_PERSIST=1 M4D_JOIN_PF=0 timeout 300 python tools/km_time.py --tag "persist pf=0"
  M4D_JOIN_PERSIST=1 M4D_JOIN_PF=2 timeout 300 python tools/km_time.py --tag "persist pf=2"
done
