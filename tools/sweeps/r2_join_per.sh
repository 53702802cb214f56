#!/bin/bash
# Join probe rows per thread per batch (kJoinPer 2 / 3 / 4): rebuilt on the box, N=1 timing.
exec > gpurun_out/r2_join_per.log 2>&1
cp paper_2101_08878_b200/csrc/key_merge.cu /tmp/key_merge.cu.orig
for per in 3 4 3 4; do
  sed "s/^constexpr int kJoinPer = 4;/constexpr int kJoinPer = $per;/" /tmp/key_merge.cu.orig > paper_2101_08878_b200/csrc/key_merge.cu
  make -s -C paper_2101_08878_b200/csrc > /dev/null 2>&1 || { echo "build failed for $per"; continue; }
  timeout 300 python tools/km_time.py --tag "per=$per"
done
cp /tmp/key_merge.cu.orig paper_2101_08878_b200/csrc/key_merge.cu
