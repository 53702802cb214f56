#!/bin/bash
# Pass 2 after the speculative pass 1: 1024- vs 512-thread CTAs (2 per SM), and 16 groups with 512.
exec > gpurun_out/r2_pass2_threads.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "pass2_threads=1024"
  M4D_PASS2_THREADS=512 timeout 300 python tools/km_time.py --tag "pass2_threads=512"
done
M4D_PASS2_THREADS=512 M4D_PASS2_GROUPS=4 timeout 300 python tools/km_time.py --tag "pass2_threads=512 groups=4"
