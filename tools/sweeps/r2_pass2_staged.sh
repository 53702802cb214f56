#!/bin/bash
# Pass 2 after the speculative pass 1: tile-staged with TMA bulk run stores (M4D_PASS2=staged) vs row scatter.
exec > gpurun_out/r2_pass2_staged.log 2>&1
M4D_PASS2=staged timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "pass2=rows"
  M4D_PASS2=staged timeout 300 python tools/km_time.py --tag "pass2=staged"
done
M4D_PASS2=staged ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spec_pass2 --launch-skip 2 --launch-count 1 python tools/prof_km.py --steps 2 2>&1 | grep -E "spec_pass2|duration|dram" | head -6
