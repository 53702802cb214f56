#!/bin/bash
exec > gpurun_out/r2_hist2_vec.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/km_time.py --tag "hist2 vec"; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:hist2 --launch-skip 2 --launch-count 2 python tools/prof_km.py --steps 2 2>&1 | grep -E "hist2|duration|dram" | head -8
