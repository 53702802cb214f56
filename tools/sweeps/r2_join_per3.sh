#!/bin/bash
exec > gpurun_out/r2_join_per3.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -2
timeout 300 python tools/km_time.py --tag "per=3 f=1" --fraction 1.0
timeout 300 python tools/km_time.py --tag "per=3 f=0.02" --fraction 0.02
M4D_JOIN=small timeout 300 python tools/km_time.py --tag "per=3 small"
