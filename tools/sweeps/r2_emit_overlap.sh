#!/bin/bash
# Join emit: the warp's output reservation read after the first emit loads (atomic round trip hidden).
exec > gpurun_out/r2_emit_overlap.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -1
for rep in 1 2 3; do timeout 300 python tools/km_time.py --tag "N=1"; done
timeout 300 python tools/km_time.py --fraction 1.0 --tag "N=1 f=1.0"
