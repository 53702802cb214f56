#!/bin/bash
# Join: matches per probe row staged without a chain re-walk (M4D_JOIN_KEEP 1 = first only, 2, 3).
exec > gpurun_out/r2_join_second.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do for k in 1 2 3; do M4D_JOIN_KEEP=$k timeout 300 python tools/km_time.py --tag "keep=$k"; done; done
for k in 1 2 3; do M4D_JOIN_KEEP=$k timeout 300 python tools/km_time.py --tag "keep=$k f=1" --fraction 1.0; done
