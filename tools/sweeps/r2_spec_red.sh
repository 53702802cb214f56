#!/bin/bash
# Speculative pass 1: full-id counts added without a return value (RED) and flushed every 15 tiles.
exec > gpurun_out/r2_spec_red.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do timeout 300 python tools/km_time.py --tag "spec red"; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tile_scatter --launch-skip 2 --launch-count 1 python tools/prof_km.py --steps 2 2>&1 | grep -E "tile_scatter|duration|dram" | head -6
