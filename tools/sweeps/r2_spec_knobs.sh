#!/bin/bash
# Knobs around the speculative pass 1 (key_merge N=1, 1e8 rows/side): tile CTA size, pass-2 groups, side concurrency.
exec > gpurun_out/r2_spec_knobs.log 2>&1
timeout 300 python tools/km_time.py --tag "default"
M4D_TILE_THREADS=256 timeout 300 python tools/km_time.py --tag "tile_threads=256"
M4D_TILE_THREADS=1024 timeout 300 python tools/km_time.py --tag "tile_threads=1024"
M4D_PASS2_GROUPS=4 timeout 300 python tools/km_time.py --tag "pass2_groups=4"
M4D_PASS2_GROUPS=2 timeout 300 python tools/km_time.py --tag "pass2_groups=2"
M4D_MERGE_SIDES=serial timeout 300 python tools/km_time.py --tag "sides=serial"
M4D_L2_PF=0 timeout 300 python tools/km_time.py --tag "l2_pf=0"
timeout 300 python tools/km_time.py --tag "default"
