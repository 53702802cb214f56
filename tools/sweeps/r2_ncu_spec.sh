#!/bin/bash
# ncu --set full of the speculative pass 1 (tile_scatter_kernel<512,0,1,1>; the gated fallback launches are captured too), key_merge N=1.
exec > gpurun_out/r2_ncu_spec1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_scatter --launch-skip 4 --launch-count 4 -o gpurun_out/r2_spec1_full -f python tools/prof_km.py --steps 2 > /dev/null 2>&1; echo ncu=$?
python tools/ncu_summary.py gpurun_out/r2_spec1_full.ncu-rep
ncu -i gpurun_out/r2_spec1_full.ncu-rep --page details 2>/dev/null | grep -E "^  [a-z_]|Achieved Occupancy|DRAM Throughput|^    Duration|Memory Throughput|L2 Hit Rate|Registers Per|Warp Cycles Per Issued" | head -40
