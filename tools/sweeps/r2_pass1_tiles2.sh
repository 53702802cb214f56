#!/bin/bash
exec > gpurun_out/r2_pass1_tiles2.log 2>&1
M4D_PASS1=tiles timeout 300 python tools/km_time.py --tag "tiles U=8"
timeout 300 python tools/km_time.py --tag "scatter"
M4D_PASS1=tiles ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/km_tiles2.csv python tools/prof_km.py --steps 1 > /dev/null 2>&1
