#!/bin/bash
# Join diagnostics (key_merge N=1, 1e8 rows/side): 0 staged emit (default), 3 direct emit, 2 count only.
exec > gpurun_out/r2_join_exp.log 2>&1
for e in 0 3 2 3 0; do M4D_JOIN_EXP=$e timeout 300 python tools/km_time.py --tag exp=$e; done
M4D_JOIN_EXP=3 timeout 300 python tools/km_time.py --tag exp=3,f=1 --fraction 1.0
timeout 300 python tools/km_time.py --tag exp=0,f=1 --fraction 1.0
