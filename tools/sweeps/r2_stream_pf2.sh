#!/bin/bash
# Prefetch distance of the tile scatter (M4D_L2_PF = tiles ahead; 0 off).
exec > gpurun_out/r2_stream_pf2.log 2>&1
for rep in 1 2; do for pf in 1 2 3 0; do M4D_L2_PF=$pf timeout 300 python tools/km_time.py --tag "pf=$pf"; done; done
