#!/bin/bash
# Pass-1 fan-out of the two-pass local partition (M4D_PASS1_BITS), key_merge N=1, 1e8 rows/side.
exec > gpurun_out/r2_pass1_bits.log 2>&1
for b in 8 7 6 8 7; do M4D_PASS1_BITS=$b timeout 300 python tools/km_time.py --tag bits=$b; done
