#!/bin/bash
# Pass-2 CTA groups per segment after the speculative pass 1 (key_merge N=1, 1e8 rows/side).
exec > gpurun_out/r2_pass2_groups.log 2>&1
for g in 8 12 16 24 32 8; do M4D_PASS2_GROUPS=$g timeout 300 python tools/km_time.py --tag "pass2_groups=$g"; done
