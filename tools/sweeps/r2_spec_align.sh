#!/bin/bash
# Speculative pass 1: region rows aligned to 128-byte lines, and TMA bulk run stores.
exec > gpurun_out/r2_spec_align.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "align=1"
  M4D_SPEC_ALIGN=8 timeout 300 python tools/km_time.py --tag "align=8"
  M4D_SPEC_ALIGN=16 timeout 300 python tools/km_time.py --tag "align=16"
done
M4D_SPEC_ALIGN=8 M4D_TILE_STORE=bulk timeout 300 python tools/km_time.py --tag "align=8 bulk"
M4D_TILE_STORE=bulk timeout 300 python tools/km_time.py --tag "align=1 bulk"
