#!/bin/bash
# Speculative pass 1 with TMA bulk run stores: tile CTA size.
exec > gpurun_out/r2_spec_bulk_threads.log 2>&1
for t in 512 256 1024 512; do M4D_TILE_THREADS=$t timeout 300 python tools/km_time.py --tag "tile_threads=$t bulk"; done
