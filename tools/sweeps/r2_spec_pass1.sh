#!/bin/bash
# Speculative pass 1 (no histogram pass; regions per (bucket, CTA), gated exact fallback) vs the histogram pass.
exec > gpurun_out/r2_spec_pass1.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -3
for rep in 1 2; do
  timeout 300 python tools/km_time.py --tag "spec"
  M4D_PASS1=hist timeout 300 python tools/km_time.py --tag "hist"
done
timeout 300 python tools/km_time.py --fraction 1.0 --tag "spec f=1.0"
