#!/bin/bash
# Semi-join Bloom filter (M4D_MERGE_FILTER) vs plain partitions, key_merge N=1, 1e8 rows/side.
exec > gpurun_out/r2_filter.log 2>&1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q -k "semi_join or single_gpu or duplicate" 2>&1 | tail -5
for f in 0.3 1.0 0.02; do
  for filt in 0 1; do
    M4D_MERGE_FILTER=$filt timeout 300 python bench.py --workload key_merge --fraction $f --skip-cpu --skip-e2e \
      --steps 10 --warmup 3 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print('filter=$filt f=$f', d['ms_per_step'], {k:v.get('ms') for k,v in r.get('kernel_groups',{}).items()}, r.get('trace_ms'))"
  done
done
