# tile scatter CTA size with atomic ranking (N=1)
for tt in 256 512 1024; do
  M4D_TILE_THREADS=$tt timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmt_$tt.json 2> gpurun_out/kmt_$tt.err
  python -c "
import json
d=json.loads(open('gpurun_out/kmt_$tt.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tt', round(d['value'],3), d['config']['digest'][0], {k: round(v['ms'],3) for k, v in r['kernel_groups'].items()})"
done
