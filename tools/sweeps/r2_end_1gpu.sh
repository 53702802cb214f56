#!/bin/bash
# End-of-round checks on one GPU at head (after the fused push counts): GPU suite, smoke, default bench line, reference arm,
# and the key_merge N=1 launch list with DRAM bytes per launch.
exec > gpurun_out/r2_end_1gpu.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/r2_end_bench_n1.json 2> gpurun_out/r2_end_bench_n1.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_end_ref_n1.json 2> gpurun_out/r2_end_ref_n1.err; echo ref=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_end_bench_n1.json') if l.startswith('{')][-1]); k=d['key_merge']
print('ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'], 'launches', d.get('gpu_launches'), 'clocks', d.get('clocks'))
print('km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k.get('parity'), 'e2e', k['e2e']['value'], 'cpu', k['cpu_baseline']['value'])
r=json.loads([l for l in open('gpurun_out/r2_end_ref_n1.json') if l.startswith('{')][-1]); print('ref', r.get('value'), r.get('unit'), (r.get('key_merge') or {}).get('value'))"
