#!/bin/bash
# Final checks on one GPU at the round head (speculative pass 1 with bulk stores): GPU suite, smoke, default bench line, reference arm,
# and the key_merge N=1 launch list with DRAM bytes per launch.
exec > gpurun_out/r2_head_1gpu.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 900 python bench.py > gpurun_out/r2_head_bench_n1.json 2> gpurun_out/r2_head_bench_n1.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_head_ref_n1.json 2> gpurun_out/r2_head_ref_n1.err; echo ref=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_head_bench_n1.json') if l.startswith('{')][-1]); k=d['key_merge']
print('ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'], 'launches', d.get('gpu_launches'), 'clocks', d.get('clocks'))
print('km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k.get('parity'), 'e2e', k['e2e']['value'], 'cpu', k['cpu_baseline']['value'])
r=json.loads([l for l in open('gpurun_out/r2_head_ref_n1.json') if l.startswith('{')][-1]); print('ref', r.get('value'), r.get('unit'), (r.get('key_merge') or {}).get('value'))"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_head_launches_km.csv python tools/prof_km.py --steps 3 > /dev/null 2>&1; echo ncu=$?
python tools/ncu_csv.py gpurun_out/r2_head_launches_km.csv > gpurun_out/r2_head_launches_km.txt; tail -30 gpurun_out/r2_head_launches_km.txt
