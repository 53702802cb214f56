#!/bin/bash
# Speculative pass 1 with TMA bulk run stores by default: key_merge tests, timing, default bench line.
exec > gpurun_out/r2_spec_bulk.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do timeout 300 python tools/km_time.py --tag "bulk (default)"; done
M4D_TILE_STORE=rows timeout 300 python tools/km_time.py --tag "rows"
timeout 300 python tools/km_time.py --fraction 1.0 --tag "bulk f=1.0"
timeout 900 python bench.py > gpurun_out/r2_spec_bulk_bench_n1.json 2> gpurun_out/r2_spec_bulk_bench_n1.err; echo bench=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_spec_bulk_bench_n1.json') if l.startswith('{')][-1]); k=d['key_merge']
print('ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), 'clocks', d.get('clocks'))
print('km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k['parity']['digest_equal'], k['parity']['row_conservation'], 'e2e', k['e2e']['value'], 'launches', k.get('gpu_launches'))"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_spec_bulk_launches.csv python tools/prof_km.py --steps 3 > /dev/null 2>&1; echo ncu=$?
python tools/ncu_csv.py gpurun_out/r2_spec_bulk_launches.csv > gpurun_out/r2_spec_bulk_launches.txt
