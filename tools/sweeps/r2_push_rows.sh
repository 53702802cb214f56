#!/bin/bash
# Push scatter tiles of 12 rows per thread (12288-row tiles, 48-row runs; spills) vs 8: tests + N=2 / N=4.
exec > gpurun_out/r2_push_rows.log 2>&1
M4D_PUSH_ROWS=12 timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q -k "worker or counted or spec or shuffle or push" 2>&1 | tail -1
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for pr in 8 12 8 12; do
  M4D_PUSH_ROWS=$pr timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_pr_${n}_$pr.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pr_${n}_$pr.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n rows=$pr step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'join_end', t['join_end'])"
done; done
