#!/bin/bash
# Tile size of the push scatter (M4D_TILE_THREADS 512 = 4096-row tiles, 1024 = 8192), N=2.
exec > gpurun_out/r2_push_tile.log 2>&1
for rep in 1 2; do for tt in 512 1024; do
  M4D_TILE_THREADS=$tt timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_pushtile_$tt.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pushtile_$tt.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=2 tile threads $tt step', round(d['ms_per_step'],3), 'plan0', t['plan0_done'], 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'join_end', t['join_end'])"
done; done
