#!/bin/bash
# L2 prefetch of the next tile in the tile scatter (M4D_TILE_PF), key_merge N=1 and N=2.
exec > gpurun_out/r2_tile_pf.log 2>&1
for pf in 1 0 1 0; do M4D_TILE_PF=$pf timeout 300 python tools/km_time.py --tag pf=$pf; done
for pf in 1 0; do
  M4D_TILE_PF=$pf timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_tilepf_$pf.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_tilepf_$pf.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=2 pf=$pf step', round(d['ms_per_step'],3), 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'join_end', t['join_end'])"
done
