#!/bin/bash
# Counted split for side 1 only (default) vs both sides (M4D_MERGE_FINE_SIDES=2), N=2 / N=4.
exec > gpurun_out/r2_fine_sides.log 2>&1
M4D_MERGE_FINE_SIDES=2 timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q -k "worker or counted or spec or shuffle" 2>&1 | tail -1
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for fs in 1 2 1 2; do
  M4D_MERGE_FINE_SIDES=$fs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_fs_${n}_$fs.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_fs_${n}_$fs.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n sides=$fs step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'split0', t['split0_start'], t['split0_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
