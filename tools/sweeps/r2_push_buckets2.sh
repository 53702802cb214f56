#!/bin/bash
# Push buckets (owners x coarse runs: 256 default, 128 = longer NVLink runs, wider split) with the counted split.
exec > gpurun_out/r2_push_buckets2.log 2>&1
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for pb in 256 128 256 128; do
  M4D_PUSH_BUCKETS=$pb timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_pb_${n}_$pb.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pb_${n}_$pb.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n buckets=$pb step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'split1', round(t['split1_end']-t['split1_start'],3), 'join_end', t['join_end'])"
done; done
