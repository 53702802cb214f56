#!/bin/bash
# Fine counts queued after side 1's plan read-back: tests + N=2 / N=4 traces.
exec > gpurun_out/r2_fine_order.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py -x -q -k "worker or counted or spec or shuffle or push" 2>&1 | tail -1
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_fo_${n}.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_fo_${n}.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'plan1', t['plan1_done'], 'push0_end', t['push0_end'], 'push1', t['push1_start'], t['push1_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
