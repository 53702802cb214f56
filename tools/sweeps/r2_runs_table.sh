#!/bin/bash
# Run tables built at table-exchange time (off the split's critical path): tests + N=2 / N=4 traces.
exec > gpurun_out/r2_runs_table.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "key_merge or km or shuffle or push or worker or owner or counted or spec" 2>&1 | tail -1
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_rt_${n}.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_rt_${n}.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'push1_end', t['push1_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
