#!/bin/bash
# Counted receiver split for side 1 (M4D_MERGE_FINE): parity tests, N=2 / N=4 traces with and without.
exec > gpurun_out/r2_fine_split.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "key_merge or km or shuffle or push or worker or owner" 2>&1 | tail -2
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for fine in 1 0 1; do
  M4D_MERGE_FINE=$fine timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_fine_${n}_$fine.json 2>gpurun_out/r2_fine_${n}_$fine.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_fine_${n}_$fine.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n fine=$fine step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'plan1', t['plan1_done'], 'push1', t['push1_start'], t['push1_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
