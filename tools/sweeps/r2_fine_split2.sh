#!/bin/bash
# Counted receiver split with 16-bit spilling counters: tests (skew, parity), N=2 / N=4 timing, 8 ranks on 4 GPUs.
exec > gpurun_out/r2_fine_split2.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q 2>&1 | tail -2
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for fine in 1 0; do
  M4D_MERGE_FINE=$fine timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_fine2_${n}_$fine.json 2>gpurun_out/r2_fine2_${n}_$fine.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_fine2_${n}_$fine.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n fine=$fine step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
[ -f tools/sweeps/r2_n8_functional.sh ] && timeout 900 bash tools/sweeps/r2_n8_functional.sh 2>&1 | tail -5
