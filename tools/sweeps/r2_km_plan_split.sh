#!/bin/bash
# key_merge N=2 / N=4 with side 0's plan alone and side 1's plan beside push 0: tests + bench traces.
exec > gpurun_out/r2_km_plan_split.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "km or key_merge or shuffle or worker or push or pull" 2>&1 | tail -2
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $G ] || continue
  for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_kmps_$n.json 2>gpurun_out/r2_kmps_$n.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_kmps_$n.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n step', round(d['ms_per_step'],3), t)"
  done
done
