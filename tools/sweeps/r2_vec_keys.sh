#!/bin/bash
# Counting passes read two keys per 16-byte load (hist2, owner plan, fine counts): tests + N=1 / N=2 / N=4.
exec > gpurun_out/r2_vec_keys.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/km_time.py --tag "N=1"; done
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do [ $n -le $G ] || continue; for rep in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_vk_${n}.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_vk_${n}.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'plan0', t['plan0_done'], 'plan1', t['plan1_done'], 'push1_end', t['push1_end'], 'join_end', t['join_end'])"
done; done
