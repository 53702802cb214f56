#!/bin/bash
# Fused push counts at N=4: multi-GPU tests, N=4 fused vs separate, default line at N=2 and N=4.
exec > gpurun_out/r2_push_fine4.log 2>&1
timeout 1200 python -m pytest tests/test_multiprocess_gpu.py tests/test_key_merge_gpu.py -x -q -k "world or multiprocess or four or counted or push" 2>&1 | tail -2
for fused in 1 0 1; do
  M4D_MERGE_FINE_FUSED=$fused timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_pf_4_${fused}.json 2>gpurun_out/r2_pf_4_${fused}.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pf_4_${fused}.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=4 fused=$fused step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'push1_end', t['push1_end'], 'split0_end', t['split0_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29900 + n)) bench.py --gpus $n > gpurun_out/r2_head_n$n.json 2> gpurun_out/r2_head_n$n.err; echo n$n=$?
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_head_n$n.json') if l.startswith('{')][-1]); k=d['key_merge']
print('default N=$n ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), '| km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k['parity']['digest_equal'], k['parity'].get('row_conservation'))"
done
