#!/bin/bash
# Fused push counts flushed with one 64-bit add per counter pair: tests, N=2 timing.
exec > gpurun_out/r2_push_fine64.log 2>&1
timeout 1200 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "push or counted or world or multiprocess or speculative or skew" 2>&1 | tail -2
for rep in 1 2; do for fused in 1 0; do
  M4D_MERGE_FINE_FUSED=$fused timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_pf64_${fused}.json 2>gpurun_out/r2_pf64_${fused}.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pf64_${fused}.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=2 fused=$fused step', round(d['ms_per_step'],3), 'parity', d['parity']['digest_equal'], 'push1_end', t['push1_end'], 'split0_end', t['split0_end'], 'split1', t['split1_start'], t['split1_end'], 'join_end', t['join_end'])"
done; done
