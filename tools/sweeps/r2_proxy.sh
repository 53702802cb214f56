#!/bin/bash
# Eager device proxy kernel: tests, then device-frame latency with and without it (2 GPUs).
exec > gpurun_out/r2_proxy.log 2>&1
timeout 900 python -m pytest tests/test_eager_device.py tests/test_multiprocess_gpu.py tests/test_transport_nvlink.py tests/test_framed_nvlink.py -x -q 2>&1 | tail -5
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --workload p2p --skip-cpu --max-size 4194304; }
for proxy in 1 0 1; do
  M4D_EAGER_PROXY=$proxy run $((29700 + RANDOM % 100)) > gpurun_out/r2_proxy_$proxy.json 2> gpurun_out/r2_proxy_$proxy.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_proxy_$proxy.json') if l.startswith('{')][-1])
print('proxy=$proxy', 'eager', d['device_eager_latency_us'], 'rdv 1B', d['latency_1B_us'], 'comm', {k: round(v['latency_us'], 2) for k, v in d['comm_path'].items()}, 'bw4M', d['value'])"
done
