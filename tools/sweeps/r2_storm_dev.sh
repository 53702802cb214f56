#!/bin/bash
# Device-frame storm: GPU tests, then the storm bench line (host + device frames) at 2 and 4 GPUs.
exec > gpurun_out/r2_storm_dev.log 2>&1
timeout 600 python -m pytest tests/test_storm.py tests/test_eager_device.py -x -q 2>&1 | tail -3
G=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $G ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800 + n)) \
    bench.py --gpus $n --workload storm --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2_storm_dev_n$n.json 2> gpurun_out/r2_storm_dev_n$n.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_storm_dev_n$n.json') if l.startswith('{')][-1])
print($n, 'host', round(d['value']), d['latency_us'], 'device', {k: d['device_frames'][k] for k in ('value', 'latency_us', 'eager_device_sends_rank0', 'proxy_copies_rank0')})"
done
