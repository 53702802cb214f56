#!/bin/bash
# Proxy idle timeout vs device-frame storm throughput and relaunches (in-process, 2 ranks on cuda:0), and 2-GPU storm.
exec > gpurun_out/r2_proxy_idle.log 2>&1
for idle in 100 1000 100 1000; do
  M4D_EAGER_PROXY_IDLE_US=$idle M4D_EAGER_DEVICE_RING=67108864 timeout 300 python tools/storm_profile.py 20000 --no-profile | grep "device 0" | sed "s/^/idle=$idle /" | cut -c1-60
done
for idle in 100 1000; do
  M4D_EAGER_PROXY_IDLE_US=$idle timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29750 + idle % 7)) bench.py --gpus 2 --workload storm --steps 3 --warmup 3 --skip-cpu > gpurun_out/r2_pidle_$idle.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pidle_$idle.json') if l.startswith('{')][-1])
print('N=2 idle=$idle host', round(d['value']), 'device', round(d['device_frames']['value']))"
done
