#!/bin/bash
# Native composites for lone small device frames: GPU tests, storm profile, p2p comm-path latency, storm bench.
exec > gpurun_out/r2_framed_dev.log 2>&1
timeout 900 python -m pytest tests/test_eager_device.py tests/test_storm.py tests/test_multiprocess_gpu.py tests/test_serializers.py tests/test_comm_stack_nvlink.py tests/test_framed_nvlink.py -x -q 2>&1 | tail -15
M4D_EAGER_DEVICE_RING=67108864 timeout 300 python tools/storm_profile.py 20000 --no-profile
timeout 300 python tools/storm_profile.py 20000 --no-profile
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 2 --workload p2p --skip-cpu --max-size 4194304 > gpurun_out/r2_framed_p2p.json 2> gpurun_out/r2_framed_p2p.err
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_framed_p2p.json') if l.startswith('{')][-1])
print('eager', d['device_eager_latency_us'], 'rdv 1B', d['latency_1B_us'], 'comm', {k: round(v['latency_us'], 2) for k, v in d['comm_path'].items()}, 'bw4M', d['value'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29765 \
    bench.py --gpus 2 --workload storm --steps 3 --warmup 1 --skip-cpu > gpurun_out/r2_storm_dev_n2.json 2> gpurun_out/r2_storm_dev_n2.err
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_storm_dev_n2.json') if l.startswith('{')][-1])
print('storm n2 host', round(d['value']), d['latency_us'], 'device', d['device_frames'])"
