#!/bin/bash
# Vectored posts (m4d_transport_post_many): tests, then the p2p sweep (osu_bw vectored vs per-post at 4 MiB).
exec > gpurun_out/r2_post_many.log 2>&1
timeout 900 python -m pytest tests/test_eager_device.py tests/test_transport_nvlink.py tests/test_multiprocess_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + rep)) bench.py --gpus 2 --workload p2p --skip-cpu > gpurun_out/r2_post_many_$rep.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_post_many_$rep.json') if l.startswith('{')][-1])
print('vectored', [(r['size']>>20, round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=(1<<20)], 'per-post 4MiB', round(d['osu_bw_4MiB_per_post_GBps']), 'lat', d['latency_1B_us'])"
done
