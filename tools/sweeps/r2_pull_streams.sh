#!/bin/bash
# Pull streams (M4D_PULL_STREAMS) x posting style: osu_bw 1-64 MiB per-post, 4 MiB vectored.
exec > gpurun_out/r2_pull_streams.log 2>&1
for ps in 1 2 4 8; do
M4D_PULL_STREAMS=$ps timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + ps)) bench.py --gpus 2 --workload p2p --skip-cpu > gpurun_out/r2_ps_$ps.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_ps_$ps.json') if l.startswith('{')][-1])
print('streams=$ps per-post', [(r['size']>>20, round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=(1<<20)], 'vectored 4MiB', round(d['osu_bw_4MiB_vectored_GBps']))"
done
