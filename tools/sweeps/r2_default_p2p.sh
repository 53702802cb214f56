#!/bin/bash
# Default bench line at N=2 with the p2p sub-record.
exec > gpurun_out/r2_default_p2p.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 > gpurun_out/r2_default_p2p_n2.json 2> gpurun_out/r2_default_p2p_n2.err; echo n2=$?
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_default_p2p_n2.json') if l.startswith('{')][-1]); k=d['key_merge']
print('N=2 ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), '| km', round(k['value'],3), 'parity', k['parity']['digest_equal'], '| p2p', json.dumps(d.get('p2p')))"
tail -3 gpurun_out/r2_default_p2p_n2.err
