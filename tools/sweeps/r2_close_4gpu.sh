#!/bin/bash
# Closing multi-GPU checks (after the speculative pass 1): full GPU suite on 4 GPUs, default bench at N=2/N=4 + reference arm, p2p, storm.
exec > gpurun_out/r2_close_4gpu.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
run() { N=$1; P=$2; shift 2; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run 2 29801 > gpurun_out/r2_close_n2.json 2> gpurun_out/r2_close_n2.err; echo n2=$?
run 4 29802 > gpurun_out/r2_close_n4.json 2> gpurun_out/r2_close_n4.err; echo n4=$?
run 2 29803 --workload p2p > gpurun_out/r2_close_p2p.json 2> gpurun_out/r2_close_p2p.err; echo p2p=$?
run 4 29804 --workload storm --steps 3 --warmup 3 > gpurun_out/r2_close_storm_n4.json 2> gpurun_out/r2_close_storm_n4.err; echo storm4=$?
run 2 29805 --workload storm --steps 3 --warmup 3 > gpurun_out/r2_close_storm_n2.json 2> gpurun_out/r2_close_storm_n2.err; echo storm2=$?
for f in n2 n4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_close_$f.json') if l.startswith('{')][-1]); k=d['key_merge']
print('$f ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), '| km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k['parity']['digest_equal'], 'e2e', round(k['e2e']['value'],1))"; done
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_close_p2p.json') if l.startswith('{')][-1])
print('p2p', d['value'], 'lat1B', d['latency_1B_us'], d.get('latency_1B_protocol'), 'rdv', d.get('rendezvous_latency_1B_us'), 'eager', d['device_eager_latency_us'], 'host', d['host_frames_1B'], 'comm', {k: round(v['latency_us'],2) for k,v in d['comm_path'].items()}, 'cpu', d.get('cpu_baseline'))
print([(r['size'], round(r['osu_bw_GBps'])) for r in d['sweep']])"
for f in n2 n4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_close_storm_$f.json') if l.startswith('{')][-1])
print('storm $f host', round(d['value']), 'device', round(d['device_frames']['value']), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"; done
