run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --workload p2p --skip-cpu; }
run 29601 > gpurun_out/r2_p2p_tma.json 2> gpurun_out/r2_p2p_tma.err; echo tma=$?
M4D_PULL_KERNEL=ldg run 29602 > gpurun_out/r2_p2p_ldg.json 2> gpurun_out/r2_p2p_ldg.err; echo ldg=$?
M4D_PULL_BATCH_BYTES=67108864 run 29603 > gpurun_out/r2_p2p_tma2.json 2> gpurun_out/r2_p2p_tma2.err; echo tma2=$?
for f in tma ldg tma2; do python -c "
import json,sys; d=json.loads([l for l in open('gpurun_out/r2_p2p_$f.json') if l.startswith('{')][-1]); print('$f', d['latency_1B_us'], [(r['size'], round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=65536])"; done
