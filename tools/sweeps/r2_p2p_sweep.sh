# osu_bw 4 / 16 / 64 MiB under pull-engine settings (2 GPUs)
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 2 --workload p2p --skip-cpu --max-size 67108864; }
for cfg in "M4D_PULL_CTAS=296" "M4D_PULL_CTAS=148" "M4D_PULL_CTAS=444" "M4D_PULL_STREAMS=2" "M4D_PULL_STREAMS=8" "M4D_PULL_BATCH_BYTES=8388608" "M4D_PULL_ILP=2"; do
  env $cfg bash -c "$(declare -f run); run" > gpurun_out/r2_ps.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_ps.json') if l.startswith('{')][-1]); print('$cfg', [(r['size']>>20, round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=(1<<20)])"
done
