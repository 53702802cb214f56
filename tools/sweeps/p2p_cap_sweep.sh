# p2p osu_bw at 4/16/64 MiB vs the pull-kernel grid cap
for cfg in "default" "M4D_PULL_CTAS=64" "M4D_PULL_CTAS=128"; do
  env $([ "$cfg" = default ] || echo $cfg) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --workload p2p --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', [(r['size']>>20, round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=(1<<20)], 'comm', {k: round(v['GBps']) for k,v in d['comm_path'].items()})"
done
