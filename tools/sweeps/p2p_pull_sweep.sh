# p2p osu_bw at 1-64 MiB vs pull-kernel ILP, messages per launch and grid cap
for cfg in "X=1" "M4D_PULL_ILP=2" "M4D_PULL_ILP=4" "M4D_PULL_BATCH=16" "M4D_PULL_BATCH=16 M4D_PULL_ILP=4" "M4D_PULL_BATCH=32 M4D_PULL_ILP=4" "M4D_PULL_CTAS=592 M4D_PULL_ILP=4" "M4D_PULL_CTAS=148 M4D_PULL_ILP=4"; do
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --workload p2p --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', [(r['size']>>20, round(r['osu_bw_GBps'])) for r in d['sweep'] if r['size']>=(1<<20)], 'comm', {k: round(v['GBps']) for k,v in d['comm_path'].items()})"
done
