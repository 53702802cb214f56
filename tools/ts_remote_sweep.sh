# N=2 transpose_sum ablations (remote-stream CTAs, L2 promotion of peer tensor maps)
for cfg in "default" "M4D_TS_REMOTE_PROMO=none" "M4D_TS_REMOTE_PROMO=128" "M4D_TS_REMOTE_CTAS=148" "M4D_TS_REMOTE_CTAS=120"; do
  env $([ "$cfg" = default ] || echo $cfg) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', d['ms_per_step'], r['kernel_ms'], r['frac'])"
done
