# transpose_sum at N = $1 GPUs: default schedule plus remote-CTA ablations
N=${1:-2}
for cfg in "default" "M4D_TS_REMOTE_CTAS=148" "M4D_TS_REMOTE_CTAS=130" "M4D_TS_REMOTE_CTAS=90"; do
  env $([ "$cfg" = default ] || echo $cfg) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('N=$N $cfg', round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(r['frac'],3))"
done
