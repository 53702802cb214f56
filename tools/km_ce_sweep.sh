# key_merge at N=2/4: copy-engine pulls split over 1 / 2 / 4 streams
for N in 2 4; do for cfg in "M4D_CE_SPLIT=1" "M4D_CE_SPLIT=2" "M4D_CE_SPLIT=4"; do
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --workload key_merge --steps 5 --warmup 3 --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $cfg', round(d['ms_per_step'],3), d['config']['digest'][0], d['roofline']['phases'])"
done; done
