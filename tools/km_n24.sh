# key_merge at N=2 and N=4 (default settings) + the 2-GPU transport/merge tests
timeout 600 python -m pytest tests/test_key_merge_gpu.py tests/test_transport_nvlink.py -m gpu -q -x --timeout 300 2>&1 | tail -1
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N --workload key_merge --steps 5 --warmup 3 --skip-e2e --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N', round(d['ms_per_step'],3), d['config']['digest'], d['roofline']['phases'])"
done
