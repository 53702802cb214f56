# key_merge receiver split: CTAs per SM sweep (N=2, push 256 buckets), tests first
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests.log 2>&1; echo "km tests exit $?"; tail -3 gpurun_out/km_tests.log
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e ; }
for r in 2 4 8 16 32; do
  M4D_RUNS_CTAS_PER_SM=$r M4D_PUSH_BUCKETS=256 run 2 > gpurun_out/km_r${r}_n2.json 2> gpurun_out/km_r${r}_n2.err
done
for f in gpurun_out/km_r*_n2.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],3), d['config'].get('digest')[0], d['roofline'].get('phases'))"; done
