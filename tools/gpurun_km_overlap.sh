# key_merge N>1 overlap: push CTA size / CTAs per SM x receiver-split CTA size (split on its own stream)
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests.log 2>&1; echo "km tests exit $?"; tail -2 gpurun_out/km_tests.log
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e ; }
for N in 2 4; do
for cfg in "1024 4 1024" "512 1 512" "512 1 1024" "512 2 512" "1024 1 512"; do
  set -- $cfg
  M4D_PUSH_TILE_THREADS=$1 M4D_PUSH_CTAS_PER_SM=$2 M4D_RUNS_THREADS=$3 run $N > gpurun_out/kmo_$1_$2_$3_n$N.json 2> gpurun_out/kmo_$1_$2_$3_n$N.err
done; done
for f in gpurun_out/kmo_*_n[24].json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value'],3), d['config']['digest'][0], r.get('phases'))"; done
