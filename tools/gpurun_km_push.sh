# key_merge fused push shuffle (defaults) vs pull, push-bucket sweep, at N=2 and N=4
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests.log 2>&1; echo "km tests exit $?"; tail -3 gpurun_out/km_tests.log
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e ; }
for N in ${NS:-2 4}; do
  M4D_MERGE_SHUFFLE=pull run $N > gpurun_out/km_pull_n$N.json 2> gpurun_out/km_pull_n$N.err
  for pb in ${PBS:-64 128 256}; do
    M4D_PUSH_BUCKETS=$pb M4D_MERGE_SHUFFLE=push run $N > gpurun_out/km_pb${pb}_n$N.json 2> gpurun_out/km_pb${pb}_n$N.err
  done
done
for f in gpurun_out/km_pull_n[24].json gpurun_out/km_pb*_n[24].json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],3), d['config'].get('digest')[0], d['roofline'].get('phases'))"; done
