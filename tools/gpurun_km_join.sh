# key_merge join variants: tests under both, N=1 bench big vs small, N=2 small
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests.log 2>&1; echo "km tests (big) exit $?"; tail -2 gpurun_out/km_tests.log
M4D_JOIN=small timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests_small.log 2>&1; echo "km tests (small) exit $?"; tail -2 gpurun_out/km_tests_small.log
for j in big small; do
  M4D_JOIN=$j timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmj_${j}_n1.json 2> gpurun_out/kmj_${j}_n1.err
  M4D_JOIN=$j timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmj_${j}_n2.json 2> gpurun_out/kmj_${j}_n2.err
done
for f in gpurun_out/kmj_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value'],3), d['config']['digest'][0], d['config']['partitions'], r.get('phases'))
print('   ', {k: {kk: (round(vv,3) if isinstance(vv,float) else vv) for kk, vv in v.items() if kk!='note'} for k, v in r['kernel_groups'].items()})"; done
tail -3 gpurun_out/kmj_big_n1.err
