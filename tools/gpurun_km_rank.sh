# tile scatter ranking: ballot multisplit vs per-warp shared atomics (tests under both, N=1 and N=2 bench)
M4D_TILE_RANK=atomic timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests_atomic.log 2>&1; echo "km tests (atomic) exit $?"; tail -2 gpurun_out/km_tests_atomic.log
for r in ballot atomic; do
  M4D_TILE_RANK=$r timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmr_${r}_n1.json 2> gpurun_out/kmr_${r}_n1.err
  M4D_TILE_RANK=$r timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmr_${r}_n2.json 2> gpurun_out/kmr_${r}_n2.err
done
for f in gpurun_out/kmr_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value'],3), d['config']['digest'][0], {k: round(v['ms'],3) for k, v in r['kernel_groups'].items()})"; done
M4D_TILE_RANK=atomic ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"tile_scatter" -c 4 python tools/prof_km.py --steps 1 2>&1 | grep -E "tile_scatter|duration|inst_exec" | sed 's/(const.*//'
