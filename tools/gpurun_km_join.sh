# key_merge join: persistent + L2-prefetch grid vs one CTA per partition
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests.log 2>&1; echo "km tests exit $?"; tail -2 gpurun_out/km_tests.log
M4D_JOIN_PERSIST=1 timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/km_tests_p.log 2>&1; echo "km tests (persist) exit $?"; tail -2 gpurun_out/km_tests_p.log
for pj in 0 1; do for j in big small; do
  M4D_JOIN=$j M4D_JOIN_PERSIST=$pj timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/kmj_${j}_p${pj}_n1.json 2> gpurun_out/kmj_${j}_p${pj}_n1.err
done; done
for f in gpurun_out/kmj_*_p*_n1.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value'],3), d['config']['digest'][0], d['config']['partitions'], {k: round(v['ms'],3) for k, v in r['kernel_groups'].items()})"; done
