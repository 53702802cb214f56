timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/r2_sides_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2_sides_tests.log
for mode in concurrent serial concurrent serial; do
M4D_MERGE_SIDES=$mode timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_sides_$mode.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_sides_$mode.json').read().strip().splitlines()[-1]); print('$mode', d['value'], d['roofline']['kernel_groups']['partition']['ms'], d['roofline']['kernel_groups']['join']['ms'])"
done
