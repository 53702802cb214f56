timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/r2_jp_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2_jp_tests.log
for j in pair big pair big; do
M4D_JOIN=$j timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_jp_$j.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_jp_$j.json').read().strip().splitlines()[-1]); print('$j', d['value'], d['roofline']['kernel_groups']['join']['ms'])"
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:join_pair -s 1 -c 1 -o gpurun_out/r2_join_pair -f python tools/prof_km.py --steps 2 > /dev/null 2>&1; echo ncu=$?
