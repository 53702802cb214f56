timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/r2_join_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/r2_join_tests.log
timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_join_n1.json 2> gpurun_out/r2_join_n1.err; echo km=$?; python -c "
import json; d=json.loads(open('gpurun_out/r2_join_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel_groups']['join'])"
M4D_JOIN=big timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_join_n1_big.json 2>&1; echo kmb=$?; python -c "
import json; d=json.loads(open('gpurun_out/r2_join_n1_big.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel_groups']['join'])"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:join_staged -s 1 -c 1 -o gpurun_out/r2_join_staged -f python tools/prof_km.py --steps 2 > /dev/null 2>&1; echo ncu=$?
