# key_merge N=1: join of finished pass-2 segments overlapped with the next segments' pass 2 (M4D_JOIN_OVERLAP chunks)
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q > gpurun_out/r2_ov_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2_ov_tests.log
for k in 1 2 4 8 16 4 1; do
M4D_JOIN_OVERLAP=$k timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_ov_$k.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_ov_$k.json').read().strip().splitlines()[-1]); print('K=$k', round(d['value'],3), d['parity']['digest_equal'], d['roofline']['trace_ms'])" || tail -3 gpurun_out/r2_ov_$k.json
done
