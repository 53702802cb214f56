for j in small big small big; do
M4D_JOIN=$j timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_js_$j.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_js_$j.json').read().strip().splitlines()[-1]); g=d['roofline']['kernel_groups']; print('$j', d['value'], d['config']['partitions'], g['partition']['ms'], g['join']['ms'])"
done
