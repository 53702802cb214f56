# Join variant x partition size x L2 prefetch at 1e8 rows/side, N=1 (M4D_JOIN, M4D_JOIN_PART_ROWS, M4D_JOIN_PF)
for cfg in "big 0 3" "small 12400 3" "small 12400 1" "small 0 3" "big 6200 3" "big 0 3"; do
  set -- $cfg
  env M4D_JOIN=$1 $( [ "$2" != 0 ] && echo M4D_JOIN_PART_ROWS=$2 ) M4D_JOIN_PF=$3 timeout 300 python bench.py --workload key_merge --skip-e2e --skip-cpu \
    > gpurun_out/jv.json 2>/dev/null
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/jv.json").read().strip().splitlines()[-1])
g = d["roofline"]["kernel_groups"]
print(f"join={sys.argv[1]} part_rows={sys.argv[2]} pf={sys.argv[3]} parts={d['config']['partitions']} step={d['value']:.3f} ms join={g['join']['ms']:.3f} part={g['partition']['ms']:.3f} digest={d['config']['digest']}")
PY
done
