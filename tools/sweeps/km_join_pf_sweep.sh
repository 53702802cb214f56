# Sweep of the join kernel's L2 bulk prefetch modes (M4D_JOIN_PF bits, M4D_JOIN_PF_AHEAD) at 1e8 rows/side, N=1
for cfg in "0" "1" "3" "4" "5" "7" "5 296" "5 74" "small:0" "small:5"; do
  set -- $cfg
  mode=$1; ahead=${2:-148}; join=big
  case $mode in small:*) join=small; mode=${mode#small:};; esac
  M4D_JOIN=$join M4D_JOIN_PF=$mode M4D_JOIN_PF_AHEAD=$ahead timeout 300 python bench.py --workload key_merge --skip-e2e --skip-cpu \
    > gpurun_out/pf.json 2>/dev/null
  python - "$join" "$mode" "$ahead" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/pf.json").read().strip().splitlines()[-1])
g = d["roofline"]["kernel_groups"]
print(f"join={sys.argv[1]} pf={sys.argv[2]} ahead={sys.argv[3]} step={d['value']:.3f} ms join={g['join']['ms']:.3f} part={g['partition']['ms']:.3f} digest={d['config']['digest']}")
PY
done
