# N=2 push-scatter occupancy sweep with the event trace (split of side 0 overlaps the push of side 1)
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e --steps 5; }
for cfg in "4 1024" "2 1024" "1 1024" "2 512" "1 512"; do
  set -- $cfg
  M4D_PUSH_CTAS_PER_SM=$1 M4D_PUSH_TILE_THREADS=$2 run $((29600 + RANDOM % 300)) > gpurun_out/r2_push_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_push_$1_$2.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('ctas/SM $1 threads $2: step', round(d['value'],3), 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'split0', round(t['split0_end']-t['split0_start'],3), 'split1', round(t['split1_end']-t['split1_start'],3), 'join_start', t['join_start'])"
done
