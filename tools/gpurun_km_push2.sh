# push scatter CTA size x push buckets with atomic ranking, N=2 and N=4
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e ; }
for N in 2 4; do for cfg in "1024 256" "512 256" "1024 128" "512 128"; do
  set -- $cfg
  M4D_PUSH_TILE_THREADS=$1 M4D_PUSH_BUCKETS=$2 run $N > gpurun_out/kmp_$1_$2_n$N.json 2> gpurun_out/kmp_$1_$2_n$N.err
  python -c "
import json
d=json.loads(open('gpurun_out/kmp_$1_$2_n$N.json').read().strip().splitlines()[-1]); r=d['roofline']
print('N=$N pt=$1 pb=$2', round(d['value'],3), d['config']['digest'][0], {k: round(v['ms'],3) for k, v in r['kernel_groups'].items()})"
done; done
