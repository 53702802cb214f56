# Functional check of the driver's 8-rank runs on a 4-GPU box (2 ranks per GPU; timings meaningless)
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run 8 29571 --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/f8_ts.json 2> gpurun_out/f8_ts.err; echo ts8=$?
run 8 29572 --workload key_merge --rows 20000000 --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/f8_km.json 2> gpurun_out/f8_km.err; echo km8=$?
M4D_MERGE_SHUFFLE=pull run 8 29573 --workload key_merge --rows 20000000 --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/f8_km_pull.json 2> gpurun_out/f8_km_pull.err; echo km8pull=$?
run 8 29574 --workload storm --steps 2 --warmup 3 > gpurun_out/f8_storm.json 2> gpurun_out/f8_storm.err; echo storm8=$?
for f in f8_ts f8_km f8_km_pull f8_storm; do tail -1 gpurun_out/$f.json | cut -c1-400; tail -2 gpurun_out/$f.err; done
