# Round-1 closing refresh on one 4-GPU box: transpose_sum N=2/4, storm N=2/4 (ours), reference arm N=1 (transpose_sum)
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run 2 29531 --steps 10 --warmup 3 > gpurun_out/ts_n2.json 2> gpurun_out/ts_n2.err; echo ts_n2=$?
run 4 29532 --steps 10 --warmup 3 > gpurun_out/ts_n4.json 2> gpurun_out/ts_n4.err; echo ts_n4=$?
run 2 29533 --workload storm --steps 3 --warmup 3 > gpurun_out/storm_n2.json 2> gpurun_out/storm_n2.err; echo storm_n2=$?
run 4 29534 --workload storm --steps 3 --warmup 3 > gpurun_out/storm_n4.json 2> gpurun_out/storm_n4.err; echo storm_n4=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err; echo ref_n1=$?
