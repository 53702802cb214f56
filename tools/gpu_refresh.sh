# Refresh the round's bench lines on a 4-GPU box: transpose_sum and key_merge at N=1,2,4
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
python bench.py > gpurun_out/ts_n1.json 2> gpurun_out/ts_n1.err; echo ts_n1=$?
run 2 29561 --steps 10 --warmup 3 > gpurun_out/ts_n2.json 2> gpurun_out/ts_n2.err; echo ts_n2=$?
run 4 29562 --steps 10 --warmup 3 > gpurun_out/ts_n4.json 2> gpurun_out/ts_n4.err; echo ts_n4=$?
python bench.py --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n1.json 2> gpurun_out/km_n1.err; echo km_n1=$?
run 2 29563 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
run 4 29564 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n4.json 2> gpurun_out/km_n4.err; echo km_n4=$?
python bench.py --impl reference > gpurun_out/ts_ref.json 2> gpurun_out/ts_ref.err; echo ts_ref=$?
