# 4-GPU checks (gpurun --gpus 4): transpose_sum and key_merge benches at N=4, storm at N=4
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 4 "${@:2}"; }
run 29531 --steps 10 --warmup 3 > gpurun_out/ts_n4.json 2> gpurun_out/ts_n4.err; echo ts_n4=$?
run 29532 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n4.json 2> gpurun_out/km_n4.err; echo km_n4=$?
run 29533 --workload storm --steps 3 --warmup 3 > gpurun_out/storm_n4.json 2> gpurun_out/storm_n4.err; echo storm_n4=$?
run 29534 --workload storm --impl reference --steps 2 --warmup 1 > gpurun_out/storm_ref_n4.json 2> gpurun_out/storm_ref_n4.err; echo storm_ref_n4=$?
