# 2-GPU benches (run under gpurun --gpus 2): p2p ours/reference, transpose_sum and key_merge at N=2
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29523 --workload p2p --steps 1 --warmup 3 > gpurun_out/p2p_ours.json 2> gpurun_out/p2p_ours.err; echo p2p_ours=$?
run 29524 --workload p2p --impl reference --steps 1 --warmup 1 > gpurun_out/p2p_ref.json 2> gpurun_out/p2p_ref.err; echo p2p_ref=$?
run 29525 --steps 10 --warmup 3 > gpurun_out/ts_n2.json 2> gpurun_out/ts_n2.err; echo ts_n2=$?
run 29526 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
