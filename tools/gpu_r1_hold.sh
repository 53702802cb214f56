# Pull-hold sweep (M4D_PULL_HOLD) on the osu_bw window timeline, then key_merge with the join prefetch default
for h in 0 1 2 3 4; do for n in 4194304 16777216; do
echo "hold=$h size=$n" | tee -a gpurun_out/p2p_hold.txt
M4D_PULL_HOLD=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_timeline.py $n 2>&1 | grep "rank 0" | tee -a gpurun_out/p2p_hold.txt
done; done
timeout 400 python bench.py --workload key_merge > gpurun_out/bench_km_n1.json 2> gpurun_out/bench_km_n1.err; echo "bench km exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --workload key_merge > gpurun_out/bench_km_n2.json 2> gpurun_out/bench_km_n2.err; echo km_n2=$?
