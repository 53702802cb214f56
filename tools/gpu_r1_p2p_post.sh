# osu_bw after launching receive-side matched pulls during the post loop; then the p2p bench line and the transport GPU tests
for i in 1 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_hold_sweep.py 2>&1 | grep "hold=" | tee -a gpurun_out/p2p_post.txt
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/p2p_timeline.py 4194304 2>&1 | grep "rank 0" | tee -a gpurun_out/p2p_post.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload p2p --steps 1 --warmup 3 > gpurun_out/p2p_ours.json 2> gpurun_out/p2p_ours.err; echo p2p_ours=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
