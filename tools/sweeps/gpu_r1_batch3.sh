for b in 16777216 33554432 16777216; do
M4D_PULL_BATCH_BYTES=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_hold_sweep.py 2>&1 | grep "batch=" | sed "s/^/bytes=$b /" | tee -a gpurun_out/p2p_batch3.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload p2p --steps 1 --warmup 3 > gpurun_out/p2p_ours.json 2> gpurun_out/p2p_ours.err; echo p2p_ours=$?
timeout 800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
