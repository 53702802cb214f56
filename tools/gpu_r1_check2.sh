# Check after the single-call pointer query: GPU tests, smoke, p2p line (2 GPUs), N=1 transpose_sum line
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload p2p --steps 1 --warmup 3 > gpurun_out/p2p_ours.json 2> gpurun_out/p2p_ours.err; echo p2p_ours=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/p2p_timeline.py 4194304 2>&1 | grep "rank 0" | tee gpurun_out/p2p_timeline2.txt
timeout 400 python bench.py > gpurun_out/bench_ts_n1.json 2> gpurun_out/bench_ts_n1.err; echo "bench exit $?"
