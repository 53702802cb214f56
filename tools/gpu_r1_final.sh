# Round-1 re-entry check: GPU tests, smoke, N=1 bench lines, 2-GPU p2p line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_ts_n1.json 2> gpurun_out/bench_ts_n1.err; echo "bench exit $?"; cut -c1-600 gpurun_out/bench_ts_n1.json
timeout 400 python bench.py --workload key_merge > gpurun_out/bench_km_n1.json 2> gpurun_out/bench_km_n1.err; echo "bench km exit $?"; cut -c1-800 gpurun_out/bench_km_n1.json
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 bench.py --gpus 2 "${@:2}"; }
run 29541 --workload p2p --steps 1 --warmup 3 --skip-cpu > gpurun_out/p2p_ours.json 2> gpurun_out/p2p_ours.err; echo p2p_ours=$?
run 29542 --workload key_merge > gpurun_out/bench_km_n2.json 2> gpurun_out/bench_km_n2.err; echo km_n2=$?
