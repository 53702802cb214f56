set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_ts_n1.json 2> gpurun_out/bench_ts_n1.err; echo "bench exit $?"; cat gpurun_out/bench_ts_n1.json | cut -c1-600
timeout 400 python bench.py --workload key_merge > gpurun_out/bench_km_n1.json 2> gpurun_out/bench_km_n1.err; echo "bench km exit $?"; cat gpurun_out/bench_km_n1.json | cut -c1-800
