nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r2_base_pytest.log
timeout 400 python bench.py --workload key_merge --skip-cpu > gpurun_out/r2_base_km.json 2> gpurun_out/r2_base_km.err; echo km=$?; cut -c1-400 gpurun_out/r2_base_km.json
