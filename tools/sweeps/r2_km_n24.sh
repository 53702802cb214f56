timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "km or key_merge or shuffle or worker or push or pull" > gpurun_out/r2_km24_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2_km24_tests.log
bash tools/sweeps/r2_push_sms.sh
