# key_merge: GPU tests, then ncu per-kernel times of one 1e8-row step
timeout 300 python -m pytest tests/test_key_merge_gpu.py -q -x --timeout 200 2>&1 | tail -1
python tools/prof_km.py --steps 1 > gpurun_out/km_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"join|scatter|hist" -c 12 python tools/prof_km.py --steps 1 2>&1 | grep -E "^  [a-z<]|duration|inst_exec" | sed 's/(const.*//'
cat gpurun_out/km_plain.log
