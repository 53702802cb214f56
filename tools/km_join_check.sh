# key_merge join check: GPU tests, then ncu time/instructions of join_kernel at 1e8 rows/side
timeout 300 python -m pytest tests/test_key_merge_gpu.py -q -x --timeout 200 2>&1 | tail -1
python tools/prof_km.py --steps 1 > gpurun_out/km_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"join" -c 1 python tools/prof_km.py --steps 1 2>&1 | grep -E "duration|inst_executed|warps_active"
cat gpurun_out/km_plain.log
