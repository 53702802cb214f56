# round-2 launch list of the default bench command (transpose_sum + key_merge sub-record) with DRAM bytes
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_default.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/r2_launches_default.log 2>&1; echo ncu=$?
