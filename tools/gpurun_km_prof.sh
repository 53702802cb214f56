# per-kernel times (ncu launch list) of an in-process 2-rank key_merge step on one GPU
python tools/prof_km_world.py --world 2 > gpurun_out/kmw_plain.log 2>&1 || { cat gpurun_out/kmw_plain.log; exit 1; }
cat gpurun_out/kmw_plain.log
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"runs_|scatter|hist|join|group|scan" -c 60 python tools/prof_km_world.py --world 2 --steps 1 2>&1 | grep -E "^  [a-z<_]|duration|inst_exec|dram__" | sed 's/(const.*//' > gpurun_out/kmw_ncu.txt
cat gpurun_out/kmw_ncu.txt
