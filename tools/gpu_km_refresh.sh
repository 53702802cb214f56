# key_merge bench lines at N=1/2/4 (weak) and M-S strong at N=2/4, plus per-kernel ncu of an
# in-process 2-rank step and the N=1 launch list (4-GPU box; JSON lines into gpurun_out/)
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
python bench.py --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n1.json 2> gpurun_out/km_n1.err; echo km_n1=$?
run 2 29563 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
run 4 29564 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n4.json 2> gpurun_out/km_n4.err; echo km_n4=$?
run 2 29601 --workload key_merge --rows 50000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n2.json 2>/dev/null; echo ms2=$?
run 4 29602 --workload key_merge --rows 25000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n4.json 2>/dev/null; echo ms4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/km_launches_n1.csv python bench.py --workload key_merge --steps 2 --warmup 1 --skip-cpu --skip-e2e > gpurun_out/km_ncu_n1.log 2>&1; echo ncu1=$?
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"runs_|scatter|hist|join" -c 40 python tools/prof_km_world.py --world 2 --steps 1 2>&1 | grep -E "^  [a-z<_]|duration|inst_exec|dram__" | sed 's/(const.*//' > gpurun_out/kmw_ncu.txt; echo ncuw=$?
