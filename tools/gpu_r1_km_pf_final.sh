# key_merge lines after the join L2 prefetch (N=1/2/4 weak, M-S strong), join variant check, launch list, ncu full of the join, GPU tests, smoke
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 400 python bench.py --workload key_merge --steps 10 --warmup 3 > gpurun_out/km_n1.json 2> gpurun_out/km_n1.err; echo km_n1=$?
M4D_JOIN=small timeout 400 python bench.py --workload key_merge --steps 10 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/km_n1_small.json 2>/dev/null; echo km_small=$?
run 2 29563 --workload key_merge --steps 10 --warmup 3 > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
run 4 29564 --workload key_merge --steps 10 --warmup 3 > gpurun_out/km_n4.json 2> gpurun_out/km_n4.err; echo km_n4=$?
run 2 29601 --workload key_merge --rows 50000000 --steps 10 --warmup 3 --skip-cpu > gpurun_out/km_ms_n2.json 2>/dev/null; echo ms2=$?
run 4 29602 --workload key_merge --rows 25000000 --steps 10 --warmup 3 --skip-cpu > gpurun_out/km_ms_n4.json 2>/dev/null; echo ms4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/km_launches_n1.csv python bench.py --workload key_merge --steps 2 --warmup 1 --skip-cpu --skip-e2e > gpurun_out/km_ncu_n1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"join" -c 1 -o gpurun_out/km_join_full -f python tools/prof_km.py --steps 1 > gpurun_out/km_join_full.log 2>&1; echo ncufull=$?
