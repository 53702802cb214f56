# key_merge tile layout: N=1 parity tests, bench line, launch list
timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q -k "single_gpu or multiset or skewed or duplicate or large_config or spec_application" > gpurun_out/r2_km_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/r2_km_tests.log
timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_km_n1.json 2> gpurun_out/r2_km_n1.err; echo km=$?; cut -c1-200 gpurun_out/r2_km_n1.json; tail -3 gpurun_out/r2_km_n1.err
M4D_MERGE_LAYOUT=bucket timeout 300 python bench.py --workload key_merge --skip-cpu --skip-e2e > gpurun_out/r2_km_n1_bucket.json 2>&1; echo kmb=$?; cut -c1-200 gpurun_out/r2_km_n1_bucket.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_km_launches.csv python bench.py --workload key_merge --steps 2 --warmup 3 --skip-cpu --skip-e2e > /dev/null 2>&1; echo ncu=$?
