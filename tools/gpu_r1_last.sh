# Closing check at HEAD: smoke, default bench line, key_merge N=1 line
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_ts_n1.json 2> gpurun_out/bench_ts_n1.err; echo bench=$?; cut -c1-300 gpurun_out/bench_ts_n1.json
timeout 400 python bench.py --workload key_merge > gpurun_out/bench_km_n1.json 2> gpurun_out/bench_km_n1.err; echo km=$?; cut -c1-300 gpurun_out/bench_km_n1.json
