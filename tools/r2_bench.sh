# default bench line (transpose_sum + key_merge sub-record) at N=1, reference arm, the 5e7 parity test
timeout 900 python bench.py > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo bench=$?; tail -3 gpurun_out/r2_bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref_n1.json 2> gpurun_out/r2_bench_ref_n1.err; echo ref=$?; tail -3 gpurun_out/r2_bench_ref_n1.err
timeout 600 python -m pytest tests/test_key_merge_gpu.py -q -k full_scale > gpurun_out/r2_full_scale.log 2>&1; echo fs=$?; tail -2 gpurun_out/r2_full_scale.log
