timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "km or key_merge or shuffle or worker or push or pull or spec" > gpurun_out/r2_fine_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r2_fine_tests.log
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e --steps 5; }
for n in 2 4; do for f in 1 0; do
  M4D_MERGE_FINE=$f run $n > gpurun_out/r2_fine_${n}_$f.json 2> gpurun_out/r2_fine_${n}_$f.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_fine_${n}_$f.json') if l.startswith('{')][-1]); print('N=$n fine=$f', round(d['value'],3), d['parity']['digest_equal'], d['roofline']['trace_ms'])" || tail -3 gpurun_out/r2_fine_${n}_$f.err
done; done
