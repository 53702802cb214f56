#!/bin/bash
# Tile scatter with bucket-major warp counters (vector loads in the per-tile scan): tests, N=1 and N=2 timing.
exec > gpurun_out/r2_tile_bmajor.log 2>&1
timeout 900 python -m pytest tests/test_key_merge_gpu.py tests/test_multiprocess_gpu.py -x -q -k "key_merge or km or shuffle or push or partition or owner" 2>&1 | tail -2
M4D_TILE_RANK=ballot timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q 2>&1 | tail -1
M4D_TILE_THREADS=1024 timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q -k "single_gpu or skew" 2>&1 | tail -1
M4D_TILE_THREADS=256 timeout 600 python -m pytest tests/test_key_merge_gpu.py -x -q -k "single_gpu or skew" 2>&1 | tail -1
for rep in 1 2; do timeout 300 python tools/km_time.py --tag "bucket-major"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 2 --workload key_merge --skip-cpu --skip-e2e --steps 10 > gpurun_out/r2_bmajor_n2.json 2>/dev/null
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_bmajor_n2.json') if l.startswith('{')][-1]); print('N=2', round(d['ms_per_step'],3), d['parity']['digest_equal'] if 'parity' in d else '')"
