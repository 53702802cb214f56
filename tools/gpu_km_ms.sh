# key_merge M-S (strong: 1e8 rows per side in total) at N=2 and N=4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --workload key_merge --rows 50000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n2.json 2>/dev/null; echo n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --workload key_merge --rows 25000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n4.json 2>/dev/null; echo n4=$?
