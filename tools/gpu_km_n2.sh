# key_merge: GPU tests + bench at N=2 (phase breakdown in roofline.phases)
timeout 400 python -m pytest tests/test_key_merge_gpu.py -q -x --timeout 300 2>&1 | tail -1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --workload key_merge --steps 5 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
