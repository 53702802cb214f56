# key_merge bench lines at N=1,2,4 (run under gpurun --gpus 4)
python bench.py --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n1.json 2> gpurun_out/km_n1.err; echo km_n1=$?
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n$N.json 2> gpurun_out/km_n$N.err; echo km_n$N=$?
done
