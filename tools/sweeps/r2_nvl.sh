# NVLink counters of the cross-GPU kernels (in-process 2-GPU drivers) + key_merge N=2 bench line
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum"
for w in km ts p2p; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_nvl_$w.csv python tools/prof_nvlink.py $w > gpurun_out/r2_nvl_$w.log 2>&1; echo $w=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --workload key_merge --skip-cpu > gpurun_out/r2_km_n2.json 2> gpurun_out/r2_km_n2.err; echo km2=$?
