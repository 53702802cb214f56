bash tools/km_join_pf_sweep.sh 2>&1 | tee gpurun_out/km_join_pf_sweep.txt
for n in 4194304 16777216; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_timeline.py $n 2>&1 | grep rank | tee -a gpurun_out/p2p_timeline.txt
done
