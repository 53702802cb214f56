for b in 8 4 16 2 8 4 16 2; do
M4D_PULL_BATCH=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_hold_sweep.py 2>&1 | grep "batch=" | tee -a gpurun_out/p2p_batch.txt
done
