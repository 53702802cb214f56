for h in 0 8 16 32 0 8 16 32; do
M4D_PULL_HOLD_MB=$h timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_hold_sweep.py 2>&1 | grep "hold=" | tee -a gpurun_out/p2p_hold2.txt
done
