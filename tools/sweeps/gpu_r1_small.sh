for v in default 262145 1048577 default 262145 1048577; do
  ( [ $v != default ] && export M4D_SMALL_PULL=$v; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/p2p_small_sweep.py 2>&1 | grep "small_pull=" | tee -a gpurun_out/p2p_small2.txt )
done
