# Refresh the round's bench lines on a 4-GPU box (JSON lines into gpurun_out/)
run() { N=$1; P=$2; shift 2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
python bench.py > gpurun_out/ts_n1.json 2> gpurun_out/ts_n1.err; echo ts_n1=$?
run 2 29561 --steps 10 --warmup 3 > gpurun_out/ts_n2.json 2> gpurun_out/ts_n2.err; echo ts_n2=$?
run 4 29562 --steps 10 --warmup 3 > gpurun_out/ts_n4.json 2> gpurun_out/ts_n4.err; echo ts_n4=$?
python bench.py --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n1.json 2> gpurun_out/km_n1.err; echo km_n1=$?
run 2 29563 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n2.json 2> gpurun_out/km_n2.err; echo km_n2=$?
run 4 29564 --workload key_merge --steps 5 --warmup 3 > gpurun_out/km_n4.json 2> gpurun_out/km_n4.err; echo km_n4=$?
run 2 29565 --workload p2p --steps 1 --warmup 3 > gpurun_out/p2p_n2.json 2> gpurun_out/p2p_n2.err; echo p2p=$?
run 2 29566 --workload p2p --impl reference --steps 1 --warmup 1 > gpurun_out/p2p_ref.json 2> gpurun_out/p2p_ref.err; echo p2p_ref=$?
run 2 29567 --workload storm --steps 3 --warmup 3 > gpurun_out/storm_n2.json 2> gpurun_out/storm_n2.err; echo storm2=$?
run 4 29568 --workload storm --steps 3 --warmup 3 > gpurun_out/storm_n4.json 2> gpurun_out/storm_n4.err; echo storm4=$?
python bench.py --impl reference > gpurun_out/ts_ref.json 2> gpurun_out/ts_ref.err; echo ts_ref=$?
python bench.py --impl reference --workload key_merge > gpurun_out/km_ref.json 2> gpurun_out/km_ref.err; echo km_ref=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
# key_merge M-S (strong: 1e8 rows per side in total) at N=2 and N=4
run 2 29601 --workload key_merge --rows 50000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n2.json 2>/dev/null; echo ms2=$?
run 4 29602 --workload key_merge --rows 25000000 --steps 5 --warmup 3 --skip-cpu > gpurun_out/km_ms_n4.json 2>/dev/null; echo ms4=$?
