# Functional check of the driver's 8-rank default run on a 4-GPU box (2 ranks per GPU; timings meaningless):
# the default line (transpose_sum + key_merge sub-record with full-size parity, e2e, CPU baseline), then the reference arm
run() { N=$1; P=$2; shift 2; timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run 8 29581 --steps 3 --warmup 3 > gpurun_out/r2_f8.json 2> gpurun_out/r2_f8.err; echo f8=$?
tail -3 gpurun_out/r2_f8.err
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_f8.json') if l.startswith('{')][-1]); k=d['key_merge']
print('ts', d['value'], d['parity']['ok'], d.get('functional_check_only'), '| km', k['value'], k['parity'])"
