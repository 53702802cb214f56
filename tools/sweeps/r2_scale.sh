# default bench line under torchrun at N=2 and N=4 (transpose_sum + key_merge sub-record), plus the reference arm
run() { N=$1; P=$2; shift 2; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N "$@"; }
run 2 29701 > gpurun_out/r2_scale_n2.json 2> gpurun_out/r2_scale_n2.err; echo n2=$?
run 4 29702 > gpurun_out/r2_scale_n4.json 2> gpurun_out/r2_scale_n4.err; echo n4=$?
run 4 29703 --impl reference > gpurun_out/r2_scale_ref_n4.json 2> gpurun_out/r2_scale_ref_n4.err; echo ref4=$?
for f in n2 n4; do python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_scale_$f.json') if l.startswith('{')][-1]); k=d['key_merge']
print('$f ts', round(d['value'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), '| km', round(k['value'],3), 'frac', round(k['roofline']['frac'],3), 'parity', k['parity']['digest_equal'], 'e2e', round(k['e2e']['value'],1), 'cpu', round(k['cpu_baseline']['value'],1))"; done
tail -c 600 gpurun_out/r2_scale_ref_n4.json
