# N=2 / N=4: push scatter confined to a subset of SMs so the previous side's receiver split runs beside it
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e --steps 5; }
for n in 2 4; do for sms in 96 112; do
  M4D_PUSH_SMS=$sms run $n > gpurun_out/r2_pushsms_${n}_$sms.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_pushsms_${n}_$sms.json') if l.startswith('{')][-1]); t=d['roofline']['trace_ms']
print('N=$n push SMs $sms: step', round(d['value'],3), 'push0', round(t['push0_end']-t['push0_start'],3), 'push1', round(t['push1_end']-t['push1_start'],3), 'split0 end', t['split0_end'], 'join_start', t['join_start'])"
done; done
