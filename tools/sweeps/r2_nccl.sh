# key_merge N=2 / N=4: NCCL all-to-all shuffle vs the fused push (trace of one step each)
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $1 --workload key_merge --skip-cpu --skip-e2e --steps 5; }
for n in 2 4; do for sh in nccl push; do
  M4D_MERGE_SHUFFLE=$sh run $n > gpurun_out/r2_sh_${n}_$sh.json 2> gpurun_out/r2_sh_${n}_$sh.err
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2_sh_${n}_$sh.json') if l.startswith('{')][-1]); print('N=$n $sh', round(d['value'],3), d['parity']['digest_equal'] if d.get('parity') else None, d['roofline']['trace_ms'])" || tail -5 gpurun_out/r2_sh_${n}_$sh.err
done; done
