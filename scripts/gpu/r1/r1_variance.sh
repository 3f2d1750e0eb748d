# Run-to-run variance of the headline bench on one box (3 back-to-back default runs, N=1).
mkdir -p gpurun_out
: > gpurun_out/variance.jsonl
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/var.log 2>&1; grep '"metric"' gpurun_out/var.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); rec={'run': $i, 'value': d['value'], 'e2e': d['e2e']['value'], 'gemm1_frac': d['roofline']['frac'], 'moe_ms': d['kernel_ms_per_layer']['moe'], 'clocks': d['clocks']}
print(json.dumps(rec)); open('gpurun_out/variance.jsonl','a').write(json.dumps(rec)+'\n')"
done
