# Pull-kernel width (CTAs) vs MoE interference: NVFP4 and bf16, N=4, MNT 32K, CV 0.2.
mkdir -p gpurun_out
: > gpurun_out/pull_ctas.jsonl
for dt in nvfp4 bf16; do
for c in 32 64 148; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29596 bench.py --gpus 4 --dtype $dt --tokens 32768 --cv 0.2 --engine pull --pull-ctas $c --no-e2e --no-dep --steps 4 --warmup 3 > gpurun_out/pc.log 2>&1; echo "$dt $c rc=$?"
grep '"metric"' gpurun_out/pc.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); rec={'dtype': '$dt', 'pull_ctas': $c, 'tokens_per_s_per_gpu': d['tokens_per_s_per_gpu'], 'exposed_ms': d['exposed_prefetch_ms_per_layer'], 'gbs': d['prefetch']['gbs'], 'moe_ms': d['kernel_ms_per_layer']['moe'], 'sm_mhz': d['clocks']['sm_mhz']}
print(json.dumps(rec)); open('gpurun_out/pull_ctas.jsonl','a').write(json.dumps(rec)+'\n')"
done; done
