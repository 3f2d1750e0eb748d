# Redundant placement (build_placement extra) at N=4, bf16, MNT 32K, CV 0.2: fewer bytes to pull per layer.
mkdir -p gpurun_out
: > gpurun_out/redundancy2.jsonl
for ex in 64 32; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29597 bench.py --gpus 4 --tokens 32768 --cv 0.2 --extra-redundancy $ex --no-e2e --steps 4 --warmup 3 > gpurun_out/red.log 2>&1; echo "extra $ex rc=$?"
grep '"metric"' gpurun_out/red.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); dep=d['dep_baseline'] or {}
rec={'extra': $ex, 'tokens_per_s_per_gpu': d['tokens_per_s_per_gpu'], 'dwdp_over_dep': dep.get('dwdp_over_dep'), 'dep_tokens_per_s_per_gpu': dep.get('tokens_per_s_per_gpu'), 'exposed_ms': d['exposed_prefetch_ms_per_layer'], 'prefetch': d['prefetch'], 'moe_ms': d['kernel_ms_per_layer']['moe'], 'engine': d['config']['prefetch_engine'], 'hbm_gb': d['hbm_gb'], 'sm_mhz': d['clocks']['sm_mhz']}
print(json.dumps(rec)); open('gpurun_out/redundancy2.jsonl','a').write(json.dumps(rec)+'\n')"
done
