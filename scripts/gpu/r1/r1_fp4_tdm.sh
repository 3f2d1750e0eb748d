# §8(f) row 4: TDM / slice-size tuning for NVFP4 at N=4 (MNT 32K, CV 0.2, copy engine): slices 1-64 MB and TDM off.
mkdir -p gpurun_out
: > gpurun_out/fp4_tdm.jsonl
for cfg in "--slice-size 1048576" "--slice-size 4194304" "--slice-size 16777216" "--slice-size 67108864" "--no-tdm"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29593 bench.py --gpus 4 --dtype nvfp4 --tokens 32768 --cv 0.2 --engine copy --no-e2e --no-dep --steps 4 --warmup 3 $cfg > gpurun_out/fp4_tdm.log 2>&1; echo "$cfg rc=$?"
grep '"metric"' gpurun_out/fp4_tdm.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); rec={'cfg': '$cfg', 'tokens_per_s_per_gpu': d['tokens_per_s_per_gpu'], 'exposed_ms': d['exposed_prefetch_ms_per_layer'], 'prefetch': d['prefetch'], 'moe_ms': d['kernel_ms_per_layer']['moe'], 'clocks': d['clocks']}
print(json.dumps(rec)); open('gpurun_out/fp4_tdm.jsonl','a').write(json.dumps(rec)+'\n')"
done
