# N=4 final build: multi-GPU parity, default bench (bf16, MNT 64K), and the NVFP4 config-4 sweep (CV 0-0.3).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/n4f3_mg.log 2>&1; echo "mg rc=$?"; tail -2 gpurun_out/n4f3_mg.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29583 bench.py --gpus 4 > gpurun_out/n4f3_b.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/n4f3_b.log > gpurun_out/n4f3_b.json
python -c "import json; d=json.load(open('gpurun_out/n4f3_b.json')); print(round(d['value']), round(d['tokens_per_s_per_gpu']), d['dep_baseline'] and round(d['dep_baseline']['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['e2e'] and round(d['e2e']['value']), d['config']['prefetch_engine'], d['clocks']['sm_mhz'])"
timeout 2400 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 --extra "--dtype nvfp4" --out gpurun_out/sweep_n4_fp4_final3.jsonl > gpurun_out/sweep_n4_fp4_final3.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_fp4_final3.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), round(d['step_roofline_frac'],3), d['clocks']['sm_mhz'])"
