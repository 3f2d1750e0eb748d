mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/n4_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/n4_tests.log
timeout 2400 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 --out gpurun_out/sweep_n4_v2.jsonl > gpurun_out/sweep_n4_v2.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_v2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), d['clocks']['sm_mhz'])"
