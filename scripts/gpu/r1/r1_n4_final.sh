mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/n4f_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/n4f_tests.log
for e in pull copy; do timeout 300 python scripts/pull_probe.py --gpus 4 --engine $e --plans 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('probe4', d['engine'], [(round(p['gbs']), p['other_ranks_gbs']) for p in d['plans']])"; done
timeout 300 python scripts/pull_probe.py --gpus 2 --engine pull --plans 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('probe2', d['engine'], [(round(p['gbs']), p['other_ranks_gbs']) for p in d['plans']])"
timeout 2400 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 --out gpurun_out/sweep_n4_final.jsonl > gpurun_out/sweep_n4_final.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_final.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), round(d['step_roofline_frac'],3), d['clocks']['sm_mhz'])"
