# NVFP4 config-4 sweep at N=4 (DWDP vs same-box DEP), plus bf16 reference points at CV 0.2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "2" > gpurun_out/fp4_mg4.log 2>&1; echo "mg rc=$?"; tail -2 gpurun_out/fp4_mg4.log
timeout 2400 python scripts/sweep.py --gpus 4 --cv 0,0.1,0.2,0.3 --tokens 32768,65536 --steps 4 --warmup 3 --extra "--dtype nvfp4" --out gpurun_out/sweep_n4_fp4.jsonl > gpurun_out/sweep_n4_fp4.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_n4_fp4.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d); continue
    print(d['mnt'], d['cv'], round(d['dwdp_tokens_per_s_per_gpu']), round(d['dep_tokens_per_s_per_gpu']), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['engine'], round(d['prefetch_gbs'] or 0), round(d['step_roofline_frac'],3), d['clocks']['sm_mhz'])"
