mkdir -p gpurun_out
timeout 2400 python scripts/sweep_decode.py --gpus 4 --batch 256,4096 --zipf 0,1.2 --fetch split --steps 3 --warmup 3 --out gpurun_out/sweep_decode_n4.jsonl > gpurun_out/sweep_decode_n4.log 2>&1; echo "decode split rc=$?"
timeout 1200 python scripts/sweep_decode.py --gpus 4 --batch 4096 --zipf 1.2 --fetch merged --steps 3 --warmup 3 --out gpurun_out/sweep_decode_n4.jsonl >> gpurun_out/sweep_decode_n4.log 2>&1; echo "decode merged rc=$?"
cat gpurun_out/sweep_decode_n4.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'error' in d: print('ERR', d['batch'], d['error'][-300:]); continue
    print(d['fetch'], d['batch'], d['zipf'], round(d['dwdp_ms_per_step'],1), round(d['dep_ms_per_step'],1), round(d['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],2), d['engine'], round(d['prefetch_gbs']), d['routing']['count_cv'] and round(d['routing']['count_cv'],2))"
