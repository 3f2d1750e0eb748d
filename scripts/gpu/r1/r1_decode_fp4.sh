# Config-5 decode points with NVFP4 experts at N=2 (split and merged fetch), beside the fp8 sweep.
mkdir -p gpurun_out
timeout 2400 python scripts/sweep_decode.py --gpus 2 --batch 256,4096 --zipf 0,1.2 --fetch split,merged --dtype nvfp4 --out gpurun_out/sweep_decode_fp4_n2.jsonl > gpurun_out/sweep_decode_fp4_n2.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_decode_fp4_n2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    print({k: (round(v,3) if isinstance(v,float) else v) for k,v in d.items() if k not in ('clocks',)})" | cut -c1-300
