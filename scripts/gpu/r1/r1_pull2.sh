mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "dwdp or multigpu or non_divisible" 2>&1 | tail -2
for e in pull hybrid; do for sz in 67108864 1048576; do timeout 300 python scripts/pull_probe.py --engine $e --plans 3 --slice-size $sz 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['engine'], d['slice_size'], [round(p['gbs']) for p in d['plans']])"; done; done
