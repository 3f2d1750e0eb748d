for e in copy pull hybrid; do timeout 300 python scripts/pull_probe.py --engine $e --plans 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['engine'], d['slice_size'], [round(p['gbs']) for p in d['plans']])"; done
timeout 300 python scripts/pull_probe.py --engine hybrid --plans 3 --slice-size 16777216 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['engine'], d['slice_size'], [round(p['gbs']) for p in d['plans']])"
timeout 300 python -m pytest tests/test_gpu.py -q -x -k "dwdp_group" 2>&1 | tail -2
