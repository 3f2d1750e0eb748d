for e in pull copy hybrid; do for c in 0 32768; do timeout 300 python scripts/pull_probe.py --engine $e --plans 2 --with-compute $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['engine'], [(round(p['gbs']), p['compute_ms'] and round(p['compute_ms'],1)) for p in d['plans']])"; done; done
nvidia-smi -q -d POWER | grep -i -E "limit|draw" | head -8
