mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr=127.0.0.1 --master-port=29531 bench.py --gpus 8 --oversubscribe --tokens 32768 --steps 2 --warmup 3 --no-e2e > gpurun_out/n8emul.log 2>&1; echo "n8 emul rc=$?"
grep metric gpurun_out/n8emul.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['config']['prefetch_engine'], d['prefetch'], round(d['exposed_prefetch_ms_per_layer'],2), d['report']['dwdp']['p2p_fully_overlapped'])" || tail -30 gpurun_out/n8emul.log
