mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/fc_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fc_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus 8 --oversubscribe --tokens 32768 --steps 2 --warmup 3 --no-e2e > gpurun_out/fc_n8emul.log 2>&1; echo "n8 emul rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
