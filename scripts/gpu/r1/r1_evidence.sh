mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/b1.log 2>&1; echo "b1 rc=$?"; grep metric gpurun_out/b1.log | head -c 1500; echo
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29512 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/pf2.log 2>&1; echo "pf2 rc=$?"; grep metric gpurun_out/pf2.log | head -c 800; echo
for e in pull copy; do timeout 300 python scripts/pull_probe.py --engine $e > gpurun_out/probe_$e.log 2>&1; echo "probe $e rc=$?"; tail -2 gpurun_out/probe_$e.log; done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name tma_pull_kernel -c 1 -o gpurun_out/pull_full -f python scripts/pull_probe.py --plans 1 > gpurun_out/ncu_pull.log 2>&1; echo "ncu pull rc=$?"
timeout 300 python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof1.log 2>&1; echo "prof1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"permute_scatter_kernel|combine_kernel|topk_kernel|router_quant_kernel" -c 4 -o gpurun_out/nongemm_full -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ng.log 2>&1; echo "ncu ng rc=$?"
