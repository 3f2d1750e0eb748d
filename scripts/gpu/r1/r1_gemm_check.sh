mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b1c.log 2>&1; echo "b1 rc=$?"; grep metric gpurun_out/b1c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_layer'], d['roofline']['achieved'], d['roofline'].get('gemm2_tflops'), d['clocks'], d['e2e']['value'])"
timeout 300 python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof1c.log 2>&1; echo "prof rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm|permute_scatter|permute_scan" --launch-skip 16 -c 5 -o gpurun_out/gemm_fix -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm_fix.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --dtype fp8 --no-cpu-baseline > gpurun_out/b1fp8.log 2>&1; echo "fp8 rc=$?"; grep metric gpurun_out/b1fp8.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_layer'], d['roofline']['achieved'], d['roofline'].get('gemm2_tflops'), d['clocks'])"
timeout 300 python -m pytest tests -q -m gpu -x -k "not multigpu" 2>&1 | tail -2
