mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x -k "not multigpu" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b1e.log 2>&1; echo "b1 rc=$?"; grep metric gpurun_out/b1e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_layer'], d['roofline']['achieved'], d['roofline'].get('gemm2_tflops'), d['clocks'], d['e2e']['value'])"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm" --launch-skip 10 -c 3 -o gpurun_out/gemm_hint2 -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gemm_hint2.log 2>&1; echo "ncu rc=$?"
