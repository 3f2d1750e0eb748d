mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu.py -x -q -k "gemm_pair or moe_forward_vs_oracle" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --profile --steps 2 > gpurun_out/b1p3.log 2>&1; echo "prof pair rc=$?"; grep metric gpurun_out/b1p3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_layer'], d['roofline']['achieved'], d['roofline'].get('gemm2_tflops'), d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_pair" --launch-skip 6 -c 2 -o gpurun_out/gemm_pair3 -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair3.log 2>&1; echo "ncu rc=$?"
