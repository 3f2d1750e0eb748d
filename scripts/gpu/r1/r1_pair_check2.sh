mkdir -p gpurun_out
DWDP_VERBOSE=1 timeout 180 python -m pytest tests/test_gpu.py -x -q -k "gemm_pair" 2>&1 | grep -E "dwdp:|passed|failed" | head -5
timeout 600 python bench.py --no-cpu-baseline --profile --steps 2 > gpurun_out/b1p2.log 2>&1; echo "prof pair rc=$?"; grep metric gpurun_out/b1p2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_ms_per_layer'], d['roofline']['achieved'], d['roofline'].get('gemm2_tflops'), d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_pair" --launch-skip 6 -c 2 -o gpurun_out/gemm_pair -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair.log 2>&1; echo "ncu rc=$?"
