# NVFP4 path: quantiser / GEMM / layer / DWDP parity tests (each under its own timeout).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_nvfp4.py -q -x -k "quant" > gpurun_out/fp4_quant.log 2>&1; echo "quant rc=$?"; tail -5 gpurun_out/fp4_quant.log
timeout 300 python -m pytest tests/test_gpu_nvfp4.py -q -x -k "gemm" > gpurun_out/fp4_gemm.log 2>&1; echo "gemm rc=$?"; tail -25 gpurun_out/fp4_gemm.log
timeout 600 python -m pytest tests/test_gpu_nvfp4.py -q > gpurun_out/fp4_all.log 2>&1; echo "all rc=$?"; tail -30 gpurun_out/fp4_all.log
