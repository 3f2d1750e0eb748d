#!/bin/bash
# Round 2: routing parity after the router_quant rewrite, then the ncu evidence.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_headline.py -q -x -p no:cacheprovider -k "route or moe_forward or headline_layer" > gpurun_out/r2_quant_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_quant_pytest.log; tail -2 gpurun_out/r2_quant_pytest.log
bash scripts/gpu/r2_ncu.sh
