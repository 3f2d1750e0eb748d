#!/bin/bash
# Full -m gpu suite on the current build (compute-sanitizer is closed on this
# GPU pool: profiles/r2_compute_sanitizer_refused.txt).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_suite.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gpu_suite.log
tail -3 gpurun_out/r2_gpu_suite.log
