#!/bin/bash
# Round 2: headline-config parity (tests/test_gpu_headline.py) + bench --check.
mkdir -p gpurun_out
nproc > gpurun_out/r2_headline_nproc.txt
timeout 1500 python -m pytest tests/test_gpu_headline.py -x -q -s > gpurun_out/r2_headline_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_headline_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --check --no-e2e --no-cpu-baseline > gpurun_out/r2_headline_bench.json 2> gpurun_out/r2_headline_bench.err
echo "bench rc=$?"
tail -3 gpurun_out/r2_headline_pytest.log
