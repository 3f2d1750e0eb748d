#!/bin/bash
# Round 2: full single-GPU suite, smoke, default N=1 bench (parity check and
# CPU baselines on), reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_suite.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gpu_suite.log; tail -3 gpurun_out/r2_gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
nproc > gpurun_out/r2_nproc.txt
