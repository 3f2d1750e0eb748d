#!/bin/bash
# Round 2 final HEAD: the whole multi-GPU test file on every GPU of the box.
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 2700 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > gpurun_out/r2_multigpu_final_n$NG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_multigpu_final_n$NG.log
tail -3 gpurun_out/r2_multigpu_final_n$NG.log
