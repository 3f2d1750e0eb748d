#!/bin/bash
# Round 2: the sm_100a MLA block -- parity tests, then native vs library timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/r2_mla_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_mla_pytest.log
tail -15 gpurun_out/r2_mla_pytest.log
timeout 600 python scripts/attn_bench.py > gpurun_out/r2_mla_bench.jsonl 2> gpurun_out/r2_mla_bench.err
echo "attn bench rc=$?"; cat gpurun_out/r2_mla_bench.jsonl; tail -5 gpurun_out/r2_mla_bench.err
