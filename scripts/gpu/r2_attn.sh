#!/bin/bash
# Round 2: MLA core with the O accumulator kept in TMEM (lazy rescale) --
# parity tests, block timing vs the library arm, ncu of the attention kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/r2_attn_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_attn_pytest.log
tail -4 gpurun_out/r2_attn_pytest.log
timeout 600 python scripts/attn_bench.py > gpurun_out/r2_attn_bench.jsonl 2> gpurun_out/r2_attn_bench.err
echo "attn bench rc=$?"; cat gpurun_out/r2_attn_bench.jsonl; tail -3 gpurun_out/r2_attn_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_attn_launches.csv \
  python scripts/attn_once.py > gpurun_out/r2_attn_launches.log 2>&1
echo "ncu launches rc=$?"; grep mla_attn gpurun_out/r2_attn_launches.csv | head -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mla_attn -c 1 -f -o gpurun_out/r2_ncu_attn \
  python scripts/attn_once.py > gpurun_out/r2_ncu_attn.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/r2_ncu_attn.log
