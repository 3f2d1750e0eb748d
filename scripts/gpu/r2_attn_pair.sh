#!/bin/bash
# Round 2: two-query-tile attention kernel (DWDP_ATTN_PAIR=1) vs the one-tile
# kernel on the same box: parity, block timing, kernel time (ncu launch list).
mkdir -p gpurun_out
for P in 1 0; do
  DWDP_ATTN_PAIR=$P timeout 900 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/r2_attn_pair$P.log 2>&1
  echo "pair=$P pytest rc=$?"; tail -1 gpurun_out/r2_attn_pair$P.log
done
for P in 1 0 1 0; do
  DWDP_ATTN_PAIR=$P timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mla_attn \
    python scripts/attn_once.py 2>/dev/null | grep mla_attn | tail -1 | awk -F'","' -v p=$P '{print "pair=" p, $NF}'
done
DWDP_ATTN_PAIR=1 timeout 600 python scripts/attn_bench.py > gpurun_out/r2_attn_pair_bench.jsonl 2> gpurun_out/r2_attn_pair_bench.err
echo "bench rc=$?"; cat gpurun_out/r2_attn_pair_bench.jsonl
