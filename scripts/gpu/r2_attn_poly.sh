#!/bin/bash
# Round 2: MLA core -- exp2 split between MUFU and an FMA-pipe polynomial (A/B).
mkdir -p gpurun_out
for P in 0 1 2 4; do
  DWDP_ATTN_POLY=$P timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -p no:cacheprovider > gpurun_out/r2_attn_poly$P.log 2>&1
  echo "poly=$P pytest rc=$?"; tail -1 gpurun_out/r2_attn_poly$P.log
done
for P in 0 1 2 4 0 1 2 4; do
  DWDP_ATTN_POLY=$P timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mla_attn \
    python scripts/attn_once.py 2>/dev/null | grep mla_attn | tail -1 | awk -F'","' -v p=$P '{print "poly=" p, $NF}'
done
