#!/bin/bash
# Round 2: QK^T accumulated in f16 (DWDP_ATTN_SF16=1) vs fp32 -- accuracy
# against the fp32 restatement, kernel time (same box).
mkdir -p gpurun_out
python scripts/attn_acc.py
DWDP_ATTN_SF16=1 python scripts/attn_acc.py
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export DWDP_ATTN_SF16=1; else unset DWDP_ATTN_SF16; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mla_attn \
    python scripts/attn_once.py 2>/dev/null | grep mla_attn | tail -1 | awk -F'","' -v p=$v '{print "sf16=" p, $NF}'
done
