#!/bin/bash
# Round 2 ncu evidence (1 GPU; each command first runs clean without ncu):
#  - launch list of the default N=1 bench (2 timed steps), kernel shares
#  - --set full of GEMM1 / GEMM2 / router / permute / combine of one R1 layer (bench --profile)
#  - --set full of the MLA attention kernel and its projections (scripts/attn_once.py)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-check"
$B > gpurun_out/r2_plain.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_n1.csv $B > /dev/null 2>&1
echo "launches rc=$?"
P="python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-check"
$P > gpurun_out/r2_plain2.log 2>&1 && \
  timeout 1500 $NCU --set full --clock-control none --import-source on \
    -k regex:"grouped_gemm_kernel|router_gemm_kernel|router_quant|topk_contig|permute_copy_bulk|combine_kernel" \
    -s 30 -c 7 -o gpurun_out/r2_ncu_layer $P > gpurun_out/r2_ncu_layer.log 2>&1
echo "layer rc=$?"
python scripts/attn_once.py > gpurun_out/r2_plain3.log 2>&1 && \
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"mla_attn_kernel|grouped_gemm_kernel" \
    -s 6 -c 6 -o gpurun_out/r2_ncu_mla python scripts/attn_once.py > gpurun_out/r2_ncu_mla.log 2>&1
echo "mla rc=$?"
