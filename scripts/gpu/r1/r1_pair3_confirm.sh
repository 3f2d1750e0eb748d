# A/B of GEMM2 on CTA pairs as the bf16 default (then built in; now opt-in, DWDP_GEMM_PAIR=3): GPU suite incl. multi-GPU parity on 2 GPUs,
# same-box N=1 A/B vs DWDP_GEMM_PAIR=0, and an N=2 bench (DWDP vs DEP, both with the default).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pc_tests.log
for rep in 1 2; do
  for v in def 0; do
    if [ $v = def ]; then E=""; else E="DWDP_GEMM_PAIR=0"; fi
    env $E timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | grep metric > gpurun_out/pc_${v}_$rep.json
    python -c "import json; d=json.load(open('gpurun_out/pc_${v}_$rep.json')); k=d['kernel_ms_per_layer']; print('$v rep $rep', round(d['value']), {x: round(k[x],3) for x in ('router','permute','gemm1','gemm2','combine','moe')}, round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
timeout 450 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29558 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/pc_n2.log 2>&1; echo "n2 rc=$?"; grep metric gpurun_out/pc_n2.log > gpurun_out/pc_n2.json
python -c "import json; d=json.load(open('gpurun_out/pc_n2.json')); print('n2', round(d['value']), round(d['tokens_per_s_per_gpu']), d['dep_baseline']['dwdp_over_dep'] if d.get('dep_baseline') else None, d['exposed_prefetch_ms_per_layer'], d['clocks']['sm_mhz'])"
