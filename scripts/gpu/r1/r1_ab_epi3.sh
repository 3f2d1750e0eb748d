# Same-box A/B of the plain-epilogue change (bf16 and fp8 GEMM2): previous vs new libdwdp.so, alternating.
mkdir -p gpurun_out
for v in prev new prev new; do
cp abtest/libdwdp_$v.so paper_2604_01621_b200/libdwdp.so
for dt in bf16 nvfp4; do
timeout 600 python bench.py --dtype $dt --no-cpu-baseline --no-e2e > gpurun_out/ab3.log 2>&1; grep metric gpurun_out/ab3.log > gpurun_out/ab3.json; python -c "import json; d=json.load(open('gpurun_out/ab3.json')); k=d['kernel_ms_per_layer']; print('$v $dt', round(d['value']), {x: round(k[x],2) for x in ('gemm1','gemm2','moe')}, d['clocks']['sm_mhz'])"
done; done
cp abtest/libdwdp_new.so paper_2604_01621_b200/libdwdp.so
