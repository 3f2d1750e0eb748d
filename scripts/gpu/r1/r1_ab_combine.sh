# Same-box A/B of a non-GEMM kernel change (new) vs the previous build (base):
# GPU suite on the new build, then alternating bf16 and NVFP4 N=1 bench runs.
mkdir -p gpurun_out
D=paper_2604_01621_b200
cp $D/libdwdp_new.so.bin $D/libdwdp.so
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/abc_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/abc_tests.log
for rep in 1 2; do
  for v in new base; do
    cp $D/libdwdp_$v.so.bin $D/libdwdp.so
    for dt in ${DTYPES:-bf16 nvfp4}; do
      timeout 400 python bench.py --dtype $dt --no-cpu-baseline --no-e2e 2>/dev/null | grep metric > gpurun_out/abc_${v}_${dt}_$rep.json
      python -c "import json,sys; d=json.load(open('gpurun_out/abc_${v}_${dt}_$rep.json')); k=d['kernel_ms_per_layer']; print('$v $dt $rep', round(d['value']), {x: round(k[x],3) for x in ('permute','combine','gemm2','moe')}, d['clocks']['sm_mhz'])"
    done
  done
done
cp $D/libdwdp_new.so.bin $D/libdwdp.so
