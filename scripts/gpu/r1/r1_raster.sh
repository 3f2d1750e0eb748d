mkdir -p gpurun_out
for R in auto m n; do
DWDP_RASTER=$R timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/rast_$R.log 2>&1; echo "raster $R rc=$?"; grep metric gpurun_out/rast_$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_layer']; print(round(d['value']), {x: round(k[x],2) for x in ('router','permute','gemm1','gemm2','combine','moe')}, d['clocks']['sm_mhz'])"
DWDP_RASTER=$R timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none --kernel-name regex:"grouped_gemm_pair" --launch-skip 6 -c 2 --csv python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | cut -d, -f5,15- | cut -c1-200
done
