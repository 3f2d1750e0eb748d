# HBM bytes per launch of the default bf16 GEMM1 (1-SM grouped_gemm_kernel<0>) for bench.py's roofline.traffic.
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --kernel-name regex:"grouped_gemm_kernel" -c 6 --csv --log-file gpurun_out/g1dram.csv python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g1dram.log 2>&1; echo "ncu rc=$?"; grep -c grouped gpurun_out/g1dram.csv
