# ncu --set full of the bf16 GEMMs (1-SM default) with source, for the GEMM2 stall picture.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_kernel" --launch-skip 3 -c 1 -o gpurun_out/bf16_gemm2 -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bf16_ncu.log 2>&1; echo "ncu rc=$?"
