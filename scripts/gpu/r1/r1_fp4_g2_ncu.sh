# ncu --set full of the NVFP4 GEMM2 (1-SM, TMA-store epilogue) with source, for the stall picture.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_kernel" --launch-skip 4 -c 1 -o gpurun_out/fp4_g2 -f python bench.py --dtype nvfp4 --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fp4_g2.log 2>&1; echo "ncu rc=$?"
