# ncu --set full of the NVFP4 GEMMs (after issuer / epilogue changes), source-level.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_kernel" --launch-skip 10 -c 3 -o gpurun_out/fp4_gemm3 -f python bench.py --dtype nvfp4 --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fp4_ncu3.log 2>&1; echo "ncu rc=$?"
