# Session-end evidence for the batched-load combine: N=1 bf16 and NVFP4 bench
# lines, then one ncu --set full capture of the combine and permute copy kernels.
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/end_b1.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/end_b1.log > gpurun_out/end_b1.json
timeout 400 python bench.py --dtype nvfp4 --no-cpu-baseline > gpurun_out/end_b4.log 2>&1; echo "nvfp4 rc=$?"; grep metric gpurun_out/end_b4.log > gpurun_out/end_b4.json
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"combine_kernel|permute_copy_bulk_kernel" -c 2 -o gpurun_out/end_ng -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dep > gpurun_out/end_ncu.log 2>&1; echo "ncu rc=$?"
