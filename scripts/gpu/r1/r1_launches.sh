mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bl.log 2>&1; echo "bench rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"grouped_gemm_pair_kernel" --launch-skip 6 -c 2 -o gpurun_out/final_gemm -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fg.log 2>&1; echo "ncu gemm rc=$?"
