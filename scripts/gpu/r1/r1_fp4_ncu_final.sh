# ncu of one NVFP4 layer with the final build: every kernel's time, HBM bytes, tensor-pipe and L2->SM traffic.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg.per_second --clock-control none --launch-skip 40 -c 16 --csv --log-file gpurun_out/fp4_layer.csv python bench.py --dtype nvfp4 --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fp4_layer.log 2>&1; echo "ncu rc=$?"
