# one full ncu capture of every kernel of the last (timed) layer of bench --profile (N=1)
mkdir -p gpurun_out
timeout 300 python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof1b.log 2>&1; echo "prof1 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
  --kernel-name regex:"grouped_gemm|topk|router_quant|permute|combine" --launch-skip 34 -c 9 \
  -o gpurun_out/layer_full -f python bench.py --profile --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_layer.log 2>&1; echo "ncu layer rc=$?"
timeout 2400 python scripts/sweep_decode.py --gpus 2 --batch 64,256,1024,4096 --zipf 0,0.8,1.2 --fetch split --steps 3 --warmup 3 --out gpurun_out/sweep_decode_n2.jsonl > gpurun_out/sweep_decode_n2.log 2>&1; echo "sweep split rc=$?"
timeout 1200 python scripts/sweep_decode.py --gpus 2 --batch 64,256,1024,4096 --zipf 0.8 --fetch merged --steps 3 --warmup 3 --out gpurun_out/sweep_decode_n2.jsonl >> gpurun_out/sweep_decode_n2.log 2>&1; echo "sweep merged rc=$?"
