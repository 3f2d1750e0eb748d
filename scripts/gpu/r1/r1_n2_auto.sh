# N=2: the step-timed auto engine choice (nvfp4 and bf16, MNT 32K, CV 0.2).
mkdir -p gpurun_out
for dt in nvfp4 bf16; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29591 bench.py --gpus 2 --dtype $dt --tokens 32768 --cv 0.2 --no-e2e > gpurun_out/n2a_$dt.log 2>&1; echo "$dt rc=$?"
grep '"metric"' gpurun_out/n2a_$dt.log > gpurun_out/n2a_$dt.json
python -c "import json; d=json.load(open('gpurun_out/n2a_$dt.json')); print(round(d['tokens_per_s_per_gpu']), d['dep_baseline'] and round(d['dep_baseline']['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), round(d['kernel_ms_per_layer']['moe'],2), d['prefetch'], d['config']['prefetch_engine'], d['clocks']['sm_mhz'])"
done
