# NVFP4 at N=2: multi-GPU parity (DWDP + DEP vs all-local, bitwise), then DWDP vs DEP benches.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/fp4_mg.log 2>&1; echo "mg rc=$?"; tail -3 gpurun_out/fp4_mg.log
for mnt in 32768 65536; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29571 bench.py --gpus 2 --dtype nvfp4 --tokens $mnt --cv 0.2 > gpurun_out/fp4_n2_$mnt.log 2>&1; echo "n2 $mnt rc=$?"
grep '"metric"' gpurun_out/fp4_n2_$mnt.log > gpurun_out/fp4_n2_$mnt.json
python -c "import json; d=json.load(open('gpurun_out/fp4_n2_$mnt.json')); print(round(d['tokens_per_s_per_gpu']), d['dep_baseline'] and round(d['dep_baseline']['dwdp_over_dep'],3), round(d['exposed_prefetch_ms_per_layer'],3), d['prefetch'], d['config']['prefetch_engine'], d['clocks']['sm_mhz'])"
done
