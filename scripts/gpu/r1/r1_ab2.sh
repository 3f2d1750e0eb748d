mkdir -p gpurun_out
bash scripts/gpu/r1_ab_pair.sh
timeout 900 python -m pytest tests -q -m gpu -x -k "not multigpu" > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
