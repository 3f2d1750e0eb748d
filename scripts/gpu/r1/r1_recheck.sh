# Re-entry check of HEAD on a fresh box: GPU tests, smoke, N=1 bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/rc_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rc_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/rc_bench_n1.json 2> gpurun_out/rc_bench_n1.err; echo "bench rc=$?"; tail -c 600 gpurun_out/rc_bench_n1.json
