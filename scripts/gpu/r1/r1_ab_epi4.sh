# SwiGLU epilogue: overlapped chunks read and released first (test on new .so), then same-box A/B prev vs new.
mkdir -p gpurun_out
cp abtest/libdwdp_new.so paper_2604_01621_b200/libdwdp.so
timeout 1200 python -m pytest tests/test_gpu.py tests/test_gpu_nvfp4.py -q -x > gpurun_out/e4_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e4_t.log
bash scripts/gpu/r1_ab_epi3.sh
