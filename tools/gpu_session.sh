python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_jit.py -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -3
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so python tools/exp_timing.py C2 2>&1 | head -8
for r in 1 2; do CASES="C2 C2:67108864 C3a" bash tools/ab.sh nosplit; done 2>&1 | tee gpurun_out/r2ac_ab.txt
