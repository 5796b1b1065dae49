python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jit.py -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -1
for r in 1 2; do CASES="C2 C2:67108864 C3a C4" bash tools/ab.sh head; done 2>&1 | tee gpurun_out/r2af_ab.txt
