python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
CASES="C2 C2:67108864 C3a C4 C1" bash tools/ab.sh nodec1 2>&1 | tee gpurun_out/r2e_ab.txt
