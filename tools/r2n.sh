python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/bulk.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
CASES="C2 C2:67108864 C3a" bash tools/ab.sh bulk 2>&1 | tee gpurun_out/r2n_ab.txt
