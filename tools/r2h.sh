python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py tests/test_gpu_jit.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
CASES="C2 C2:67108864 C3a C4" bash tools/ab.sh old 2>&1 | tee gpurun_out/r2h_ab.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2h_bench.json 2>&1
