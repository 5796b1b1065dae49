python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
bash tools/ab.sh nodec0 2>&1 | tee gpurun_out/r2c_ab.txt
