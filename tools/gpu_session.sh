python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/nw4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/nw4 parity: /"
CASES="C4 C2 C2:67108864 C3a C4:67108864" bash tools/ab.sh nw4 nw4ns 2>&1 | tee gpurun_out/r2ab_ab.txt
