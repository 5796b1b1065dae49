python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 600 python tools/quick_time.py C4 2>&1 | grep Gb/s | tee gpurun_out/r2l.txt
timeout 600 python tools/quick_time.py C4 67108864 2>&1 | grep Gb/s | tee -a gpurun_out/r2l.txt
