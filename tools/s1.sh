python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
o=gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > ${o}_smi.txt 2>&1
timeout 600 python tools/quick_time.py C2 > ${o}_qt.txt 2>&1
timeout 300 python tools/quick_time.py C2 67108864 >> ${o}_qt.txt 2>&1
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so timeout 300 python tools/exp_timing.py C2 > ${o}_timing_c2.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > ${o}_bench_c2.json 2> ${o}_bench_c2.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rs > ${o}_gputest.txt 2>&1; tail -3 ${o}_gputest.txt
cat ${o}_qt.txt
