python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so python tools/exp_timing.py C2 2>&1 | tee gpurun_out/r2i_timing.txt
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so python tools/exp_timing.py C2 67108864 2>&1 | tee -a gpurun_out/r2i_timing.txt
