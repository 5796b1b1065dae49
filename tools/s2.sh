python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
o=gpurun_out/s2
for n in 16777216 67108864; do
PBVD_TIMING_SAVE=${o}_timing_$n.npy PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so timeout 300 python tools/exp_timing.py C2 $n > ${o}_timing_$n.txt 2>&1
done
