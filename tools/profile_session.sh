#!/bin/bash
# Measurement session on one B200 (run under gpurun): GPU tests, bench lines
# (C2 default, C5 on 1 GPU, C3a/C3b/C4, the two-kernel mode), the ncu launch
# list of the bench, ncu full captures of the fused kernel (C2, C2 at 2^26
# bits, C4) and the per-chunk timeline.  Outputs: gpurun_out/<tag>_*.
tag=${1:-r02c}
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
o=gpurun_out/$tag
nvidia-smi > ${o}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rs > ${o}_gputest.txt 2>&1; tail -3 ${o}_gputest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > ${o}_bench_c2.json 2> ${o}_bench_c2.err; tail -c 300 ${o}_bench_c2.json
timeout 1200 python bench.py --workload C5 --steps 3 --warmup 3 > ${o}_bench_c5.json 2> ${o}_bench_c5.err; tail -c 200 ${o}_bench_c5.json
for w in C3a C3b C4; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > ${o}_bench_$w.json 2> ${o}_bench_$w.err; tail -c 200 ${o}_bench_$w.json; done
timeout 900 python bench.py --kernels two --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > ${o}_bench_c2_two.json 2> ${o}_bench_c2_two.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o ${o}_fused_C2 python tools/one_decode.py C2 2 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o ${o}_fused_C4 python tools/one_decode.py C4 2 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o ${o}_fused_c2_2p26 python tools/one_decode.py C2 2 0 1 67108864 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o ${o}_fused_C3a python tools/one_decode.py C3a 2 0 1 > /dev/null 2>&1
if [ -f paper_1608_00066_b200/build/variants/timing.so ]; then
  PBVD_TIMING_SAVE=${o}_timing_c2.npy PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so timeout 300 python tools/exp_timing.py C2 > ${o}_timing_c2.txt 2>&1
fi
timeout 900 python tools/e2e_quick.py C2 C3a C4 > ${o}_e2e.txt 2>&1
ls -la gpurun_out | grep $tag
