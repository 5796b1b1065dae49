#!/bin/bash
# Round measurement session on one B200 (run under gpurun): GPU tests, bench
# lines (C2 default, C5 on 1 GPU, C3a/C3b/C4, the two-kernel mode), the ncu
# launch list of the bench, full ncu captures of the dominant kernels, the
# S0-vs-min-PM BER sweep, the per-warp timeline and the e2e pipeline.
# Outputs go to gpurun_out/<tag>_*; copy the summaries into profiles/.
tag=${1:-r02}
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
o=gpurun_out/$tag
nvidia-smi > ${o}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rs > ${o}_gputest.txt 2>&1; tail -3 ${o}_gputest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > ${o}_bench_c2.json 2> ${o}_bench_c2.err; tail -c 400 ${o}_bench_c2.json
timeout 1200 python bench.py --workload C5 --steps 3 --warmup 3 > ${o}_bench_c5.json 2> ${o}_bench_c5.err; tail -c 300 ${o}_bench_c5.json
for w in C3a C3b C4; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > ${o}_bench_$w.json 2> ${o}_bench_$w.err; tail -c 200 ${o}_bench_$w.json; done
timeout 900 python bench.py --kernels two --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > ${o}_bench_c2_two.json 2> ${o}_bench_c2_two.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for c in C2 C4 C3a; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
      -o ${o}_fused_$c python tools/one_decode.py $c 2 0 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o ${o}_fused_c2_2p26 python tools/one_decode.py C2 2 0 1 67108864 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 1 -c 1 \
    -o ${o}_tb_c2 python tools/one_decode.py C2 2 0 0 > /dev/null 2>&1
timeout 1200 python tools/ber_sweep.py --code k7 --ebn0 3 --L 7 14 21 28 42 63 --bits 268435456 --start both \
    --json ${o}_ber_fig4.json > ${o}_ber_fig4.txt 2>&1
timeout 1200 python tools/ber_sweep.py --code k7 --ebn0 4 4.5 5 --L 42 --bits 1073741824 --start both \
    --json ${o}_ber_k7.json > ${o}_ber_k7.txt 2>&1
if [ -f paper_1608_00066_b200/build/variants/timing.so ]; then
  PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/timing.so timeout 300 python tools/exp_timing.py C2 > ${o}_timing_c2.txt 2>&1
fi
timeout 900 python tools/e2e_quick.py C2 C3a C4 > ${o}_e2e.txt 2>&1
ls -la gpurun_out | grep $tag
