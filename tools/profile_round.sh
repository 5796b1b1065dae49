#!/bin/bash
# bench + ncu launch list + full ncu captures (C2): the fused kernel (default)
# and, for comparison, the two kernels of the paper's structure; plus C5 on 1 GPU
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 900 python bench.py --kernels two --no-e2e --no-cpu-baseline > gpurun_out/bench_two.json 2> gpurun_out/bench_two.err; tail -c 600 gpurun_out/bench_two.json
timeout 1200 python bench.py --workload C5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 600 gpurun_out/bench_c5.json
for w in C3a C3b C4; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -c 300 gpurun_out/bench_$w.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/fused_full python tools/one_decode.py C2 2 0 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/fwd_full python tools/one_decode.py C2 2 0 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 1 -c 1 \
    -o gpurun_out/tb_full python tools/one_decode.py C2 2 0 0 > /dev/null 2>&1
ls -la gpurun_out | tail -10
