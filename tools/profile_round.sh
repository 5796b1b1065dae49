#!/bin/bash
# bench + ncu launch list + full ncu captures of the two kernels (C2)
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/fwd_full python tools/one_decode.py C2 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb_kernel -s 1 -c 1 \
    -o gpurun_out/tb_full python tools/one_decode.py C2 2 > /dev/null 2>&1
ls -la gpurun_out | tail -6
