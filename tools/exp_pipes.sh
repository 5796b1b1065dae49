#!/bin/bash
# pipe split experiments: FMA_SPLIT variants (timing) + ncu pipe counters of the C2 forward kernel
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 600 ncu --clock-control none -k regex:fwd_kernel -s 1 -c 1 --metrics \
sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__inst_executed_pipe_fp16.sum,sm__inst_executed_pipe_uniform.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
  python tools/one_decode.py C2 2 2>&1 | grep -E "sm__|smsp__|gpu__" 
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/fwd_r2 python tools/one_decode.py C2 2 > /dev/null 2>&1
CONFIGS="C2" bash tools/exp_variants.sh "-DPBVD_FMA_SPLIT=0" "-DPBVD_FMA_SPLIT=1" "-DPBVD_FMA_SPLIT=2"
