python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
for v in timing timing_pf2 timing_pf6; do
  echo "=== $v"
  PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so python tools/exp_timing.py C2 2>&1 | head -12
done 2>&1 | tee gpurun_out/r2r_timing.txt
CASES="C2 C2:67108864" bash tools/ab.sh pf4 2>&1 | tee gpurun_out/r2r_ab.txt
