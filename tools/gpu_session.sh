python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
for v in t_np t_p t_p2x30; do
  echo "=== $v"
  PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so python tools/exp_timing.py C2 2>&1 | head -7
done 2>&1 | tee gpurun_out/r2t_timing.txt
CASES="C2 C2:67108864" bash tools/ab.sh np p2x30 2>&1 | tee gpurun_out/r2t_ab.txt
