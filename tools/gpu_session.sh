python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
CASES="C4 C4:67108864 C2" bash tools/ab.sh old 2>&1 | tee gpurun_out/r2u_ab.txt
for v in default old; do
  if [ $v = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  QT_FUSED=0 timeout 300 python tools/quick_time.py C4 2>&1 | grep Gb/s | sed "s/^/[$v two] /"
done 2>&1 | tee -a gpurun_out/r2u_ab.txt
