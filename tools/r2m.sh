python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
CASES="C2 C2:67108864 C3a" bash tools/ab.sh skip nohint 2>&1 | tee gpurun_out/r2m_ab.txt
for v in default skip; do
  if [ $v = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fwd_kernel -s 1 -c 1 python tools/one_decode.py C2 2 0 1 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/$v /"
done | tee gpurun_out/r2m_dram.txt
