python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do CASES="C2 C2:67108864" bash tools/ab.sh storeall; done 2>&1 | tee gpurun_out/r2x_ab.txt
for v in default storeall; do
  if [ $v = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:fwd_kernel -s 1 -c 1 python tools/one_decode.py C2 2 0 1 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/$v /"
done | tee gpurun_out/r2x_dram.txt
