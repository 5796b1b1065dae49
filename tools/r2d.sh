python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
for v in default nodec0; do
  if [ $v = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/r2d_$v python tools/one_decode.py C2 2 0 1 67108864 > /dev/null 2>&1
done
unset PBVD_LIB
ls -la gpurun_out
