python -m paper_1608_00066_b200.build > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x --timeout 1200 -p no:cacheprovider -k "C3 or punct or config or small or golden" 2>&1 | tail -2
for r in 1 2 3; do
for v in default base; do
  if [ "$v" = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  for c in C2 "C2 67108864" C3a C3b; do QT_LANES=2 timeout 300 python tools/quick_time.py $c 2>&1 | grep Gb/s | sed "s/^/[$v] /"; done
done; unset PBVD_LIB; done
