python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 600 -p no:cacheprovider -k "not c5" 2>&1 | tail -3
PBVD_FWD_WARPS_PER_SM=12 CASES="C2 C2:67108864 C3a C4" bash tools/ab.sh nodec1 2>&1 | tee gpurun_out/r2g_ab.txt
for n in 16777216 67108864; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/r2g_c2_$n python tools/one_decode.py C2 2 0 1 $n > /dev/null 2>&1
done
ls gpurun_out
