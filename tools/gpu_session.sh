python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -p no:cacheprovider -k host 2>&1 | tail -2
for r in 1 2; do
timeout 900 python tools/e2e_sweep.py C2 4,0 0 2>&1
timeout 900 python tools/e2e_sweep.py C2 0 -1 2>&1
done | tee gpurun_out/r2z_e2e.txt
for c in C3a C4; do timeout 900 python tools/e2e_sweep.py $c 0,4 -1,0 2>&1; done | tee -a gpurun_out/r2z_e2e.txt
