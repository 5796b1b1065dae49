python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
for a in "C2 3" "C2 2" "C3a 2" "C4 2"; do
PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/htrace.so timeout 300 python tools/e2e_trace.py $a 2>&1 | tail -20
done | tee gpurun_out/r2v_trace.txt
