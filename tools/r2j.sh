python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
CASES="C2 C2:67108864" bash tools/ab.sh pf r5x12 r5x12pf 2>&1 | tee gpurun_out/r2j_ab.txt
