python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
for c in C2 C4 C3a; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 1 -c 1 \
    -o gpurun_out/r2k_$c python tools/one_decode.py $c 2 0 1 > /dev/null 2>&1
done
ls gpurun_out | grep r2k
