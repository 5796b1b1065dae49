python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
for w in 0 8 12 16; do
  echo "== warps/SM cap $w"
  PBVD_FWD_WARPS_PER_SM=$w CASES="C2 C2:67108864 C3a" bash tools/ab.sh old 2>&1
done 2>&1 | tee gpurun_out/r2f_occ.txt
