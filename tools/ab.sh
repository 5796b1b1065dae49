#!/bin/bash
# A/B timing: the in-tree build vs build/variants/*.so (tools/build_variant.sh)
# usage: CASES="C2 C2:67108864 C4" bash tools/ab.sh [variant ...]
CASES=${CASES:-"C2 C2:67108864 C3a C4"}
for v in default "$@"; do
  if [ "$v" = default ]; then unset PBVD_LIB; else export PBVD_LIB=$PWD/paper_1608_00066_b200/build/variants/$v.so; fi
  for cs in $CASES; do
    c=${cs%%:*}; n=${cs#*:}; [ "$n" = "$cs" ] && n=""
    echo "[$v] $(timeout 300 python tools/quick_time.py $c $n 2>&1 | grep Gb/s | head -3 | tr '\n' ' ')"
  done
done
unset PBVD_LIB
