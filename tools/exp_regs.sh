#!/bin/bash
for v in "-DPBVD_MAXREG=128" "-DPBVD_MAXREG=200" "-DPBVD_MAXREG=104"; do
  PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null || exit 1
  echo "== $v"
  for c in C2 C3a; do python tools/quick_time.py $c 2>&1 | grep "lanes=2"; done
  python tools/quick_time.py C2 67108864 | grep "lanes=2"
  python tools/quick_time.py C4 | grep "lanes=4"
done
python -m paper_1608_00066_b200.build --force > /dev/null
