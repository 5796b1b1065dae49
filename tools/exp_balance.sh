#!/bin/bash
python -m paper_1608_00066_b200.build > /dev/null || exit 1
for n in 16777216 18874368 19398656 20447232 33554432; do python tools/quick_time.py C2 $n 2>&1 | grep "lanes=2"; done
PBVD_NVCC_EXTRA="-DPBVD_EXP_NO_TB" python -m paper_1608_00066_b200.build --force > /dev/null
echo "== no TB walk (timing only)"
for n in 16777216 19398656; do python tools/quick_time.py C2 $n 2>&1 | grep "lanes=2"; done
python -m paper_1608_00066_b200.build --force > /dev/null
