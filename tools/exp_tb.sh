#!/bin/bash
# traceback experiments: parity + timing for fused ring sizes
python -m paper_1608_00066_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -3
for c in C2 C3a C4; do QT_FUSED="1 0" timeout 300 python tools/quick_time.py $c 2>&1 | grep Gb/s; done
QT_FUSED="1 0" python tools/quick_time.py C2 67108864 | grep Gb/s
for tt in 12 18; do
  PBVD_NVCC_EXTRA="-DPBVD_FUSED_TT=$tt" python -m paper_1608_00066_b200.build --force > /dev/null || exit 1
  echo "== FUSED_TT=$tt"
  for c in C2 C4; do QT_FUSED="1" timeout 300 python tools/quick_time.py $c 2>&1 | grep Gb/s; done
  QT_FUSED="1" python tools/quick_time.py C2 67108864 | grep Gb/s
done
python -m paper_1608_00066_b200.build --force > /dev/null
