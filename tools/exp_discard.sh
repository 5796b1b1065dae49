#!/bin/bash
for v in "-DPBVD_SKIP_ROWS=1" "-DPBVD_SKIP_ROWS=1 -DPBVD_TB_DISCARD=1"; do
  PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
done
CONFIGS="C2" bash tools/exp_variants.sh "" "-DPBVD_SKIP_ROWS=1" "-DPBVD_TB_DISCARD=1" "-DPBVD_SKIP_ROWS=1 -DPBVD_TB_DISCARD=1"
for v in "" "-DPBVD_SKIP_ROWS=1 -DPBVD_TB_DISCARD=1"; do PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null; echo "== 2^26 C3a C4 $v"; python tools/quick_time.py C2 67108864 | grep lanes=2; python tools/quick_time.py C3a | grep lanes=2; python tools/quick_time.py C4 | grep lanes=4; done
python -m paper_1608_00066_b200.build --force > /dev/null
