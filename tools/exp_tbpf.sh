#!/bin/bash
python -m paper_1608_00066_b200.build > /dev/null || exit 1
CONFIGS="C2" bash tools/exp_variants.sh "" "-DPBVD_TB_PREFETCH=1" "-DPBVD_TB_PREFETCH=1 -DPBVD_FUSED_TT=12" "-DPBVD_TB_PREFETCH=1 -DPBVD_IN_HINT=1"
for v in "" "-DPBVD_TB_PREFETCH=1"; do PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null; echo "== 2^26 $v"; python tools/quick_time.py C2 67108864 | grep lanes=2; done
python -m paper_1608_00066_b200.build --force > /dev/null
