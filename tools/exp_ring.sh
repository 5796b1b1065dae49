#!/bin/bash
CONFIGS="C2" bash tools/exp_variants.sh "" "-DPBVD_FUSED_NBUF=4" "-DPBVD_FUSED_NBUF=6 -DPBVD_FUSED_TT=12" "-DPBVD_FUSED_NBUF=8 -DPBVD_FUSED_TT=12" "-DPBVD_FUSED_NBUF=5 -DPBVD_FUSED_TT=18"
for v in "" "-DPBVD_FUSED_NBUF=6 -DPBVD_FUSED_TT=12"; do PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null; echo "== 2^26 / C4 $v"; python tools/quick_time.py C2 67108864 | grep lanes=2; python tools/quick_time.py C4 | grep lanes=4; done
python -m paper_1608_00066_b200.build --force > /dev/null
