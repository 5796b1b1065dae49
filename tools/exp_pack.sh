#!/bin/bash
python -m paper_1608_00066_b200.build > /dev/null || exit 1
CONFIGS="C2" bash tools/exp_variants.sh "" "-DPBVD_PACK_TREE=1" "-DPBVD_FMA_SPLIT=2" "-DPBVD_PACK_TREE=1 -DPBVD_FMA_SPLIT=2" "-DPBVD_FMA_SPLIT=0"
