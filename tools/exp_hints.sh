#!/bin/bash
python -m paper_1608_00066_b200.build > /dev/null || exit 1
CONFIGS="C2" bash tools/exp_variants.sh "" "-DPBVD_DEC_HINT=1" "-DPBVD_DEC_HINT=2" "-DPBVD_IN_HINT=1" "-DPBVD_DEC_HINT=1 -DPBVD_IN_HINT=1"
