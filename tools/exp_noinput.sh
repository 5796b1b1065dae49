#!/bin/bash
# experiment: forward kernel without the soft-input path (timing only; wrong output)
PBVD_NVCC_EXTRA="-DPBVD_EXP_NO_INPUT" python -m paper_1608_00066_b200.build --force > /dev/null
CONFIGS="C2 C4" ; for c in $CONFIGS; do python tools/quick_time.py $c 2>&1 | grep Gb/s; done
python -m paper_1608_00066_b200.build --force > /dev/null
