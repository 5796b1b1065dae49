#!/bin/bash
# quick GPU iteration: build, parity tests, timings
python -m paper_1608_00066_b200.build || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -4
for c in ${CONFIGS:-C2 C4 C3b C1}; do timeout 300 python tools/quick_time.py $c 2>&1 | grep Gb/s; done
