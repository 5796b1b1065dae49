#!/bin/bash
# compare compile-time variants (timing only) at a given stream size:
#   N=67108864 bash tools/exp_variants_n.sh "" "-DFOO=1" ...
for v in "$@"; do
  PBVD_NVCC_EXTRA="$v" python -m paper_1608_00066_b200.build --force > /dev/null || exit 1
  echo "== $v"
  for c in ${CONFIGS:-C2}; do python tools/quick_time.py $c ${N:-} 2>&1 | grep Gb/s | grep "lanes=${LANES:-2}"; done
done
python -m paper_1608_00066_b200.build --force > /dev/null
