#!/bin/bash
# build several A/B variants: tools/build_variants.sh "name:flags" "name:flags" ...
# (each into paper_1608_00066_b200/build/variants/<name>.so), then restore the
# default build (also when a variant fails to compile)
mkdir -p paper_1608_00066_b200/build/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  if PBVD_NVCC_EXTRA="$flags" python -m paper_1608_00066_b200.build --force > /tmp/bv_$name.log 2>&1; then
    cp paper_1608_00066_b200/libpbvd.so paper_1608_00066_b200/build/variants/$name.so
    echo "built $name ($flags)"
  else
    echo "FAILED $name ($flags): see /tmp/bv_$name.log"
  fi
done
python -m paper_1608_00066_b200.build --force > /dev/null
