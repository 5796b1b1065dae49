#!/bin/bash
# build several A/B variants: tools/build_variants.sh "name:flags" "name:flags" ...
# (each into paper_1608_00066_b200/build/variants/<name>.so), then restore the default build
mkdir -p paper_1608_00066_b200/build/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  PBVD_NVCC_EXTRA="$flags" python -m paper_1608_00066_b200.build --force > /dev/null || exit 1
  cp paper_1608_00066_b200/libpbvd.so paper_1608_00066_b200/build/variants/$name.so
  echo "built $name ($flags)"
done
python -m paper_1608_00066_b200.build --force > /dev/null
