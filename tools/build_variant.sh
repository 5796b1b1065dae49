#!/bin/bash
# build an A/B variant of libpbvd.so with extra nvcc flags into build/variants/<name>.so
# (loaded with PBVD_LIB=...), then restore the default in-tree build
name=$1; shift
mkdir -p paper_1608_00066_b200/build/variants
cp paper_1608_00066_b200/libpbvd.so /tmp/libpbvd_default.so
PBVD_NVCC_EXTRA="$*" python -m paper_1608_00066_b200.build --force > /dev/null || exit 1
cp paper_1608_00066_b200/libpbvd.so paper_1608_00066_b200/build/variants/$name.so
python -m paper_1608_00066_b200.build --force > /dev/null
