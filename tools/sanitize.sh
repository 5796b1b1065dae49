#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small decodes
python -m paper_1608_00066_b200.build > /dev/null || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  for args in "k7 3000 64 20 2" "k7 3000 64 20 4" "k9 2000 64 20 8" "k3 500 16 8 1" "k7 2000 96 30 2 3/4"; do
    out=$(timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/debug_case.py $args 2>&1)
    rc=$?
    echo "$tool [$args] rc=$rc $(echo "$out" | grep -E 'ERROR SUMMARY|bad bytes' | tr '\n' ' ')"
  done
done
# newer entry points (mirrored outputs, JIT codes, continuous stream, table depuncture, host pipeline)
for tool in memcheck racecheck synccheck initcheck; do
  out=$(timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/debug_new_paths.py 2>&1)
  rc=$?
  echo "$tool [new paths] rc=$rc $(echo "$out" | grep -E 'ERROR SUMMARY|total bad' | tr '\n' ' ')"
done
