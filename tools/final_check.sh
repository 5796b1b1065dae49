#!/bin/bash
# Round-end check on one B200: the driver's steps (GPU tests, smoke, default
# bench) plus the C5 bench line; outputs gpurun_out/<tag>_*
tag=${1:-final}
python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out; o=gpurun_out/$tag
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rs > ${o}_gputest.txt 2>&1; tail -2 ${o}_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.txt 2>&1; tail -1 ${o}_smoke.txt
timeout 900 python bench.py > ${o}_bench_default.json 2> ${o}_bench_default.err; tail -c 200 ${o}_bench_default.json
timeout 1200 python bench.py --workload C5 --steps 3 --warmup 3 > ${o}_bench_c5.json 2> ${o}_bench_c5.err; tail -c 200 ${o}_bench_c5.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${o}_bench_reference.json 2> ${o}_bench_reference.err; tail -c 200 ${o}_bench_reference.json
