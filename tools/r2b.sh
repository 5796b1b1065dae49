python -m paper_1608_00066_b200.build > /dev/null || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/r2b_nproc.txt; free -g >> gpurun_out/r2b_nproc.txt
timeout 1700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rs > gpurun_out/r2b_gputest.txt 2>&1; tail -15 gpurun_out/r2b_gputest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -c 3500 gpurun_out/r2b_bench.json
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/r2b_bench_c5.json 2> gpurun_out/r2b_bench_c5.err; tail -c 1500 gpurun_out/r2b_bench_c5.json; tail -5 gpurun_out/r2b_bench_c5.err
