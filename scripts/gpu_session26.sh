set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 1200 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log; grep -i "error\|Traceback" gpurun_out/bench_c4.log | head
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --split > gpurun_out/bench_c1_split.log 2>&1; tail -1 gpurun_out/bench_c1_split.log
