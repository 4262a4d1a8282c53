set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
