set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
