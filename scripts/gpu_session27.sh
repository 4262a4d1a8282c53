set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
CFGS="1 2 4" bash scripts/ab_bench.sh
