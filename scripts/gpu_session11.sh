set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 600 python scripts/tune.py --config 3 --nt 30 --random-init --by 8,16 --chunks 0,1,2,3,4,6 > gpurun_out/tune_c3.log 2>&1; cat gpurun_out/tune_c3.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
