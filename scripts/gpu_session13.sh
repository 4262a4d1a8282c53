set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for i in 1 2; do timeout 300 python scripts/tune.py --nt 100 --random-init --by 16,8 --chunks 0 > gpurun_out/tune_c1r.log 2>&1; cat gpurun_out/tune_c1r.log; done
timeout 300 python scripts/tune.py --config 3 --nt 30 --random-init --by 16,8 --chunks 0 > gpurun_out/tune_c3.log 2>&1; cat gpurun_out/tune_c3.log
