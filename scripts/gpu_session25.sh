set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for c in 1 3; do timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/tune_c$c.log 2>&1; grep -v BEST gpurun_out/tune_c$c.log | tail -2; done
timeout 300 python scripts/tune.py --config 2 --grad --nt 40 --vy 2 --ctas 0 > gpurun_out/tune_c2g.log 2>&1; grep -v BEST gpurun_out/tune_c2g.log | tail -1
