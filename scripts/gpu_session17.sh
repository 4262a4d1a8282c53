set -x
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
for c in 1 3; do timeout 300 python scripts/tune.py --config $c --nt 40 --vy 1,2 --ctas 0,148,296 > gpurun_out/tune_c$c.log 2>&1; tail -7 gpurun_out/tune_c$c.log; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
