set -x
mkdir -p gpurun_out
timeout 300 python scripts/e2e_probe.py 1 > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
