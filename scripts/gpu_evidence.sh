# evidence refresh (run under gpurun): GPU tests, smoke, bench lines configs[1..4] +
# reference arm, ncu launch list of the default bench command, full captures on configs[1]/[3]
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | cut -c1-300
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-200
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log | cut -c1-200
timeout 1200 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-200
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
CMD="python bench.py --steps 1 --warmup 3 --nt 40 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for c in 1 3; do
CMD2="python scripts/tune.py --config $c --nt 8 --random-init --vy 2 --ctas 0"
$CMD2 > gpurun_out/plain_tune_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 4 -c 1 -o gpurun_out/prof_r01f_c$c $CMD2 > gpurun_out/ncu_full_c$c.log 2>&1
tail -1 gpurun_out/ncu_full_c$c.log
done
