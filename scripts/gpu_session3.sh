set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 600 python scripts/tune.py --nt 60 --chunks 0,2,4,5,6,7,8,9,10,14 > gpurun_out/tune_c1.log 2>&1; tail -4 gpurun_out/tune_c1.log
CMD="python bench.py --steps 1 --warmup 3 --nt 30 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 100 -c 1 -o gpurun_out/prof_fwd2 $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
