set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/tune.py --nt 100 --random-init --by 16 --chunks 0,7 > gpurun_out/tune_c1r.log 2>&1; cat gpurun_out/tune_c1r.log
CMD2="python scripts/tune.py --nt 12 --random-init --by 16 --chunks 0"
$CMD2 > gpurun_out/plain_tune.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 14 -c 1 -o gpurun_out/prof_stencil3 $CMD2 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
