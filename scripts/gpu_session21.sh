set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 300 -k "forward_3d or gradient_parity_tma or split or config3" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for pd in 4 8; do for c in 3 1; do SF_L2_PREFETCH=$pd timeout 300 python scripts/tune.py --config $c --nt 40 --vy 1,2 --ctas 0 > gpurun_out/tune_c${c}_pd$pd.log 2>&1; echo pd $pd; grep -v BEST gpurun_out/tune_c${c}_pd$pd.log | tail -2; done; done
CMD2="python scripts/tune.py --config 3 --nt 6 --random-init --vy 2 --ctas 0"
$CMD2 > gpurun_out/plain_tune_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 3 -c 1 -o gpurun_out/prof_v3d_c3 $CMD2 > gpurun_out/ncu_full_c3.log 2>&1
tail -1 gpurun_out/ncu_full_c3.log
