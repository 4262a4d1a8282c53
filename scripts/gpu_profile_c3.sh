set -x
mkdir -p gpurun_out
CMD="python scripts/tune.py --config 3 --nt 6 --random-init --by 8 --chunks 0"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 6 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
