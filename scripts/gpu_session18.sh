set -x
mkdir -p gpurun_out
for c in 1 3; do timeout 300 python scripts/tune.py --config $c --nt 40 --vy 1,2 --ctas 0 > gpurun_out/tune_c$c.log 2>&1; tail -3 gpurun_out/tune_c$c.log; done
CMD2="python scripts/tune.py --config 1 --nt 12 --random-init --vy 2 --ctas 0"
$CMD2 > gpurun_out/plain_tune_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 8 -c 1 -o gpurun_out/prof_v3_c1 $CMD2 > gpurun_out/ncu_full_c1.log 2>&1
tail -2 gpurun_out/ncu_full_c1.log
