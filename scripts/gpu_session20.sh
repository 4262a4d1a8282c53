set -x
mkdir -p gpurun_out
for vy in 1 2; do
CMD2="python scripts/tune.py --config 3 --nt 6 --random-init --vy $vy --ctas 0"
$CMD2 > gpurun_out/plain_tune_c3_vy$vy.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 3 -c 1 -o gpurun_out/prof_v3_c3_vy$vy $CMD2 > gpurun_out/ncu_full_c3_vy$vy.log 2>&1
tail -1 gpurun_out/ncu_full_c3_vy$vy.log
done
