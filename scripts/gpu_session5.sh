set -x
mkdir -p gpurun_out
timeout 600 python scripts/tune.py --nt 100 --random-init --chunks 0,1,2,3,4,6,7,9,14 > gpurun_out/tune_c1_rand.log 2>&1; tail -3 gpurun_out/tune_c1_rand.log
CMD="python scripts/tune.py --nt 20 --random-init --by 16 --chunks 2"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 30 -c 1 -o gpurun_out/prof_fwd_rand $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
