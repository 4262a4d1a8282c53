# ncu evidence (round 1, second pass): launch list of the bench command and full captures
# of the stencil kernel on configs[1] (so8) and configs[3] (so16), random-init wavefield.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --nt 40 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for c in 1 3; do
CMD2="python scripts/tune.py --config $c --nt 12 --random-init --by 16 --chunks 0"
$CMD2 > gpurun_out/plain_tune_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 8 -c 1 -o gpurun_out/prof_stencil_c$c $CMD2 > gpurun_out/ncu_full_c$c.log 2>&1
tail -3 gpurun_out/ncu_full_c$c.log
done
