# evidence refresh (run under gpurun): GPU tests, smoke, bench lines configs[1..4] + reference
# arm + the 1-GPU split schedules, ncu launch list of the default bench command, full
# captures of the stencil on configs[1]/[3]/[4].  Outputs under gpurun_out/ev/.
set -x
R=${ROUND:-r02}
mkdir -p gpurun_out/ev
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev/gpu_tests.log 2>&1; tail -2 gpurun_out/ev/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; tail -1 gpurun_out/ev/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 15 > gpurun_out/ev/bench_c1.log 2>&1; tail -1 gpurun_out/ev/bench_c1.log | cut -c1-300
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/bench_c2.log 2>&1; tail -1 gpurun_out/ev/bench_c2.log | cut -c1-200
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/bench_c3.log 2>&1; tail -1 gpurun_out/ev/bench_c3.log | cut -c1-200
timeout 1200 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev/bench_c4.log 2>&1; tail -1 gpurun_out/ev/bench_c4.log | cut -c1-200
timeout 600 python bench.py --config 0 --steps 5 --warmup 3 --no-cpu-baseline --graph > gpurun_out/ev/bench_c0_graph.log 2>&1; tail -1 gpurun_out/ev/bench_c0_graph.log | cut -c1-200
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --split > gpurun_out/ev/bench_c1_split2.log 2>&1; tail -1 gpurun_out/ev/bench_c1_split2.log | cut -c1-200
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --split --one-launch > gpurun_out/ev/bench_c1_split1.log 2>&1; tail -1 gpurun_out/ev/bench_c1_split1.log | cut -c1-200
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_ref.log 2>&1; tail -1 gpurun_out/ev/bench_ref.log | cut -c1-200
CMD="python bench.py --steps 1 --warmup 3 --nt 40 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ev/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 150 --csv --log-file gpurun_out/ev/launches.csv $CMD > gpurun_out/ev/ncu_launch.log 2>&1
# the layout / work split sf_autotune picks in bench.py for each config (the "kernel_tuning" of
# its bench line): configs[1] 7-warp chunked, [3] 8-warp chunked, [4] 8-warp balanced
declare -A TUNE=([1]="--vy 2 --balance 0" [3]="--vy 4 --balance 0" [4]="--vy 4 --balance 1")
# points x algorithmic bytes per point of the captured launch (configs[4]: its 128-column launch)
declare -A PTS=([1]="37933056 20" [3]="268435456 16" [4]="61440000 16")
mkdir -p /tmp/ev
for c in 1 3 4; do
CMD2="python scripts/tune.py --config $c --nt 8 --random-init ${TUNE[$c]} --ctas 0"
$CMD2 > gpurun_out/ev/plain_tune_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tma3d -s 4 -c 1 -o /tmp/ev/prof_${R}_c$c $CMD2 > gpurun_out/ev/ncu_full_c$c.log 2>&1
tail -1 gpurun_out/ev/ncu_full_c$c.log
# summaries on the box (the reports themselves exceed the 64 MiB merge-back)
set -- ${PTS[$c]}
python scripts/ncu_summary.py full /tmp/ev/prof_${R}_c$c.ncu-rep gpurun_out/ev/${R}_stencil_ncu_c$c.json --points $1 --bytes-per-point $2
python scripts/ncu_quick.py /tmp/ev/prof_${R}_c$c.ncu-rep > gpurun_out/ev/${R}_stencil_ncu_c${c}_quick.txt 2>&1
done
python scripts/ncu_summary.py launches gpurun_out/ev/launches.csv gpurun_out/ev/${R}_bench_launches.json
# gradient configs: DRAM traffic of every stencil launch of one timed step (NVTX range sf_timed:
# the setup-time tuning runs unprofiled), weighted per mode to the full config's average update
for c in 2 4; do
CMD3="python bench.py --config $c --nt 41 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD3 > gpurun_out/ev/plain_step_c$c.log 2>&1 && \
ncu --nvtx --nvtx-include "sf_timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:k_tma3d --csv --log-file gpurun_out/ev/${R}_step_traffic_c$c.csv $CMD3 > gpurun_out/ev/ncu_step_c$c.log 2>&1
L=1; [ $c = 4 ] && L=2
python scripts/ncu_step_traffic.py gpurun_out/ev/${R}_step_traffic_c$c.csv gpurun_out/ev/${R}_step_traffic_c$c.json --config $c --nt-run 41 --launches-per-update $L
done
