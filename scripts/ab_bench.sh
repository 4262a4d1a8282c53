# A/B of two libsf builds on whole bench steps (bench.py, device time per step), A B A B
set -x
mkdir -p gpurun_out
CFGS=${CFGS:-"1 2"}
for rep in 1 2; do for v in A B; do for c in $CFGS; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abb_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(tail -1 gpurun_out/abb_${v}_c${c}_$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"], d["gpu_launches"])')"
done; done; done
