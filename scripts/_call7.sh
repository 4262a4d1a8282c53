mkdir -p gpurun_out/c7
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1; }
for rep in 1 2 3; do for c in 3 4 1; do for v in C T2 D3; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c7/ab_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(tail -1 gpurun_out/c7/ab_${v}_c${c}_$rep.log | summ)"
done; done; done
for c in 3 4 1; do for v in C T2 D3; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/c7/tune_${v}_c${c}.log 2>&1
echo "tune $v c$c $(grep -v BEST gpurun_out/c7/tune_${v}_c${c}.log | tail -1)"
done; done
