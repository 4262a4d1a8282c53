mkdir -p gpurun_out/c3
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c3/gpu_tests.log 2>&1; tail -3 gpurun_out/c3/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c3/smoke.log 2>&1; tail -1 gpurun_out/c3/smoke.log
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["per_update_us"], d["clocks"]["sm_mhz"], d["gpu_launches"])'; }
for rep in 1 2; do for c in 1 2 4; do for v in A B1 B; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3/ab_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(tail -1 gpurun_out/c3/ab_${v}_c${c}_$rep.log | summ)"
done; done
for c in 2 4; do
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-plane > gpurun_out/c3/noplane_c${c}_$rep.log 2>&1
echo "noplane c$c rep$rep $(tail -1 gpurun_out/c3/noplane_c${c}_$rep.log | summ)"
done; done
for c in 1; do for v in A B; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/c3/tune_${v}_c${c}.log 2>&1
echo "tune $v c$c $(grep -v BEST gpurun_out/c3/tune_${v}_c${c}.log | tail -1)"
done; done
