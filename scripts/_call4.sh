mkdir -p gpurun_out/c4
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c4/gpu_tests.log 2>&1; tail -3 gpurun_out/c4/gpu_tests.log; grep FAILED gpurun_out/c4/gpu_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c4/smoke.log 2>&1; tail -1 gpurun_out/c4/smoke.log
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["per_update_us"], d["clocks"]["sm_mhz"], d["gpu_launches"])'; }
for rep in 1 2; do for c in 1 2 3 4; do for v in A C0 C; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4/ab_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(tail -1 gpurun_out/c4/ab_${v}_c${c}_$rep.log | summ)"
done; done; done
for c in 1 3; do for v in A C0 C; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/c4/tune_${v}_c${c}.log 2>&1
echo "tune $v c$c $(grep -v BEST gpurun_out/c4/tune_${v}_c${c}.log | tail -1)"
done; done
timeout 600 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --split > gpurun_out/c4/split_c1.log 2>&1; echo "split(two-launch) c1 $(tail -1 gpurun_out/c4/split_c1.log | summ)"
SF_FULLSIZE=1,2 SF_PARITY_OUT=gpurun_out/parity timeout 1200 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c4/full12.log 2>&1; tail -2 gpurun_out/c4/full12.log
