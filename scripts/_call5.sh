mkdir -p gpurun_out/c5
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c5/gpu_tests.log 2>&1; tail -2 gpurun_out/c5/gpu_tests.log; grep FAILED gpurun_out/c5/gpu_tests.log | head
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["per_update_us"], d["clocks"]["sm_mhz"], d["gpu_launches"])' 2>&1 | tail -1; }
for rep in 1 2; do for c in 1 2 3 4; do for v in A C; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5/ab_${v}_c${c}_$rep.log 2>&1
echo "$v c$c rep$rep $(tail -1 gpurun_out/c5/ab_${v}_c${c}_$rep.log | summ)"
done; done; done
for c in 1 3; do for v in A C; do
SF_LIB_PATH=$PWD/build/ab/libsf_$v.so timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > gpurun_out/c5/tune_${v}_c${c}.log 2>&1
echo "tune $v c$c $(grep -v BEST gpurun_out/c5/tune_${v}_c${c}.log | tail -1)"
done; done
for c in 1 3; do
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --split > gpurun_out/c5/split2_c$c.log 2>&1; echo "split two-launch c$c $(tail -1 gpurun_out/c5/split2_c$c.log | summ)"
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --split --one-launch > gpurun_out/c5/split1_c$c.log 2>&1; echo "split one-launch c$c $(tail -1 gpurun_out/c5/split1_c$c.log | summ)"
done
SF_FULLSIZE=1,2 SF_PARITY_OUT=gpurun_out/parity timeout 1200 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c5/full12.log 2>&1; tail -2 gpurun_out/c5/full12.log
