mkdir -p gpurun_out/c8
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "slab or one_launch or receiver_surface or gradient or adjoint" > gpurun_out/c8/gpu_tests.log 2>&1; tail -2 gpurun_out/c8/gpu_tests.log
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["per_update_us"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1; }
for rep in 1 2; do for c in 2 1 4; do for fl in "" "--pdl" "--no-prof" "--pdl --no-prof"; do
tag=$(echo "x$fl" | tr -d ' -')
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $fl > gpurun_out/c8/b_${tag}_c${c}_$rep.log 2>&1
echo "c$c rep$rep [$fl] $(tail -1 gpurun_out/c8/b_${tag}_c${c}_$rep.log | summ)"
done; done; done
