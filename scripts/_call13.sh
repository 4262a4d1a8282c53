mkdir -p gpurun_out/c13
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "wide_layout or autotune or all_orders" > gpurun_out/c13/t.log 2>&1; tail -3 gpurun_out/c13/t.log
for c in 3 4; do
timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2,3 --ctas 0 > gpurun_out/c13/tune_c$c.log 2>&1; cat gpurun_out/c13/tune_c$c.log | grep -v BEST
done
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"], d["config"]["kernel_tuning"])' 2>&1 | tail -1; }
for c in 3 4; do
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c13/b_c$c.log 2>&1; echo "bench c$c $(tail -1 gpurun_out/c13/b_c$c.log | summ)"
done
