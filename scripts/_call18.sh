mkdir -p gpurun_out/c18
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1; }
for rep in 1 2 3; do for fl in "" "--split" "--split --one-launch"; do
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $fl > /tmp/b.log 2>&1; echo "c1 rep$rep [$fl] $(tail -1 /tmp/b.log | summ)"
done; done
SF_FULLSIZE=2h SF_PARITY_OUT=gpurun_out/parity timeout 1500 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c18/full2h.log 2>&1; tail -2 gpurun_out/c18/full2h.log
