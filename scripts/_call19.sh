summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1; }
for rep in 1 2; do for fl in "--split --one-launch" "--split --one-launch --prof-every 1" "--split --one-launch --no-pdl" "--split --one-launch --no-autotune" ""; do
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $fl > /tmp/b.log 2>&1; echo "c1 rep$rep [$fl] $(tail -1 /tmp/b.log | summ)"
done; done
