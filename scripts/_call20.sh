timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "slab or one_launch or p2p" > /tmp/t.log 2>&1; tail -2 /tmp/t.log; grep -E "^E|FAILED" /tmp/t.log | head
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"])' 2>&1 | tail -1; }
for rep in 1 2; do for fl in "" "--split" "--split --one-launch"; do
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $fl > /tmp/b.log 2>&1; echo "c1 rep$rep [$fl] $(tail -1 /tmp/b.log | summ)"
done; done
for c in 1 3; do timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 > /tmp/tu.log 2>&1; echo "tune c$c $(grep -v BEST /tmp/tu.log | tail -1)"; done
