set -x
for c in 2 4; do
timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --snap-half > gpurun_out/bench_c${c}_h.log 2>&1; tail -1 gpurun_out/bench_c${c}_h.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"], d["config"]["snapshots"])'
done
