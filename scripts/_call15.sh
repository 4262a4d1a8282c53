mkdir -p gpurun_out/c15
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "loop2d or config0 or 2d or graph" > gpurun_out/c15/t.log 2>&1; tail -3 gpurun_out/c15/t.log; grep -E "^E|FAILED" gpurun_out/c15/t.log | head
summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["gpu_launches"], (d.get("e2e") or {}).get("value"))' 2>&1 | tail -1; }
timeout 300 python bench.py --config 0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c15/b0.log 2>&1; echo "c0 loop2d $(tail -1 gpurun_out/c15/b0.log | summ)"
timeout 300 python bench.py --config 0 --steps 5 --warmup 3 --no-cpu-baseline --graph > gpurun_out/c15/b0g.log 2>&1; echo "c0 loop2d+graph $(tail -1 gpurun_out/c15/b0g.log | summ)"
