summ() { python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["gpu_launches"], (d.get("e2e") or {}).get("value"))' 2>&1 | tail -1; }
for v in "" "SF_LIB_PATH=$PWD/build/ab/libsf_L8.so"; do
env $v timeout 300 python bench.py --config 0 --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.log 2>&1; echo "c0 [$v] $(tail -1 /tmp/b.log | summ)"
done
