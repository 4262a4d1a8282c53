set -x
mkdir -p gpurun_out
for rep in 1 2; do
for f in "" "--sep"; do timeout 300 python scripts/tune.py --config 1 --nt 40 --vy 2 --ctas 0 $f > gpurun_out/t.log 2>&1; echo "c1 $f $(grep -v BEST gpurun_out/t.log | tail -1)"; done
done
timeout 300 python scripts/tune.py --config 2 --grad --nt 40 --vy 2 --ctas 0 --sep > gpurun_out/t.log 2>&1; echo "c2g sep $(grep -v BEST gpurun_out/t.log | tail -1)"
timeout 300 python scripts/tune.py --config 2 --grad --nt 40 --vy 2 --ctas 0 > gpurun_out/t.log 2>&1; echo "c2g arr $(grep -v BEST gpurun_out/t.log | tail -1)"
