set -x
mkdir -p gpurun_out
for c in 1 2; do timeout 300 python scripts/tune.py --config $c --nt 40 --vy 2 --ctas 0 --sep > gpurun_out/tune_sep_c$c.log 2>&1; grep -v BEST gpurun_out/tune_sep_c$c.log | tail -1; done
timeout 300 python scripts/tune.py --config 1 --nt 40 --vy 2 --ctas 0 > gpurun_out/tune_arr_c1.log 2>&1; grep -v BEST gpurun_out/tune_arr_c1.log | tail -1
timeout 300 python scripts/tune.py --config 2 --grad --nt 40 --vy 2 --ctas 0 --sep > gpurun_out/tune_sep_c2g.log 2>&1; grep -v BEST gpurun_out/tune_sep_c2g.log | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --damp-array > gpurun_out/bench_c1_arr.log 2>&1; tail -1 gpurun_out/bench_c1_arr.log
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
