set -x
mkdir -p gpurun_out
for c in 0 2 3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 5 --no-e2e > gpurun_out/bench_c$c.log 2>&1; tail -1 gpurun_out/bench_c$c.log; done
timeout 600 python scripts/tune.py --config 3 --nt 40 --random-init --by 8 --chunks 0,1,2,3,4,5,6,8 > gpurun_out/tune_c3.log 2>&1; tail -1 gpurun_out/tune_c3.log
timeout 600 python scripts/tune.py --config 1 --nt 60 --grad --by 8,16 --chunks 0,2,4,7 > gpurun_out/tune_c1_grad.log 2>&1; tail -1 gpurun_out/tune_c1_grad.log
