set -x
mkdir -p gpurun_out
for pd in 0 2 4 8 12; do SF_L2_PREFETCH=$pd timeout 300 python scripts/tune.py --nt 100 --random-init --by 16 --chunks 2 > gpurun_out/tune_pd$pd.log 2>&1; echo PD=$pd; tail -1 gpurun_out/tune_pd$pd.log; done
for pd in 0 4 8; do SF_L2_PREFETCH=$pd timeout 300 python scripts/tune.py --config 3 --nt 30 --random-init --by 8 --chunks 4 > gpurun_out/tune3_pd$pd.log 2>&1; echo C3 PD=$pd; tail -1 gpurun_out/tune3_pd$pd.log; done
