mkdir -p gpurun_out/c1
(free -g; nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.sm,power.limit --format=csv) > gpurun_out/c1/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c1/smoke.log 2>&1; tail -2 gpurun_out/c1/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c1/gpu_tests.log 2>&1; tail -3 gpurun_out/c1/gpu_tests.log
SF_FULLSIZE=0,1 SF_PARITY_OUT=gpurun_out/parity timeout 1500 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c1/full01.log 2>&1; tail -3 gpurun_out/c1/full01.log
