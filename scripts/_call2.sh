mkdir -p gpurun_out/c2
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c2/smoke.log 2>&1; tail -2 gpurun_out/c2/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "slab_decomposition or high_order_damped" > gpurun_out/c2/gpu_tests.log 2>&1; tail -3 gpurun_out/c2/gpu_tests.log
for c in 2 3 4; do
SF_FULLSIZE=$c SF_PARITY_OUT=gpurun_out/parity timeout 3000 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c2/full$c.log 2>&1; tail -2 gpurun_out/c2/full$c.log
done
