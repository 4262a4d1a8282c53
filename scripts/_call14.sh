mkdir -p gpurun_out/c14
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "slab or one_launch or p2p or receiver_surface" > gpurun_out/c14/t.log 2>&1; tail -3 gpurun_out/c14/t.log; grep -E "^E|FAILED" gpurun_out/c14/t.log | head -20
