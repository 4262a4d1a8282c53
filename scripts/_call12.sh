mkdir -p gpurun_out/c12
SF_FULLSIZE=4 SF_PARITY_OUT=gpurun_out/parity timeout 1800 python -m pytest tests/test_fullsize_parity.py -q -s -p no:cacheprovider > gpurun_out/c12/full4.log 2>&1; tail -3 gpurun_out/c12/full4.log
