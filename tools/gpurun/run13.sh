mkdir -p gpurun_out
GENINV_C5_RECORD=gpurun_out/r02_c5_full_parity.json timeout 1500 python -m pytest tests/test_gpu_c5_full.py -q -s -p no:cacheprovider > gpurun_out/c5_full_test.log 2>&1; echo "rc=$?" >> gpurun_out/c5_full_test.log
