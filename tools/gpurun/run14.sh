mkdir -p gpurun_out
timeout 3000 python -m pytest tests/test_gpu_c4_full.py tests/test_gpu_parity_report.py tests/test_gpu_parity.py -m slow -q -s -p no:cacheprovider > gpurun_out/slow14.log 2>&1; echo "rc=$?" >> gpurun_out/slow14.log
