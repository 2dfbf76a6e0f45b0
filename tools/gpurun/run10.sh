mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/pytest10.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest10.log
