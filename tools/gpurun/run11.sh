mkdir -p gpurun_out
timeout 1200 python tools/c5_full_report.py gpurun_out/c5_full.json > gpurun_out/c5_full.log 2>&1
