mkdir -p gpurun_out
GENINV_C5_DUMP=gpurun_out/c5_flagged.npz timeout 1200 python tools/c5_full_report.py gpurun_out/c5_full.json > gpurun_out/c5_full.log 2>&1
