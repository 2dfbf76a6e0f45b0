set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv > gpurun_out/smi.txt
for c in 0 8192 4096; do GENINV_GRAM_CHUNK_ROWS=$c timeout 600 python tools/c4_rho.py >> gpurun_out/c4_rho.jsonl 2>> gpurun_out/c4_rho.err; done
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest1.log
