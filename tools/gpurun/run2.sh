mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gpurun/dbg_solve.py > gpurun_out/dbg_solve.log 2>&1
for c in 0 8192; do GENINV_GRAM_CHUNK_ROWS=$c timeout 600 python tools/c4_rho.py >> gpurun_out/c4_rho2.jsonl 2>> gpurun_out/c4_rho2.err; done
